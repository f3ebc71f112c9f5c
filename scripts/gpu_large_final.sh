# Final-tree large configs: C3/C3MQ/C4/C5 at N = 1 (full scale, sampled parity),
# then C3 (strong) and C5 (weak) at N = 2 and 4.  Run with gpurun --gpus 4.
TAG=${1:-lf}
mkdir -p gpurun_out
for c in c3 c3mq c4 c5; do
timeout 1500 python bench.py --config $c --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_${c}_n1.json 2> gpurun_out/bench_${TAG}_${c}_n1.err; echo ${c}_n1=$? >> gpurun_out/status_$TAG.txt
done
for n in 2 4; do
for c in c3 c5; do
timeout 1500 python bench.py --config $c --gpus $n --steps 2 --warmup 1 --no-parity > gpurun_out/bench_${TAG}_${c}_n$n.json 2> gpurun_out/bench_${TAG}_${c}_n$n.err; echo ${c}_n$n=$? >> gpurun_out/status_$TAG.txt
done
done
