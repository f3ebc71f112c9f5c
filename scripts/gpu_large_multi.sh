# C3 (strong) and C5 (weak) at N = 2 and NG ranks (spawned), full scale
TAG=$1; NG=${2:-4}
mkdir -p gpurun_out
for n in 2 $NG; do
for c in c3 c5; do
timeout 1500 python bench.py --config $c --gpus $n --steps 2 --warmup 1 --no-parity > gpurun_out/bench_${TAG}_${c}_n$n.json 2> gpurun_out/bench_${TAG}_${c}_n$n.err; echo ${c}_n$n=$? >> gpurun_out/status_$TAG.txt
done
done
