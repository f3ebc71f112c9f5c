# Full-scale C3/C4/C5 on one GPU
TAG=$1
mkdir -p gpurun_out
for c in c3 c3mq c4 c5; do
timeout 1500 python bench.py --config $c --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo $c=$? >> gpurun_out/status_$TAG.txt
done
