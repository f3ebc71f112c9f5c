# Weak-scaling check of the default bench at N = 1, 2, NG (spawned ranks).
TAG=$1; NG=${2:-4}
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-parity --no-e2e > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err; echo n1=$? >> gpurun_out/status_$TAG.txt
for n in 2 $NG; do
timeout 900 python bench.py --gpus $n --no-cpu --no-parity > gpurun_out/bench_${TAG}_n$n.json 2> gpurun_out/bench_${TAG}_n$n.err; echo n$n=$? >> gpurun_out/status_$TAG.txt
done
timeout 900 python bench.py --gpus $NG --no-cpu --no-parity --no-e2e --no-graph > gpurun_out/bench_${TAG}_n${NG}_nograph.json 2> gpurun_out/bench_${TAG}_n${NG}_nograph.err; echo n${NG}_nograph=$? >> gpurun_out/status_$TAG.txt
