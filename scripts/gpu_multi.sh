# Multi-GPU check: map_gathered test, then bench at N=1 and N=$NG (spawned
# ranks, --gpus) with 1/2/4 blocks.  bash scripts/gpu_multi.sh TAG NG
TAG=$1; NG=${2:-2}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k map_gathered > gpurun_out/pytest_multi_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
timeout 600 python bench.py --no-cpu --no-parity > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err; echo n1=$? >> gpurun_out/status_$TAG.txt
for B in 1 2 4 8; do
timeout 900 python bench.py --gpus $NG --blocks $B --no-cpu --no-parity > gpurun_out/bench_${TAG}_n${NG}_b$B.json 2> gpurun_out/bench_${TAG}_n${NG}_b$B.err; echo n${NG}_b$B=$? >> gpurun_out/status_$TAG.txt
done
