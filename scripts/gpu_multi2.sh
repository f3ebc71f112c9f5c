# bash scripts/gpu_multi2.sh TAG NG : N=1 A/B (concurrent buckets) and N=NG with B=1,2,4
TAG=$1; NG=${2:-2}
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-parity --no-e2e > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err; echo n1=$? >> gpurun_out/status_$TAG.txt
FM_BUILD_CONCURRENT=0 timeout 600 python bench.py --no-cpu --no-parity --no-e2e > gpurun_out/bench_${TAG}_n1seq.json 2> gpurun_out/bench_${TAG}_n1seq.err; echo n1seq=$? >> gpurun_out/status_$TAG.txt
for B in 1 2 4; do
timeout 900 python bench.py --gpus $NG --blocks $B --no-cpu --no-parity --no-e2e > gpurun_out/bench_${TAG}_n${NG}_b$B.json 2> gpurun_out/bench_${TAG}_n${NG}_b$B.err; echo n${NG}_b$B=$? >> gpurun_out/status_$TAG.txt
done
