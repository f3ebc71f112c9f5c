# GPU tests + full default bench (e2e + cpu legs): bash scripts/gpu_bench_full.sh TAG
TAG=${1:-b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench=$? >> gpurun_out/status_$TAG.txt
timeout 300 python scripts/e2e_breakdown.py > gpurun_out/e2e_bd_$TAG.txt 2>&1
