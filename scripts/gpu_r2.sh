# Round-2 GPU check: all GPU tests, the bench with parity/e2e/cpu legs, the
# reference arm, and a launch list.  Usage: bash scripts/gpu_r2.sh TAG [pytest-args]
TAG=${1:-r2}
shift
mkdir -p gpurun_out
nproc > gpurun_out/nproc_$TAG.txt; lscpu >> gpurun_out/nproc_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$? >> gpurun_out/status_$TAG.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; echo ref=$? >> gpurun_out/status_$TAG.txt
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo launches=$? >> gpurun_out/status_$TAG.txt
