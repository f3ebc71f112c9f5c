# Quick GPU check: GPU tests + a short bench (no e2e / cpu legs) + launch list.
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench=$? >> gpurun_out/status_$TAG.txt
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo launches=$? >> gpurun_out/status_$TAG.txt
