# A/B on the GPU: GPU tests, then the bench (device timing only) under each
# environment setting given as arguments (e.g. "FM_SELECT_GROUPS=1").
# usage: bash scripts/gpu_ab.sh TAG [ENV=VAL ...]
TAG=${1:-ab}
shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${TAG}_base.json 2>&1; echo bench=$? >> gpurun_out/status_$TAG.txt
i=0
for kv in "$@"; do
  i=$((i+1))
  env $kv timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${TAG}_v$i.json 2>&1; echo "v$i($kv)=$?" >> gpurun_out/status_$TAG.txt
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo launches=$? >> gpurun_out/status_$TAG.txt
