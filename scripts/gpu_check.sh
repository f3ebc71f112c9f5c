# GPU tests, two bench runs (device timing) and a warm launch list.
mkdir -p gpurun_out
T=${1:-ck}
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${T}.log 2>&1; echo pytest=$? >> gpurun_out/status_$T.txt
for rep in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${T}_base_$rep.json 2>&1; echo bench_$rep=$? >> gpurun_out/status_$T.txt
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/warm_$T.csv $CMD > gpurun_out/ncu_warm_$T.log 2>&1; echo warm=$? >> gpurun_out/status_$T.txt
