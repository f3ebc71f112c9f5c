# Warm-cache per-kernel durations of one bench step (ncu --cache-control none):
# the GPU-busy part of the step, to set against its wall (event) time.
TAG=$1
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/warm_$TAG.csv $CMD > gpurun_out/ncu_warm_$TAG.log 2>&1; echo warm=$? >> gpurun_out/status_$TAG.txt
