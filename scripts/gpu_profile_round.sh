# One GPU call: GPU tests, the bench, and ncu evidence for the top kernels.
# usage (from the repo root on the GPU box): bash scripts/gpu_profile_round.sh [tag]
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench=$? >> gpurun_out/status_$TAG.txt
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo launches=$? >> gpurun_out/status_$TAG.txt
# (the ncu --set full capture is a separate gpurun call: scripts/gpu_ncu_only.sh)
