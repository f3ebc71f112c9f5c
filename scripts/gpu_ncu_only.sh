# ncu --set full of the hot kernels of one bench step (after a plain run of the same command).
TAG=${1:-n}
REGEX=${2:-"k_build|k_select|k_apply"}
CONFIG=${3:-c2}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --config $CONFIG"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$REGEX" -c ${4:-3} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncufull=$? >> gpurun_out/status_$TAG.txt
