# ncu --set full of one kernel regex with a library variant: bash scripts/gpu_ncu_var.sh TAG REGEX VARIANT [COUNT]
TAG=$1; REGEX=$2; VAR=$3; CNT=${4:-1}
mkdir -p gpurun_out
if [ "$VAR" != base ]; then export FM_LIB_PATH=$PWD/paper_2510_18838_b200/_lib/var/libfieldmap_$VAR.so; fi
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$REGEX" -c $CNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncufull=$? >> gpurun_out/status_$TAG.txt
