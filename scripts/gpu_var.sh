# A/B of library variants on the GPU (bench device timing only):
# bash scripts/gpu_var.sh TAG VARIANT [VARIANT ...]  (VARIANT = name under _lib/var)
TAG=$1; shift
mkdir -p gpurun_out
timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${TAG}_base.json 2>&1; echo base=$? >> gpurun_out/status_$TAG.txt
for v in "$@"; do
  FM_LIB_PATH=$PWD/paper_2510_18838_b200/_lib/var/libfieldmap_$v.so timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${TAG}_$v.json 2>&1; echo $v=$? >> gpurun_out/status_$TAG.txt
done
