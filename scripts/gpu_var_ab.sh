# A/B of variant libraries (scripts/build_variant.py NAME ...) against the
# in-tree build, alternating, device timing only.
# usage: bash scripts/gpu_var_ab.sh TAG NAME...
mkdir -p gpurun_out
T=$1; shift
V=$PWD/paper_2510_18838_b200/_lib/var
for rep in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${T}_base_$rep.json 2>&1; echo base_$rep=$? >> gpurun_out/status_$T.txt
  for v in "$@"; do
    FM_LIB_PATH=$V/libfieldmap_$v.so timeout 300 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${T}_${v}_$rep.json 2>&1; echo ${v}_$rep=$? >> gpurun_out/status_$T.txt
  done
done
