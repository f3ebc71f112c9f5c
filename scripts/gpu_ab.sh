# A/B timing of library variants: bash scripts/gpu_ab.sh TAG name1 name2 ...
# ("base" = the in-tree libfieldmap.so; others = _lib/var/libfieldmap_NAME.so)
TAG=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then unset FM_LIB_PATH; else export FM_LIB_PATH=$PWD/paper_2510_18838_b200/_lib/var/libfieldmap_$v.so; fi
  for rep in 1 2; do
    timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/ab_${TAG}_${v}_$rep.log 2>&1
    echo "$v rep$rep rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}_${v}_$rep.log) $(grep -o '"phases_ms_per_step": {[^}]*}' gpurun_out/ab_${TAG}_${v}_$rep.log)" >> gpurun_out/ab_$TAG.txt
  done
done
