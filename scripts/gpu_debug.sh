# Bounds-checked run of the whole GPU suite (compute-sanitizer is closed on
# this pool): build the variant first, here, with
#   python scripts/build_variant.py debug -DFM_DEBUG
# (every FM_DCHECK in csrc/ active: printf + __trap on a failed check), then
#   gpurun -- bash scripts/gpu_debug.sh
mkdir -p gpurun_out
FM_LIB_PATH=$PWD/paper_2510_18838_b200/_lib/var/libfieldmap_debug.so timeout 2400 \
  python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_debug.log 2>&1
echo debug=$? >> gpurun_out/pytest_debug.log
