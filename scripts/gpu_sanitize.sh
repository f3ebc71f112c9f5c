# compute-sanitizer over small cases of every kernel: bash scripts/gpu_sanitize.sh TAG TOOL
TAG=$1; TOOL=${2:-memcheck}
mkdir -p gpurun_out
K="supports_beyond_256 or patch_supports_random or c1_supports_bitwise or adaptive_supports_bitwise or fit_many_variants or prepared_transfer_adaptive or extension_nd_vs_oracle or apply_local_rows or locate_batch_bitwise or patch_supports_bitwise or all_size_buckets or map_chunked or per_axis_metric or singular_transfer or empty_targets or map_gathered"
timeout 2400 compute-sanitizer --tool $TOOL --error-exitcode 99 --print-limit 50 --log-file gpurun_out/sanitize_${TAG}_$TOOL.txt \
  python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$K" > gpurun_out/sanitize_${TAG}_${TOOL}_pytest.log 2>&1
echo "$TOOL rc=$?" >> gpurun_out/status_$TAG.txt
