# A/B of environment settings on the default bench (device timing only),
# alternating with the baseline.  usage: bash scripts/gpu_env_ab.sh TAG "ENV=V" ...
# (extra bench arguments in $BENCH_ARGS, e.g. BENCH_ARGS="--config c3")
mkdir -p gpurun_out
T=$1; shift
for rep in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-parity $BENCH_ARGS > gpurun_out/bench_${T}_base_$rep.json 2>&1; echo base_$rep=$? >> gpurun_out/status_$T.txt
  i=0
  for kv in "$@"; do
    i=$((i+1))
    env $kv timeout 300 python bench.py --no-e2e --no-cpu --no-parity $BENCH_ARGS > gpurun_out/bench_${T}_v${i}_$rep.json 2>&1; echo "v${i}_$rep($kv)=$?" >> gpurun_out/status_$T.txt
  done
done
