# Grid density A/B with the full parity block (the eager path and the graph use the same density).
mkdir -p gpurun_out
T=${1:-dn}
for c in 0.5 0.35 0.25; do
  FM_CELLS_PER_POINT=$c timeout 400 python bench.py --no-e2e --no-cpu > gpurun_out/bench_${T}_c$c.json 2>&1; echo c$c=$? >> gpurun_out/status_$T.txt
done
timeout 400 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${T}_base.json 2>&1; echo base=$? >> gpurun_out/status_$T.txt
