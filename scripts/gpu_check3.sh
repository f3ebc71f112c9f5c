# GPU tests + C2 bench + C3 bench (5 steps).
mkdir -p gpurun_out
T=${1:-ck}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${T}.log 2>&1; echo pytest=$? >> gpurun_out/status_$T.txt
for rep in 1 2; do
timeout 400 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${T}_c2_$rep.json 2>&1; echo c2_$rep=$? >> gpurun_out/status_$T.txt
done
timeout 600 python bench.py --no-e2e --no-cpu --no-parity --config c3 --steps 4 --warmup 3 > gpurun_out/bench_${T}_c3.json 2>&1; echo c3=$? >> gpurun_out/status_$T.txt
