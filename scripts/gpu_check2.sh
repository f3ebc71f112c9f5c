# GPU tests, the default bench with its parity block, and C3 at both grid densities.
mkdir -p gpurun_out
T=${1:-ck}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${T}.log 2>&1; echo pytest=$? >> gpurun_out/status_$T.txt
timeout 400 python bench.py --no-e2e --no-cpu > gpurun_out/bench_${T}_base.json 2>&1; echo bench=$? >> gpurun_out/status_$T.txt
timeout 600 python bench.py --no-e2e --no-cpu --config c3 > gpurun_out/bench_${T}_c3.json 2>&1; echo c3=$? >> gpurun_out/status_$T.txt
FM_CELLS_PER_POINT=1.0 timeout 600 python bench.py --no-e2e --no-cpu --no-parity --config c3 > gpurun_out/bench_${T}_c3d1.json 2>&1; echo c3d1=$? >> gpurun_out/status_$T.txt
