# Final-tree checks: GPU suite, the FM_DEBUG bounds-checked suite, C1 and C3 bench lines.
mkdir -p gpurun_out
T=${1:-fin}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${T}.log 2>&1; echo pytest=$? >> gpurun_out/status_$T.txt
FM_LIB_PATH=$PWD/paper_2510_18838_b200/_lib/var/libfieldmap_debug.so timeout 2400 \
  python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_debug_${T}.log 2>&1; echo debug=$? >> gpurun_out/status_$T.txt
timeout 600 python bench.py --config c1 > gpurun_out/bench_${T}_c1.json 2> gpurun_out/bench_${T}_c1.err; echo c1=$? >> gpurun_out/status_$T.txt
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 > gpurun_out/bench_${T}_c3.json 2> gpurun_out/bench_${T}_c3.err; echo c3=$? >> gpurun_out/status_$T.txt
