# Round-2 evidence: GPU tests, the default bench (all legs), launch list, and
# ncu --set full of the top kernels (each after its command ran clean).
TAG=${1:-r2final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$? >> gpurun_out/status_$TAG.txt
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 ; echo launches=$? >> gpurun_out/status_$TAG.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_select_t|k_build|k_apply" -c 5 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncufull=$? >> gpurun_out/status_$TAG.txt
timeout 900 python bench.py --impl reference > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; echo ref=$? >> gpurun_out/status_$TAG.txt
