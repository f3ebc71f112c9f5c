# Full GPU test suite + large configs at a reduced scale
TAG=$1; SCALE=${2:-0.125}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
for c in c3 c3mq; do
timeout 1200 python bench.py --config $c --scale $SCALE --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo $c=$? >> gpurun_out/status_$TAG.txt
done
timeout 600 python bench.py --no-e2e --no-cpu --no-parity > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; echo c2=$? >> gpurun_out/status_$TAG.txt
