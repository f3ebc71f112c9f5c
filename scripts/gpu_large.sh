# Large configs: new GPU tests, then c3/c3mq/c4/c5 at a reduced scale (checks)
TAG=$1; SCALE=${2:-0.125}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "metric or chunked" > gpurun_out/pytest_large_$TAG.log 2>&1; echo pytest=$? >> gpurun_out/status_$TAG.txt
for c in c3 c3mq c4 c5; do
timeout 1200 python bench.py --config $c --scale $SCALE --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo $c=$? >> gpurun_out/status_$TAG.txt
done
