set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_x.log
for w in avgpool dwconv; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; done
