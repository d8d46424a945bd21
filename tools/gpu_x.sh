set -x
mkdir -p gpurun_out
for w in gemm conv2d bgemm; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; done
