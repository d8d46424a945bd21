set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "gemm" 2>&1 | tail -15 > gpurun_out/pytest_gemm.log
for w in gemm bgemm; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; done
timeout 600 python bench.py --workload gpt2 --steps 3 --warmup 3 > gpurun_out/bench_gpt2.log 2>&1
