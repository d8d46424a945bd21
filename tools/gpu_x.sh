set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "gemm" 2>&1 | tail -3 > gpurun_out/pytest_gemm.log
timeout 300 python bench.py --workload bgemm --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_bgemm.log 2>&1
timeout 600 python bench.py --workload gpt2 --steps 3 --warmup 3 > gpurun_out/bench_gpt2.log 2>&1
