set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_pipe.py tests/test_capi.py -x -q 2>&1 | tail -25 > gpurun_out/pytest_pipe.log
timeout 600 python bench.py --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_conv2d.log 2>&1
GENSOR_HOST_PIPE=0 timeout 600 python bench.py --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_conv2d_nopipe.log 2>&1
