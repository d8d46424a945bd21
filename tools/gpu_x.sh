set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "conv" 2>&1 | tail -3 > gpurun_out/pytest_conv.log
timeout 120 python tools/time_noflush.py '{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}' > gpurun_out/noflush.log 2>&1
timeout 300 python bench.py --workload conv2d --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_conv2d.log 2>&1
