set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -25 > gpurun_out/pytest_tc.log
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
for v in tc_tf32 tc_bf16; do timeout 120 python tools/time_op.py "$C" $v >> gpurun_out/conv_v2.log 2>&1; done
timeout 300 python bench.py --workload conv2d --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_conv2d.log 2>&1
