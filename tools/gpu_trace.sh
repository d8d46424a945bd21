set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k conv 2>&1 | tail -5 > gpurun_out/pytest_tc.log
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
for v in tc_tf32 tc_bf16; do timeout 120 python tools/time_op.py "$C" $v >> gpurun_out/conv_v3.log 2>&1; done
GENSOR_CONV_TRACE=gpurun_out/conv3_trace.txt timeout 120 python tools/time_op.py "$C" tc_tf32 3 > /dev/null 2>&1
