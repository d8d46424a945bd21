set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q -k "conv or s2d" 2>&1 | tail -5 > gpurun_out/pytest_x.log
L2='{"kind":"conv2d","I":[128,512,9,9],"K":[512,512,3,3],"S":1}'
python tools/time_op.py "$L2" tc_tf32 10 > gpurun_out/x_l2_tc.log 2>&1
GENSOR_CONV_FAMILY=gemm python tools/time_op.py "$L2" tc_tf32 10 > gpurun_out/x_l2_gemm.log 2>&1
