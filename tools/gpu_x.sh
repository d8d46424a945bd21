set -x
mkdir -p gpurun_out
G='{"kind":"gemm","M":1024,"K":1024,"N":1024}'
for cs in 1 2 4 8; do GENSOR_GEMM_CLUSTER=$cs python tools/time_op.py "$G" tc_tf32 30 > gpurun_out/g_cs$cs.log 2>&1; done
GENSOR_GEMM_CLUSTER=8 timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "gemm" 2>&1 | tail -3 > gpurun_out/pytest_g8.log
