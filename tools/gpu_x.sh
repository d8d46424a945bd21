set -x
mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_host_pipe.py -x -q -k "conv or s2d" 2>&1 | tail -3 > gpurun_out/pytest_x.log
python tools/time_op.py "$C" tc_tf32 30 > gpurun_out/x_p2.log 2>&1
GENSOR_PREPASS2=0 python tools/time_op.py "$C" tc_tf32 30 > gpurun_out/x_p1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 6 --csv --log-file gpurun_out/x_p2_launches.csv python tools/time_op.py "$C" tc_tf32 2 > /dev/null 2>&1
