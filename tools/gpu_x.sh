set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "conv" 2>&1 | tail -3 > gpurun_out/pytest_conv.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_conv" -c 4 --csv --log-file gpurun_out/launches_conv3.csv python tools/time_op.py '{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}' tc_tf32 3 > /dev/null 2>&1
timeout 120 python tools/time_noflush.py '{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}' > gpurun_out/noflush.log 2>&1
timeout 120 python tools/time_noflush.py '{"kind":"gemm","M":1024,"K":1024,"N":1024}' >> gpurun_out/noflush.log 2>&1
