set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_sequences.py tests/test_gpu_host_pipe.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_x.log
for L in '{"kind":"conv2d","I":[128,256,14,14],"K":[1024,256,1,1],"S":1}' '{"kind":"conv2d","I":[128,1024,14,14],"K":[256,1024,1,1],"S":1}'; do
python tools/time_op.py "$L" tc_tf32 10 >> gpurun_out/x_chunk.log 2>&1
GENSOR_CONV1X1_GEMM=0 python tools/time_op.py "$L" tc_tf32 10 >> gpurun_out/x_chunk0.log 2>&1
done
