set -x
mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
for x in 0 7; do
GENSOR_CONV_XFLAGS=$x GENSOR_CONV_TRACE=gpurun_out/conv_trace_x$x.txt timeout 120 python tools/time_op.py "$C" tc_tf32 5 >> gpurun_out/conv_x2.log 2>&1
done
