set -x
mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
for b in 2 4; do GENSOR_PREPASS_BAND=$b python tools/time_op.py "$C" tc_tf32 30 > gpurun_out/x_b$b.log 2>&1; done
