set -x
mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
python tools/time_op.py "$C" tc_tf32 30 > gpurun_out/x_tile.log 2>&1
S='{"kind":"conv2d","I":[128,3,229,229],"K":[64,3,7,7],"S":2}'
python tools/time_op.py "$S" tc_tf32 10 > gpurun_out/x_stem_tile.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/smi.log
