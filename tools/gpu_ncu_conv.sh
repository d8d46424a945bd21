# Headline conv: ncu launch list of the bench command (per-launch times, cold/serialised) and one
# `--set full` capture of the conv kernel, summarised into profiles/ncu/ by the caller.
set -x
mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --suite "" --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_conv_ns|k_conv_tc" -s 2 -c 1 -o gpurun_out/prof_conv -f python tools/time_op.py "$C" tc_tf32 3 > gpurun_out/ncu_conv.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:"k_conv_ns|k_conv_tc" -s 3 -c 1 --csv --log-file gpurun_out/traffic_conv2d.csv python tools/time_op.py "$C" auto 1 > /dev/null 2>&1
