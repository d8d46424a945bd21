mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python tools/x3_probe.py 128x256x64 1024x64x1024 1024x1024x1024 2>&1 | grep 3xtf32; done > gpurun_out/r2i_x3.log
cat gpurun_out/r2i_x3.log
