mkdir -p gpurun_out
timeout 300 python tools/x3_probe.py 128x128x64 128x160x64 128x256x64 128x1024x64 1024x64x1024 256x512x128 > gpurun_out/r2g_x3.log 2>&1; cat gpurun_out/r2g_x3.log | grep -v "^$" | tail -14
