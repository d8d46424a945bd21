mkdir -p gpurun_out
timeout 300 python tools/x3_probe.py 1024x1024x1024 512x1024x512 > gpurun_out/r2f_x3a.log 2>&1; tail -5 gpurun_out/r2f_x3a.log
timeout 300 python tools/x3_probe.py 128x64x64 > gpurun_out/r2f_x3b.log 2>&1; tail -5 gpurun_out/r2f_x3b.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tools/x3_probe.py 128x64x64 > gpurun_out/r2f_x3c.log 2>&1; head -60 gpurun_out/r2f_x3c.log
