mkdir -p gpurun_out
touch paper_2502_11407_b200/csrc/kernels/exec.cu paper_2502_11407_b200/csrc/kernels/conv_tc.cu paper_2502_11407_b200/csrc/kernels/gemm_tc.cu
make -s -j8 -C paper_2502_11407_b200/csrc DEV=1 2>&1 | grep -v spilled | head -5
for d in 0 1 2 3; do echo "dbg=$d"; GENSOR_X3_DBG=$d timeout 300 python tools/x3_probe.py 128x256x64 1024x64x1024 2>&1 | grep 3xtf32; done > gpurun_out/r2h_x3.log
cat gpurun_out/r2h_x3.log
timeout 300 python tools/conv_trace.py > gpurun_out/r2h_conv_trace.log 2>&1; cat gpurun_out/r2h_conv_trace.log
