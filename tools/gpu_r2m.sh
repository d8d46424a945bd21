mkdir -p gpurun_out
touch paper_2502_11407_b200/csrc/kernels/exec.cu paper_2502_11407_b200/csrc/kernels/conv_flat.cu; make -s -j8 -C paper_2502_11407_b200/csrc > /dev/null 2>&1
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 -k regex:"k_conv_flat_pair" -s 2 -c 1 -o gpurun_out/r2m_pair -f python tools/time_op.py "$C" tc_tf32 3 > gpurun_out/r2m_ncu.log 2>&1
tail -2 gpurun_out/r2m_ncu.log
