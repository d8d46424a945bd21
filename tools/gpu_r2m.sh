mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_conv_flat" -s 2 -c 1 -o gpurun_out/r2m_flat2 -f python tools/time_op.py "$C" tc_tf32 3 > gpurun_out/r2m_ncu.log 2>&1
tail -2 gpurun_out/r2m_ncu.log
