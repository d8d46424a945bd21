mkdir -p gpurun_out
V='{"kind":"gemv","M":32768,"N":4096}'
timeout 300 ncu --set full -k regex:"k_simt_gemv" -s 1 -c 1 -o gpurun_out/r2w_gemv -f python tools/time_op.py "$V" simt_f32 2 > gpurun_out/r2w.log 2>&1
tail -2 gpurun_out/r2w.log
