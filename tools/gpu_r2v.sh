mkdir -p gpurun_out
G='{"kind":"gemm","M":1024,"K":1024,"N":1024}'
timeout 300 ncu --set full --import-source on -k regex:"k_simt_gemm" -s 1 -c 1 -o gpurun_out/r2v_simt -f python tools/time_op.py "$G" simt_f32 2 > gpurun_out/r2v.log 2>&1
tail -2 gpurun_out/r2v.log
