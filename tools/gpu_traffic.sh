# DRAM traffic of each workload's dominant kernel (ncu, one launch after warm-up), for the
# roofline "traffic" field: profiles/ncu_traffic.json
set -x
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
run() { timeout 300 ncu --metrics $M --clock-control none -k regex:"$2" -s 3 -c 1 --csv --log-file gpurun_out/traffic_$1.csv python tools/time_op.py "$3" auto 1 > /dev/null 2>&1; }
run conv2d "k_conv_ns|k_conv_tc" '{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
run gemm "k_gemm_tc" '{"kind":"gemm","M":1024,"K":1024,"N":1024}'
run bgemm "k_gemm_tc" '{"kind":"gemm","M":512,"K":64,"N":512,"dtype_bytes":2,"batch":192}'
run rowsum "k_gemv" '{"kind":"gemv","M":32768,"N":4096}'
run softmax "k_softmax" '{"kind":"softmax","M":32768,"N":4096}'
run dwconv "k_window" '{"kind":"dwconv2d","I":[32,256,114,114],"K":[256,1,3,3],"S":1}'
run avgpool "k_window" '{"kind":"avgpool2d","I":[32,256,114,114],"F":3,"S":1}'
