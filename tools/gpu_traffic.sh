# DRAM traffic of every launch of one execute per bench workload (timed-step L2 state: our own
# 256 MiB flush before the execute, ncu cache control off), for the roofline "traffic" field:
# tools/traffic_merge.py sums the launches into profiles/ncu_traffic.json.
mkdir -p gpurun_out/traffic
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,gpu__time_duration.sum
for w in conv2d gemm gemm_fp32 bgemm rowsum softmax dwconv avgpool; do
  timeout 300 ncu --nvtx --nvtx-include "traffic/" --cache-control none --clock-control none --metrics $M --csv \
    --log-file gpurun_out/traffic/$w.csv python tools/traffic.py $w > gpurun_out/traffic/$w.json 2> gpurun_out/traffic/$w.err
done
python tools/traffic_merge.py gpurun_out/traffic > gpurun_out/traffic/merged.json
cat gpurun_out/traffic/merged.json
