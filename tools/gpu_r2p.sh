mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2p_launch.csv python tools/time_op.py "$C" tc_tf32 3 > /dev/null 2>&1
python - <<'P'
import csv
rows=list(csv.reader(open("gpurun_out/r2p_launch.csv")))
h=[r for r in rows if "Kernel Name" in r][0]; i0=rows.index(h)
ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
for r in rows[i0+1:]:
    if "flat" in r[ki] or "gb::" in r[ki]: print(r[ki][:40], r[mi], r[vi])
P
