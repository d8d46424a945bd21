set -x
mkdir -p gpurun_out
timeout 300 python bench.py --workload conv2d --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_conv2d.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_conv" -c 20 --csv --log-file gpurun_out/launches_conv2.csv python tools/time_op.py '{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}' tc_tf32 5 > /dev/null 2>&1
