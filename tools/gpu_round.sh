# GPU-box batch: parity tests, bench lines, launch list + one full ncu capture per hot kernel.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -40 > gpurun_out/pytest_stream.log
for w in rowsum softmax dwconv avgpool; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; done
for k in k_gemv_bulk k_window_bulk; do w=rowsum; [ $k = k_window_bulk ] && w=dwconv
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k -f python bench.py --workload $w --steps 1 --warmup 3 --suite "" --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1; done
