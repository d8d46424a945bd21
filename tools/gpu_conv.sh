# GPU-box batch: tensor-core conv/gemm evidence (bench lines, per-launch breakdown, ncu captures).
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q -k "avgpool or window" 2>&1 | tail -5 > gpurun_out/pytest_stream2.log
timeout 300 python bench.py --workload avgpool --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_avgpool.log 2>&1
for w in conv2d gemm bgemm; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; done
timeout 300 python bench.py --workload conv2d --variant tc_bf16 --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/bench_conv2d_bf16.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_conv.csv python bench.py --workload conv2d --steps 3 --warmup 3 --suite "" --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_conv_tc|k_nchw|k_weights" -s 3 -c 3 -o gpurun_out/prof_conv -f python bench.py --workload conv2d --steps 1 --warmup 3 --suite "" --no-cpu-baseline > gpurun_out/ncu_conv.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc" -s 3 -c 1 -o gpurun_out/prof_gemm -f python bench.py --workload gemm --steps 1 --warmup 3 --suite "" --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
