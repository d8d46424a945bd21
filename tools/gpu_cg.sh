set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "conv_gemm" 2>&1 | tail -30 > gpurun_out/pytest_cg.log
timeout 900 python bench.py --workload resnet50 --steps 3 --warmup 3 > gpurun_out/bench_resnet50.log 2>&1
