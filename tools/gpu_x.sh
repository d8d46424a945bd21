set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sequences.py tests/test_gpu_host_pipe.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_x.log
timeout 600 python tools/sweep_seq.py resnet50 > gpurun_out/sweep_resnet.log 2>&1
timeout 900 python bench.py --workload resnet50 --steps 3 --warmup 3 > gpurun_out/bench_resnet50.log 2>&1
