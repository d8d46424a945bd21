set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "conv" 2>&1 | tail -3 > gpurun_out/pytest_cg.log
timeout 900 python tools/sweep_seq.py resnet50 > gpurun_out/sweep_resnet.log 2>&1
