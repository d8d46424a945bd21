set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_all_gpu.log
bash tools/gpu_full.sh
timeout 600 python tools/sweep_seq.py resnet50 > gpurun_out/sweep_resnet.log 2>&1
