mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2j_pytest_gpu.log 2>&1
tail -15 gpurun_out/r2j_pytest_gpu.log
