mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_generic.py -m gpu -q -p no:cacheprovider -k "3xtf32 or full_size" > gpurun_out/r2c_pytest.log 2>&1
tail -30 gpurun_out/r2c_pytest.log
