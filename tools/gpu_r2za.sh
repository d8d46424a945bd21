mkdir -p gpurun_out
touch paper_2502_11407_b200/csrc/kernels/exec.cu paper_2502_11407_b200/csrc/kernels/conv_flat.cu; make -s -j8 -C paper_2502_11407_b200/csrc DEV=1 > /dev/null 2>&1
bash tools/gpu_r2n.sh
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider -k "conv_tc" > gpurun_out/r2za_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2za_tests.log
