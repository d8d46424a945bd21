set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q -k softmax 2>&1 | tail -3 > gpurun_out/pytest_x.log
python tools/time_op.py '{"kind":"softmax","M":98304,"N":512}' auto 20 > gpurun_out/x_sm512.log 2>&1
python tools/time_op.py '{"kind":"softmax","M":32768,"N":4096}' auto 20 > gpurun_out/x_sm4096.log 2>&1
python tools/time_op.py '{"kind":"softmax","M":65536,"N":256}' auto 20 > gpurun_out/x_sm256.log 2>&1
