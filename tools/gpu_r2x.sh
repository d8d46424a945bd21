mkdir -p gpurun_out
touch paper_2502_11407_b200/csrc/kernels/exec.cu; make -s -j8 -C paper_2502_11407_b200/csrc DEV=1 > /dev/null 2>&1
G='{"kind":"gemm","M":1024,"K":1024,"N":1024}'
for bn in 64 128 256; do for st in 4 6 8; do for cs in 1 2; do
  r=$(GENSOR_GEMM_BN=$bn GENSOR_GEMM_STAGES=$st GENSOR_GEMM_CLUSTER=$cs timeout 120 python tools/time_op.py "$G" tc_tf32 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us'], round(d['tflops'],1), d['plan'].get('stages'), d['plan'].get('cluster_n'))" 2>&1)
  echo "BN=$bn st=$st cs=$cs -> $r"
done; done; done
