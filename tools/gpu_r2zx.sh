mkdir -p gpurun_out
rm -rf paper_2502_11407_b200/build; make -s -j$(nproc) -C paper_2502_11407_b200/csrc DEV=1 2>&1 | grep -v warning | tail -1
for op in '{"kind":"gemm","M":1024,"K":1024,"N":1024}' '{"kind":"gemm","M":512,"K":64,"N":512,"dtype_bytes":2,"batch":192}' '{"kind":"gemm","M":8192,"K":768,"N":2304,"dtype_bytes":2}' '{"kind":"gemm","M":8192,"K":768,"N":768,"dtype_bytes":2}'; do
  for pp in 0 1; do echo "$op pair=$pp"; GENSOR_GEMM_PAIR=$pp timeout 120 python tools/time_op.py "$op" auto 30 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['us'], round(d['tflops'],1), d['plan'].get('cta_pair'), d['plan'].get('BN'))"; done
done
