mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2zg_pytest_gpu.log 2>&1; tail -2 gpurun_out/r2zg_pytest_gpu.log
S=/usr/local/cuda/bin/compute-sanitizer
op='{"kind":"gemm","M":512,"K":128,"N":512,"dtype_bytes":2,"batch":40}'
timeout 600 $S --tool memcheck python tools/run_once.py "$op" tc_bf16 2>&1 | grep -E "ERROR SUMMARY|cta_pair" | sed 's/.*"cta_pair": \([a-z]*\).*/cta_pair=\1/'
timeout 600 $S --tool synccheck python tools/run_once.py "$op" tc_bf16 2>&1 | grep -E "ERROR SUMMARY"
timeout 900 python bench.py --workload gpt2 --steps 10 --warmup 3 > gpurun_out/r2zg_gpt2.jsonl 2> gpurun_out/r2zg_gpt2.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zg_gpt2.jsonl").read().strip().splitlines()[-1])
print(round(d["value"],1), round(d["ms_per_step"],3))
for k,v in d["per_op"].items(): print(" ", k, v["n"], round(v["ms"],3), round(v["tflops"],1), round(v["gbs"],0), v["variant"])
P
