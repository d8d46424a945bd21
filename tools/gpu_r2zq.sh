mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2zq_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2zq_pytest_gpu.log
S=/usr/local/cuda/bin/compute-sanitizer
for op in '{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}' '{"kind":"gemm","M":512,"K":128,"N":512,"dtype_bytes":2,"batch":40}' '{"kind":"gemm","M":1024,"K":1024,"N":1024}' '{"kind":"conv2d","I":[2,128,14,14],"K":[128,128,3,3],"S":1}'; do
  for t in memcheck synccheck; do timeout 600 $S --tool $t python tools/run_once.py "$op" 2>&1 | grep -E "ERROR SUMMARY" | head -1; done
done
timeout 1200 python bench.py --steps 30 --warmup 5 > gpurun_out/r2zq_bench.jsonl 2> gpurun_out/r2zq_bench.err; tail -2 gpurun_out/r2zq_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zq_bench.jsonl").read().strip().splitlines()[-1])
print("headline", round(d["value"],1), d["unit"], round(d["ms_per_step"]*1e3,2), d["step_ms_distribution"], "frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"],2), d["clocks"])
for k,v in (d.get("suite") or {}).items(): print(" ", k, round(v.get("value",0),1), v.get("unit"), round(v.get("ms_per_step",0)*1e3,2), "frac", round(v["roofline"]["frac"],3) if v.get("roofline") else v.get("error"))
for k,v in (d.get("sequences") or {}).items(): print(" ", k, round(v.get("value",0),1), round(v.get("ms_per_step",0),3), "ms", v.get("error"))
P
