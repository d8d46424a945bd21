mkdir -p gpurun_out
start=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s_bench.jsonl 2> gpurun_out/r2s_bench.err
echo "wall $(( $(date +%s) - start )) s"; tail -3 gpurun_out/r2s_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2s_bench.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"])
print(json.dumps(d["sequences"], indent=1))
for k,v in d["suite"].items(): print(k, v.get("value"), v.get("roofline",{}).get("frac"), v.get("error"))
P
