# checkpoint: full GPU suite, smoke, default bench (as the driver runs it), reference arm, ncu launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2y_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2y_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; tail -2 gpurun_out/r2y_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2y_bench.jsonl 2> gpurun_out/r2y_bench.err; tail -2 gpurun_out/r2y_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2y_ref.jsonl 2> gpurun_out/r2y_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2y_launches.csv python bench.py --steps 2 --warmup 1 --suite "" --no-cpu-baseline --no-sequences > gpurun_out/r2y_ncu_bench.log 2>&1
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2y_bench.jsonl").read().strip().splitlines()[-1])
print("headline", round(d["value"],1), d["unit"], round(d["ms_per_step"]*1e3,2), "us frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"],2), "launches", d["gpu_launches"])
for k,v in (d.get("suite") or {}).items(): print(" ", k, round(v.get("value",0),1), v.get("unit"), round(v.get("ms_per_step",0)*1e3,2), "frac", round(v["roofline"]["frac"],3) if v.get("roofline") else v.get("error"))
for k,v in (d.get("sequences") or {}).items(): print(" ", k, round(v.get("value",0),1), round(v.get("ms_per_step",0),3), "ms", v.get("error"))
r=json.loads(open("gpurun_out/r2y_ref.jsonl").read().strip().splitlines()[-1]); print("ref", r.get("value"), r.get("unit"), r.get("cpu_baseline",{}).get("cores"))
P
