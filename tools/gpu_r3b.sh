mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3b_pytest_gpu.log 2>&1; tail -2 gpurun_out/r3b_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3b_smoke.log 2>&1; tail -1 gpurun_out/r3b_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 30 --warmup 5 > gpurun_out/r3b_bench.jsonl 2> gpurun_out/r3b_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r3b_bench.jsonl").read().strip().splitlines()[-1])
print("headline", round(d["value"],1), round(d["ms_per_step"]*1e3,2), d["step_ms_distribution"], "frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"],2), d["e2e"]["pipeline"], d["clocks"])
print({k: round(v["value"],1) for k,v in d["suite"].items()}, {k: round(v["ms_per_step"],3) for k,v in d["sequences"].items()})
P
