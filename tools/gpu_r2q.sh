mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2q_pytest_gpu.log 2>&1; tail -5 gpurun_out/r2q_pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/r2q_bench.jsonl 2> gpurun_out/r2q_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2q_bench.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["achieved"], d["e2e"]["value"], d.get("launch_breakdown_ms"), d["config"]["kernel_plan"].get("mma_issue"))
P
