mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -p no:cacheprovider -k "flat_from_state or groups_distinct or conv_tc" > gpurun_out/r2zh_flat.log 2>&1; tail -15 gpurun_out/r2zh_flat.log
S=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $S --tool memcheck python -m pytest tests/test_gpu_tc.py -q -p no:cacheprovider -k "flat_from_state and 2-64-12-15" 2>&1 | grep -E "ERROR SUMMARY|passed|failed" | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2zh_bench.jsonl 2> gpurun_out/r2zh_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zh_bench.jsonl").read().strip().splitlines()[-1])
print(round(d["value"],1), round(d["ms_per_step"]*1e3,2), d["config"]["schedule"], d["config"]["kernel_plan"]["cta_pair"], d["rerank"])
P
timeout 900 python bench.py --workload graph_vs_tree --steps 10 --warmup 3 > gpurun_out/r2zh_gvt.jsonl 2> gpurun_out/r2zh_gvt.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zh_gvt.jsonl").read().strip().splitlines()[-1])
print(json.dumps(d)[:3000])
P
