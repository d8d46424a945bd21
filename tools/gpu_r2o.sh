mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_contract.py -q -x -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; tail -3 gpurun_out/r2o_tests.log
timeout 300 python bench.py --steps 30 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/r2o_bench.jsonl 2> gpurun_out/r2o_bench.err
tail -3 gpurun_out/r2o_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2o_bench.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["achieved"], d["e2e"]["value"], d.get("launch_breakdown_ms"), d["config"]["kernel_plan"].get("mma_issue"))
P
