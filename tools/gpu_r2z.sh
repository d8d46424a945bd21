mkdir -p gpurun_out
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
timeout 120 python tools/run_once.py "$C" tc_tf32 > gpurun_out/r2z_once.log 2>&1; echo "once rc=$?"; tail -3 gpurun_out/r2z_once.log
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_contract.py -q -x -p no:cacheprovider -k "conv or baseline or contract or workspace or stream or fresh" > gpurun_out/r2z_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2z_tests.log
timeout 300 python bench.py --steps 30 --warmup 5 --suite "" --no-cpu-baseline --no-sequences > gpurun_out/r2z_bench.jsonl 2> gpurun_out/r2z_bench.err; tail -2 gpurun_out/r2z_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2z_bench.jsonl").read().strip().splitlines()[-1])
print(round(d["value"],1), round(d["ms_per_step"]*1e3,2), round(d["roofline"]["frac"],3), d.get("launch_breakdown_ms"), d["config"]["kernel_plan"].get("cta_pair"), d["config"]["kernel_plan"].get("stages"))
P
