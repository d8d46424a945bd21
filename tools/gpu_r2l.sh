# conv_flat first light: parity, contract, headline bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider -k "conv_tc or baseline" > gpurun_out/r2l_tc.log 2>&1
tail -15 gpurun_out/r2l_tc.log
timeout 300 python -m pytest tests/test_gpu_contract.py -q -x -p no:cacheprovider > gpurun_out/r2l_contract.log 2>&1
tail -5 gpurun_out/r2l_contract.log
timeout 300 python bench.py --steps 20 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/r2l_bench.jsonl 2> gpurun_out/r2l_bench.err
tail -3 gpurun_out/r2l_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2l_bench.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"], d["config"]["kernel_plan"], d["e2e"]["value"], d.get("launch_breakdown_ms"))
P
