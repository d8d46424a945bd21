mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_contract.py -q -p no:cacheprovider -x > gpurun_out/r2zm_tests.log 2>&1; tail -15 gpurun_out/r2zm_tests.log
S=/usr/local/cuda/bin/compute-sanitizer
for t in memcheck synccheck; do timeout 600 $S --tool $t python tools/run_once.py '{"kind":"conv2d","I":[2,64,12,15],"K":[64,64,3,3],"S":1}' tc_tf32 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|cta_pair" | sed 's/.*"cta_pair": \([a-z]*\).*/cta_pair=\1/' | head -3; done
timeout 600 $S --tool memcheck python tools/run_once.py '{"kind":"conv2d","I":[2,32,12,14],"K":[48,32,3,3],"S":1}' tc_tf32 2>&1 | grep -E "ERROR SUMMARY" | head -2
timeout 600 python bench.py --steps 30 --warmup 5 --no-sequences > gpurun_out/r2zm_bench.jsonl 2> gpurun_out/r2zm_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zm_bench.jsonl").read().strip().splitlines()[-1])
print(round(d["value"],1), round(d["ms_per_step"]*1e3,2), d["step_ms_distribution"], d["roofline"]["frac"], d["config"]["kernel_plan"]["cta_pair"], d["e2e"]["value"])
P
tail -3 gpurun_out/r2zm_bench.err
timeout 600 python tools/conv_programs.py > gpurun_out/r2zm_conv_programs.jsonl 2>&1; cat gpurun_out/r2zm_conv_programs.jsonl | cut -c1-400
