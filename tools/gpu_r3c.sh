mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_contract.py tests/test_gpu_sequences.py -q -p no:cacheprovider -x > gpurun_out/r3c_tests.log 2>&1; tail -3 gpurun_out/r3c_tests.log
S=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $S --tool memcheck python tools/run_once.py '{"kind":"conv2d","I":[3,64,20,30],"K":[64,64,3,3],"S":1}' tc_tf32 2>&1 | grep -E "ERROR SUMMARY|cta_pair" | sed 's/.*"cta_pair": \([a-z]*\).*/cta_pair=\1/' | head -3
timeout 600 $S --tool synccheck python tools/run_once.py '{"kind":"conv2d","I":[3,64,20,30],"K":[64,64,3,3],"S":1}' tc_tf32 2>&1 | grep -E "ERROR SUMMARY" | head -3
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 --no-sequences --suite "" --no-cpu-baseline > gpurun_out/r3c_bench$i.jsonl 2> gpurun_out/r3c_bench.err
python - <<P
import json
d=json.loads(open("gpurun_out/r3c_bench$i.jsonl").read().strip().splitlines()[-1])
print(round(d["value"],1), round(d["ms_per_step"]*1e3,2), d["step_ms_distribution"], d["roofline"]["frac"], d["config"]["kernel_plan"]["cta_pair"])
P
done
