mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_contract.py -q -p no:cacheprovider -x -k "conv" > gpurun_out/r2zr_tests.log 2>&1; tail -2 gpurun_out/r2zr_tests.log
for i in 1 2 3; do timeout 600 python bench.py --steps 40 --warmup 5 --no-sequences --suite "" --no-cpu-baseline > gpurun_out/r2zr_bench$i.jsonl 2> gpurun_out/r2zr_bench.err
python - <<P
import json
d=json.loads(open("gpurun_out/r2zr_bench$i.jsonl").read().strip().splitlines()[-1])
print(round(d["value"],1), round(d["ms_per_step"]*1e3,2), d["step_ms_distribution"], d["roofline"]["frac"])
P
done
