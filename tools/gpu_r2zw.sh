mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2zw_pytest_gpu.log 2>&1; tail -2 gpurun_out/r2zw_pytest_gpu.log
S=/usr/local/cuda/bin/compute-sanitizer
for t in memcheck racecheck synccheck; do timeout 600 $S --tool $t python tools/run_once.py '{"kind":"conv2d","I":[3,32,19,19],"K":[96,32,3,3],"S":2}' tc_tf32 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY" | head -1; done
for i in 1 2; do timeout 900 python bench.py --workload resnet50 --steps 10 --warmup 3 > gpurun_out/r2zw_resnet$i.jsonl 2> gpurun_out/r2zw_resnet.err
python - <<P
import json
d=json.loads(open("gpurun_out/r2zw_resnet$i.jsonl").read().strip().splitlines()[-1])
print("resnet50", round(d["value"],1), round(d["ms_per_step"],3))
P
done
