mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2zi_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2zi_pytest_gpu.log
timeout 900 python bench.py --workload resnet50 --steps 10 --warmup 3 > gpurun_out/r2zi_resnet.jsonl 2> gpurun_out/r2zi_resnet.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zi_resnet.jsonl").read().strip().splitlines()[-1])
print(round(d["value"],1), round(d["ms_per_step"],3))
P
