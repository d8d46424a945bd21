mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_generic.py tests/test_gpu_stream.py -m gpu -q -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1
tail -40 gpurun_out/r2b_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --suite gemm_fp32,gemm --no-cpu-baseline > gpurun_out/r2b_bench.jsonl 2> gpurun_out/r2b_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2b_bench.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"]); print(json.dumps(d["suite"], indent=1))
P
