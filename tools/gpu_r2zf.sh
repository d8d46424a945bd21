mkdir -p gpurun_out
echo skip tests
timeout 600 python bench.py --steps 20 --warmup 5 --suite gemm,bgemm --no-cpu-baseline > gpurun_out/r2zf_bench.jsonl 2> gpurun_out/r2zf_bench.err; tail -2 gpurun_out/r2zf_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zf_bench.jsonl").read().strip().splitlines()[-1])
for k,v in (d.get("suite") or {}).items(): print(k, round(v.get("value",0),1), round(v.get("ms_per_step",0)*1e3,2), v.get("error"))
for k,v in (d.get("sequences") or {}).items(): print(k, round(v.get("value",0),1), round(v.get("ms_per_step",0),3), v.get("error"))
P
touch paper_2502_11407_b200/csrc/kernels/exec.cu; make -s -j8 -C paper_2502_11407_b200/csrc DEV=1 > /dev/null 2>&1
GENSOR_GEMM_PAIR=0 timeout 600 python bench.py --steps 20 --warmup 5 --suite gemm,bgemm --no-cpu-baseline > gpurun_out/r2zf_bench0.jsonl 2> gpurun_out/r2zf_bench0.err; tail -2 gpurun_out/r2zf_bench0.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2zf_bench0.jsonl").read().strip().splitlines()[-1])
print("-- no pair")
for k,v in (d.get("suite") or {}).items(): print(k, round(v.get("value",0),1), round(v.get("ms_per_step",0)*1e3,2), v.get("error"))
for k,v in (d.get("sequences") or {}).items(): print(k, round(v.get("value",0),1), round(v.get("ms_per_step",0),3), v.get("error"))
P
