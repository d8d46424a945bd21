mkdir -p gpurun_out
for i in 1; do timeout 300 python bench.py --steps 30 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/r2r_bench$i.jsonl 2> gpurun_out/r2r_bench.err; done
touch paper_2502_11407_b200/csrc/kernels/exec.cu; make -s -j8 -C paper_2502_11407_b200/csrc DEV=1 > /dev/null 2>&1
GENSOR_CONV_FLAT=0 timeout 300 python bench.py --steps 30 --warmup 5 --suite "" --no-cpu-baseline > gpurun_out/r2r_bench_ns.jsonl 2>> gpurun_out/r2r_bench.err
python - <<'P'
import json
for f in ["r2r_bench1","r2r_bench2","r2r_bench_ns"]:
    d=json.loads(open(f"gpurun_out/{f}.jsonl").read().strip().splitlines()[-1])
    print(f, round(d["value"],1), round(d["ms_per_step"]*1e3,2), round(d["roofline"]["frac"],3), d["e2e"]["value"], d.get("launch_breakdown_ms"), d["config"]["kernel_plan"]["family"])
P
