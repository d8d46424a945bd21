bash tools/gpu_r2n.sh
touch paper_2502_11407_b200/csrc/kernels/exec.cu paper_2502_11407_b200/csrc/kernels/conv_flat.cu; make -s -j8 -C paper_2502_11407_b200/csrc > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_contract.py -q -x -p no:cacheprovider -k "conv or baseline or contract or workspace or stream or fresh" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 40 --warmup 5 --suite "" --no-cpu-baseline --no-sequences > gpurun_out/r2ze_bench$i.jsonl 2> gpurun_out/r2ze_bench.err; done
python - <<'P'
import json
for i in (1,2):
    d=json.loads(open(f"gpurun_out/r2ze_bench{i}.jsonl").read().strip().splitlines()[-1])
    print("bench", round(d["value"],1), round(d["ms_per_step"]*1e3,2), round(d["roofline"]["frac"],3), d.get("launch_breakdown_ms"))
P
