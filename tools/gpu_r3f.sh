# round-2 checkpoint: full GPU suite, smoke, default bench (as the driver runs it), reference arm,
# graph vs tree, conv programs, ncu launch list, per-launch DRAM traffic, --set full of conv_flat
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r3f_pytest_gpu.log 2>&1; tail -3 gpurun_out/r3f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3f_smoke.log 2>&1; tail -2 gpurun_out/r3f_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 30 --warmup 5 > gpurun_out/r3f_bench.jsonl 2> gpurun_out/r3f_bench.err; tail -2 gpurun_out/r3f_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r3f_ref.jsonl 2> gpurun_out/r3f_ref.err
timeout 900 python bench.py --workload graph_vs_tree --steps 20 --warmup 5 > gpurun_out/r3f_gvt.jsonl 2> gpurun_out/r3f_gvt.err
timeout 600 python tools/conv_programs.py > gpurun_out/r3f_conv_programs.jsonl 2> gpurun_out/r3f_conv_programs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r3f_launches.csv python bench.py --steps 2 --warmup 1 --suite "" --no-cpu-baseline --no-sequences > gpurun_out/r3f_ncu_bench.log 2>&1
C='{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}'
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_conv_flat_pair" -s 2 -c 1 -o gpurun_out/r3f_conv_flat_pair -f python tools/time_op.py "$C" tc_tf32 3 > gpurun_out/r3f_ncu_full.log 2>&1
tail -2 gpurun_out/r3f_ncu_full.log
bash tools/gpu_traffic.sh > gpurun_out/r3f_traffic.log 2>&1; tail -3 gpurun_out/r3f_traffic.log
python - <<'P'
import json
d=json.loads(open("gpurun_out/r3f_bench.jsonl").read().strip().splitlines()[-1])
print("headline", round(d["value"],1), d["unit"], round(d["ms_per_step"]*1e3,2), "us frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"],2), "launches", d["gpu_launches"], d["clocks"])
for k,v in (d.get("suite") or {}).items(): print(" ", k, round(v.get("value",0),1), v.get("unit"), round(v.get("ms_per_step",0)*1e3,2), "frac", round(v["roofline"]["frac"],3) if v.get("roofline") else v.get("error"))
for k,v in (d.get("sequences") or {}).items(): print(" ", k, round(v.get("value",0),1), round(v.get("ms_per_step",0),3), "ms", v.get("error"))
r=json.loads(open("gpurun_out/r3f_ref.jsonl").read().strip().splitlines()[-1]); print("ref", r.get("value"), r.get("unit"), r.get("cpu_baseline",{}).get("cores"))
g=json.loads(open("gpurun_out/r3f_gvt.jsonl").read().strip().splitlines()[-1]); print("gvt", g["value"], g.get("reranked_geomean"))
for k,v in g["per_op"].items(): print(" ", k, round(v["graph"]["ms"]*1e3,2), round(v["tree"]["ms"]*1e3,2), "est", round(v["graph"]["est_ms"]*1e3,2))
P
cat gpurun_out/r3f_conv_programs.jsonl | cut -c1-300
bash tools/gpu_san.sh > gpurun_out/r3f_sanitizer.log 2>&1; grep -c "0 errors\|0 hazards" gpurun_out/r3f_sanitizer.log; grep -B1 -E "ERROR SUMMARY: [1-9]|hazards displayed \([1-9]" gpurun_out/r3f_sanitizer.log | head
