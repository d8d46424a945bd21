mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_cli.py -q -x -p no:cacheprovider > gpurun_out/r2u_tests.log 2>&1; tail -5 gpurun_out/r2u_tests.log
timeout 900 python bench.py --workload graph_vs_tree --variant simt_f32 --steps 5 --warmup 2 > gpurun_out/r2u_gvt_simt.jsonl 2> gpurun_out/r2u_gvt.err
tail -2 gpurun_out/r2u_gvt.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2u_gvt_simt.jsonl").read().strip().splitlines()[-1])
print("geo", d["value"], d.get("reranked_geomean"))
for k,v in d["per_op"].items(): print(k, "graph %.4f rr %.4f tree %.4f"%(v["graph"]["ms"],v["graph_reranked"]["ms"],v["tree"]["ms"]), v.get("topk_distinct_plans"), [round(x,4) for x in v.get("topk_rerank_ms",[])], v["graph"].get("plan",{}).get("fast") if isinstance(v["graph"].get("plan"),dict) else "")
P
