mkdir -p gpurun_out
timeout 1200 python bench.py --workload graph_vs_tree --steps 10 --warmup 3 > gpurun_out/r2t_gvt.jsonl 2> gpurun_out/r2t_gvt.err
tail -2 gpurun_out/r2t_gvt.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2t_gvt.jsonl").read().strip().splitlines()[-1])
print("geo", d["value"], d.get("reranked_geomean"))
for k,v in d["per_op"].items(): print(k, "graph %.4f rr %.4f tree %.4f"%(v["graph"]["ms"],v["graph_reranked"]["ms"],v["tree"]["ms"]), v.get("topk_distinct_plans"), [round(x,4) for x in v.get("topk_rerank_ms",[])])
P
