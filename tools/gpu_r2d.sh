mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_generic.py tests/test_gpu_contract.py -m gpu -q -p no:cacheprovider > gpurun_out/r2d_pytest.log 2>&1
tail -15 gpurun_out/r2d_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --suite gemm_fp32,gemm,bgemm --no-cpu-baseline > gpurun_out/r2d_bench.jsonl 2> gpurun_out/r2d_bench.err
tail -3 gpurun_out/r2d_bench.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2d_bench.jsonl").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d.get("rerank")); print(json.dumps(d["suite"], indent=1))
P
timeout 900 python bench.py --workload graph_vs_tree --steps 10 --warmup 3 > gpurun_out/r2d_gvt.jsonl 2> gpurun_out/r2d_gvt.err
tail -3 gpurun_out/r2d_gvt.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/r2d_gvt.jsonl").read().strip().splitlines()[-1])
print("geo", d["value"], d["reranked_geomean"])
for k,v in d["per_op"].items(): print(k, "graph %.4f rr %.4f tree %.4f"%(v["graph"]["ms"],v["graph_reranked"]["ms"],v["tree"]["ms"]), v["topk_distinct_plans"], [round(x,4) for x in v["topk_rerank_ms"]])
P
