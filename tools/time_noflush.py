"""Developer experiment: does the L2-flush kernel between steps cost the next launch (smem
carveout reconfiguration)? Times an op back-to-back vs after a flush, and after a flush issued
by a kernel that already prefers the max shared-memory carveout."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_11407_b200 as g
doc = json.loads(sys.argv[1]); variant = sys.argv[2] if len(sys.argv) > 2 else "auto"
op = g.TensorOpSpec.parse_text(json.dumps(doc))
sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
k = g.Kernel(op, sched, 0, variant)
dt = torch.bfloat16 if op.dtype_bytes == 2 else torch.float32
xs = [torch.rand(int(np.prod(t["true_dims"])) * op.batch, device="cuda").to(dt) for t in op.tensors[:-1]]
out = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])) * op.batch, device="cuda", dtype=dt)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(pre, n=20):
    ts = []
    for _ in range(n):
        pre()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); k.execute(xs, out); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return round(statistics.median(ts), 2)
for _ in range(3): k.execute(xs, out)
torch.cuda.synchronize()
res = {"back_to_back": run(lambda: None), "after_flush": run(lambda: flush.zero_()),
       "after_same_kernel": run(lambda: k.execute(xs, out))}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
ev[0].record()
for i in range(20):
    k.execute(xs, out); ev[i + 1].record()
ev[-1].synchronize()
res["stream_of_20_per_launch"] = round(ev[0].elapsed_time(ev[-1]) * 1e3 / 20, 2)
print(json.dumps({"op": doc, "variant": k.info["variant_name"], "us": res}))
