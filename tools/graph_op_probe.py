"""Developer probe: one op launched eagerly vs replayed from a CUDA graph (L2 flushed)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_11407_b200 as g
doc = json.loads(sys.argv[1])
op = g.TensorOpSpec.parse_text(json.dumps(doc))
k = g.Kernel(op, g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1)), 0, "auto")
dt = torch.bfloat16 if op.dtype_bytes == 2 else torch.float32
xs = [torch.rand(int(np.prod(t["true_dims"])) * op.batch, device="cuda").to(dt) for t in op.tensors[:-1]]
out = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])) * op.batch, device="cuda", dtype=dt)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3): k.execute(xs, out, st)
torch.cuda.synchronize()
ref = out.clone()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=st):
    k.execute(xs, out, torch.cuda.current_stream())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn, n=21):
    ts = []
    for _ in range(n):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st); fn(); e.record(st)
        e.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return sorted(ts)[n // 2]
eager = timeit(lambda: k.execute(xs, out, st))
out.zero_(); torch.cuda.synchronize()
replay = timeit(lambda: graph.replay())
torch.cuda.synchronize()
print(json.dumps({"op": doc, "eager_us": eager, "graph_us": replay, "same": bool(torch.equal(out, ref))}))
