"""Developer probe: a sequence step launched eagerly vs replayed from a CUDA graph."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_11407_b200 as g
from paper_2502_11407_b200 import sequences as S
name = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
seq = S.sharded(name, 1)
hw = g.HardwareSpec.b200(0)
kern, bufs = {}, {}
for key, sp in S.distinct(seq).items():
    op = g.TensorOpSpec.parse_text(json.dumps(sp))
    k = g.Kernel(op, g.optimize(op, hw, g.EngineConfig(mode="b200", top_k=1)), 0, "auto")
    dt = torch.bfloat16 if op.dtype_bytes == 2 else torch.float32
    xs = [torch.rand(int(np.prod(t["true_dims"])) * op.batch, device="cuda").to(dt) for t in op.tensors[:-1]]
    out = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])) * op.batch, device="cuda", dtype=dt)
    kern[key], bufs[key] = k, (xs, out)
keys = [json.dumps(sp, sort_keys=True) for _, sp in seq]
def step(st):
    for key in keys:
        kern[key].execute(bufs[key][0], bufs[key][1], st)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3): step(st)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=st):
    step(torch.cuda.current_stream())
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn, n=5):
    ts = []
    for _ in range(n):
        with torch.cuda.stream(st):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st); fn(); e.record(st)
        e.synchronize(); ts.append(s.elapsed_time(e))
    return sorted(ts)[n // 2]
eager = timeit(lambda: step(st))
replay = timeit(lambda: graph.replay())
print(json.dumps({"seq": name, "ops": len(keys), "eager_ms": eager, "graph_ms": replay}))
