"""Developer probe: execute_host timing (pipelined chunks vs one shot) for one op."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2502_11407_b200 as g
doc = json.loads(sys.argv[1])
op = g.TensorOpSpec.parse_text(json.dumps(doc))
sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
k = g.Kernel(op, sched, 0, "auto")
hs = [torch.rand(int(np.prod(t["true_dims"])) * op.batch).pin_memory() for t in op.tensors[:-1]]
ho = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])) * op.batch).pin_memory()
k.execute_host(hs, ho)
print(json.dumps(k.info.get("host_pipe")))
ts = []
for _ in range(10):
    t0 = time.perf_counter(); k.execute_host(hs, ho); ts.append(time.perf_counter() - t0)
print("execute_host median ms", sorted(ts)[5] * 1e3)
