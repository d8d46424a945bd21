"""Developer tool: per-launch device times of one op's kernel (CUDA events around each internal
launch), no correctness checks — for A/B experiments on the GPU box.
  python tools/time_op.py '{"kind":"conv2d","I":[16,64,58,58],"K":[64,64,3,3],"S":1}' [variant] [iters]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_11407_b200 as g  # noqa: E402

doc = json.loads(sys.argv[1])
variant = sys.argv[2] if len(sys.argv) > 2 else "auto"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
op = g.TensorOpSpec.parse_text(json.dumps(doc))
sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
k = g.Kernel(op, sched, 0, variant)
dt = torch.bfloat16 if op.dtype_bytes == 2 else torch.float32
xs = [torch.rand(int(np.prod(t["true_dims"])) * op.batch, device="cuda").to(dt) for t in op.tensors[:-1]]
out = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])) * op.batch, device="cuda", dtype=dt)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
k.set_timing(True)
for _ in range(3):
    k.execute(xs, out)
torch.cuda.synchronize()
acc = {}
for _ in range(iters):
    flush.zero_()
    torch.cuda._sleep(80_000)
    k.execute(xs, out)
    for name, ms in k.timings():
        acc.setdefault(name, []).append(ms * 1e3)
res = {n: round(statistics.median(v), 2) for n, v in acc.items()}
print(json.dumps({"op": doc, "variant": k.info["variant_name"], "us": res, "plan": k.info["plan"],
                  "tflops": op.flops / (sum(res.values()) * 1e-6) / 1e12}))
