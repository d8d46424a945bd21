"""Developer tool: per-distinct-op device time of a sequence (resnet50 / gpt2) on cuda:0."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_11407_b200 as g  # noqa: E402
from paper_2502_11407_b200 import sequences as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
seq = S.sharded(name, 1)
counts = {}
for _, sp in seq:
    k = json.dumps(sp, sort_keys=True)
    counts[k] = counts.get(k, 0) + 1
hw = g.HardwareSpec.b200(0)
rows = []
for key, n in counts.items():
    spec = json.loads(key)
    op = g.TensorOpSpec.parse_text(key)
    sched = g.optimize(op, hw, g.EngineConfig(mode="b200", top_k=1))
    k = g.Kernel(op, sched, 0, "auto")
    dt = torch.bfloat16 if op.dtype_bytes == 2 else torch.float32
    xs = [torch.rand(int(np.prod(t["true_dims"])) * op.batch, device="cuda").to(dt) for t in op.tensors[:-1]]
    out = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])) * op.batch, device="cuda", dtype=dt)
    for _ in range(3):
        k.execute(xs, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        k.execute(xs, out)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    us = statistics.median(ts)
    rows.append((n * us, n, us, op.flops / (us * 1e-6) / 1e12, k.info["variant_name"], k.info["plan"].get("family"),
                 k.info["plan"].get("BN"), spec))
rows.sort(key=lambda r: -r[0])
tot = sum(r[0] for r in rows)
for r in rows:
    print(f"{r[0]:9.1f}us {100*r[0]/tot:5.1f}% x{r[1]:2d} {r[2]:8.1f}us {r[3]:7.1f}TF {r[4]} {r[5]} BN={r[6]} {json.dumps(r[7])}")
print("total", tot, "us")
