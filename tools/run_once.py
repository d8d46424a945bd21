"""Developer tool: one execute of an op (for compute-sanitizer / cuda-gdb on the GPU box).
  python tools/run_once.py '<op json>' [variant]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_11407_b200 as g  # noqa: E402

doc = json.loads(sys.argv[1])
variant = sys.argv[2] if len(sys.argv) > 2 else "auto"
op = g.TensorOpSpec.parse_text(json.dumps(doc))
sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
k = g.Kernel(op, sched, 0, variant)
print(json.dumps(k.info["plan"]))
dt = torch.bfloat16 if op.dtype_bytes == 2 else torch.float32
xs = [torch.rand(int(np.prod(t["true_dims"])) * op.batch, device="cuda").to(dt) for t in op.tensors[:-1]]
out = torch.empty(int(np.prod(op.tensors[-1]["true_dims"])) * op.batch, device="cuda", dtype=dt)
k.execute(xs, out)
torch.cuda.synchronize()
print("ok", float(out.float().abs().sum()))
