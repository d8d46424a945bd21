"""How the L2 flush method shapes a step: after a WRITE flush (256 MiB zero_, the bench's method)
the L2 is full of dirty lines, so every line a step allocates first evicts one (an extra HBM
write); after a READ flush the L2 holds clean lines. Times a 13.8 MB copy (the NHWC pre-pass's
traffic) and the headline conv under both."""
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_11407_b200 as g  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
x = torch.rand(16 * 64 * 58 * 58, device="cuda")
y = torch.empty_like(x)
doc = {"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1}
op = g.TensorOpSpec.parse_text(json.dumps(doc))
k = g.Kernel(op, g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1)), 0, "auto")
w = torch.rand(64 * 64 * 9, device="cuda")
o = torch.empty(16 * 64 * 56 * 56, device="cuda")


def timed(fn, mode, n=30):
    ts = []
    for _ in range(n):
        if mode == "write":
            flush.zero_()
        elif mode == "read":
            flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


for mode in ("write", "read", "none"):
    print(mode, "copy 13.8 MB: %.2f us" % timed(lambda: y.copy_(x), mode),
          " conv: %.2f us" % timed(lambda: k.execute([x, w], o), mode), flush=True)
