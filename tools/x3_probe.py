"""Developer probe: the 3xTF32 GEMM on a few shapes, error vs the oracle (run under
compute-sanitizer when debugging)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2502_11407_b200 as g  # noqa: E402
from oracle import oracle as O  # noqa: E402

shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or [(128, 64, 64), (1024, 1024, 1024)]
hw = g.HardwareSpec.b200(0)
for M, K, N in shapes:
    doc = {"kind": "gemm", "M": M, "K": K, "N": N}
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    s = g.optimize(op, hw, g.EngineConfig(mode="b200", top_k=1))
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, M * K).astype(np.float32)
    b = rng.uniform(-1, 1, K * N).astype(np.float32)
    ref = O.reference_compute(doc, [a, b], threads=8)
    for v in ("tc_tf32", "tc_3xtf32"):
        k = g.Kernel(op, s, 0, v)
        out = torch.full((M * N,), float("nan"), device="cuda")
        k.execute([torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()], out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().astype(np.float64)
        bad = np.isnan(got).reshape(M, N)
        rows = np.where(bad.any(1))[0]
        cols = np.where(bad.any(0))[0]
        print(M, K, N, v, "err", np.nanmax(np.abs(got - ref)) / np.abs(ref).max(), "nan", int(bad.sum()),
              "rows", rows[:3], rows[-3:] if len(rows) else "", "cols", cols[:3], cols[-3:] if len(cols) else "", flush=True)
