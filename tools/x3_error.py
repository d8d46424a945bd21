"""Developer tool (GPU box): 3xTF32 accuracy, max |error| / max |C| and normwise against the fp64 oracle."""
import json, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2502_11407_b200 as g
from oracle import oracle as O
for doc in ({"kind":"gemm","M":1024,"K":1024,"N":1024}, {"kind":"gemm","M":256,"K":4096,"N":192}):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    s = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
    k = g.Kernel(op, s, 0, "tc_3xtf32")
    rng = np.random.default_rng(0)
    xs = [rng.uniform(-1, 1, int(np.prod(t["true_dims"]))).astype(np.float32) for t in op.tensors[:-1]]
    ref = O.reference_compute(doc, xs, threads=16)
    out = torch.empty(ref.size, device="cuda")
    k.execute([torch.from_numpy(x).cuda() for x in xs], out); torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    print(doc, "max|d|/max|ref|", np.abs(got - ref).max() / np.abs(ref).max(), "normwise", np.linalg.norm(got - ref) / np.linalg.norm(ref))
