"""gensor_execute_host on large ops: the chunked copy/compute pipeline (exec.cu HostPipe) must
return exactly what one device execute of the whole op returns (the chunks split only spatial
axes, so every output keeps its accumulation order), and stay within the variant's tolerance of
the oracle on a sampled subset."""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
g = pytest.importorskip("paper_2502_11407_b200")

pytestmark = pytest.mark.gpu

OPS = [
    {"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1},
    {"kind": "conv2d", "I": [24, 128, 30, 30], "K": [128, 128, 3, 3], "S": 1},
    {"kind": "gemm", "M": 3000, "K": 512, "N": 1024},
    {"kind": "gemm", "M": 512, "K": 64, "N": 512, "dtype_bytes": 2, "batch": 40},
    {"kind": "gemv", "M": 20000, "N": 1024},
    {"kind": "softmax", "M": 5000, "N": 1000},
    {"kind": "avgpool2d", "I": [15, 64, 80, 80], "F": 3, "S": 1},
    {"kind": "dwconv2d", "I": [17, 64, 100, 100], "K": [64, 1, 3, 3], "S": 2},
    {"kind": "conv2d", "I": [20, 3, 115, 115], "K": [64, 3, 7, 7], "S": 2},      # space-to-depth stem
]


CASES = [(d, "auto") for d in OPS] + [
    # the state-driven SIMT family: sub-kernels lowered from the clamped state
    ({"kind": "gemv", "M": 8192, "N": 1024}, "simt_f32"),
    ({"kind": "gemm", "M": 4096, "K": 512, "N": 512}, "simt_f32"),
]


@pytest.mark.parametrize("doc,variant", CASES, ids=lambda x: x if isinstance(x, str) else x["kind"] + str(x.get("I", x.get("M"))))
def test_execute_host_matches_device(doc, variant):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
    k = g.Kernel(op, sched, 0, variant)
    bf16 = op.dtype_bytes == 2
    dt = torch.bfloat16 if bf16 else torch.float32
    gen = torch.Generator().manual_seed(0)
    hs = [(torch.rand(int(np.prod(t["true_dims"])) * op.batch, generator=gen) * 2 - 1).to(dt).pin_memory()
          for t in op.tensors[:-1]]
    nout = int(np.prod(op.tensors[-1]["true_dims"])) * op.batch
    dev_out = torch.full((nout,), float("nan"), dtype=dt, device="cuda")
    k.execute([h.cuda() for h in hs], dev_out)
    torch.cuda.synchronize()
    host_out = torch.full((nout,), float("nan"), dtype=dt).pin_memory()
    k.execute_host(hs, host_out)
    total = sum(h.numel() * h.element_size() for h in hs) + host_out.numel() * host_out.element_size()
    if total >= 18 << 20:  # >= 2 chunks of ~9 MB: the chunked pipeline ran
        assert k.info.get("host_pipe"), k.info
    assert not torch.isnan(host_out.float()).any()
    assert torch.equal(host_out, dev_out.cpu()), (doc, (host_out.float() - dev_out.cpu().float()).abs().max())
