"""Parity of every distinct operator of the configs[4] sequences (ResNet-50 at batch 1, GPT-2 at
batch 1) on the variant `auto` picks, against the CPU oracle's reference_compute — the shapes the
end-to-end benchmark runs (1x1 / strided / stem convs on conv_gemm, 3x3 on conv_tc, the pools,
attention GEMMs, softmax). Tolerances per variant as in test_gpu_tc.py / test_gpu_stream.py."""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
g = pytest.importorskip("paper_2502_11407_b200")
from oracle import oracle as O  # noqa: E402
from paper_2502_11407_b200 import sequences as S  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"tc_tf32": 2e-3, "tc_bf16": 1e-2, "stream": 2e-6, "simt_f32": 2e-6}


def _ops():
    out = []
    for name, seq in (("resnet50", S.resnet50(1)), ("gpt2", S.gpt2(1, layers=1))):
        for key, spec in S.distinct(seq).items():
            if spec.get("N") == 50304:  # LM head: 40 GFLOP, too slow for the CPU oracle
                continue
            out.append(pytest.param(spec, id=f"{name}:{key}"))
    return out


@pytest.mark.parametrize("spec", _ops())
def test_sequence_op_parity(spec):
    op = g.TensorOpSpec.parse_text(json.dumps(spec))
    sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
    k = g.Kernel(op, sched, 0, "auto")
    variant = k.info["variant_name"]
    rng = np.random.default_rng(0)
    bf16 = op.dtype_bytes == 2
    xs = []
    for t in op.tensors[:-1]:
        x = rng.uniform(-1, 1, int(np.prod(t["true_dims"])) * op.batch).astype(np.float32)
        if bf16:
            x = torch.from_numpy(x).bfloat16().float().numpy()
        xs.append(x)
    dt = torch.bfloat16 if bf16 else torch.float32
    dev = [torch.from_numpy(x).to(dt).cuda() for x in xs]
    out = torch.full((int(np.prod(op.tensors[-1]["true_dims"])) * op.batch,), float("nan"), dtype=dt, device="cuda")
    k.execute(dev, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().astype(np.float64)
    ref = O.reference_compute(spec, xs, threads=8)
    assert not np.isnan(got).any()
    if spec["kind"] == "softmax":
        assert (np.abs(got - ref) / ref).max() <= 2e-6
    else:
        err = np.abs(got - ref).max() / max(1e-30, np.abs(ref).max())
        assert err <= TOL[variant], (variant, k.info["plan"].get("family"), err)
