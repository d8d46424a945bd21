"""The execute contract of include/gensor_b200.h on the GPU:
  * one kernel handle may be executed on several streams at once (per-stream workspaces, no
    shared mutable device state): concurrent executes give bit-identical results to serial ones;
  * gensor_execute_ws runs on a caller-owned workspace;
  * a fresh workspace's first execute and a changed filter bank on the same handle are correct
    (the conv families' filter pre-pass is ordered before the conv grid reads it — programmatic
    dependent launch);
Integer-valued inputs U{-2..2} make every family bit-exact against the oracle."""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
g = pytest.importorskip("paper_2502_11407_b200")
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

OPS = {
    "conv_flat": {"kind": "conv2d", "I": [4, 64, 30, 30], "K": [64, 64, 3, 3], "S": 1},
    "conv_ns": {"kind": "conv2d", "I": [4, 48, 30, 30], "K": [64, 48, 3, 3], "S": 1},
    "conv_gemm": {"kind": "conv2d", "I": [3, 32, 19, 19], "K": [96, 32, 3, 3], "S": 2},
    "conv_tc": {"kind": "conv2d", "I": [2, 128, 14, 14], "K": [128, 128, 3, 3], "S": 1},
    "gemm_tc": {"kind": "gemm", "M": 384, "K": 256, "N": 320},
}


def _setup(doc, seed=0):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(seed=0, mode="b200", top_k=1))
    k = g.Kernel(op, sched, 0, "tc_tf32")
    rng = np.random.default_rng(seed)
    xs = [rng.integers(-2, 3, size=int(np.prod(t["true_dims"]))).astype(np.float32) for t in op.tensors[:-1]]
    nout = int(np.prod(op.tensors[-1]["true_dims"]))
    return op, k, xs, nout


@pytest.mark.parametrize("family", list(OPS))
def test_one_handle_two_streams_concurrently(family):
    doc = OPS[family]
    op, k, _, nout = _setup(doc)
    assert k.info["plan"]["family"] == family
    rng = np.random.default_rng(1)
    sets = [[rng.integers(-2, 3, size=int(np.prod(t["true_dims"]))).astype(np.float32) for t in op.tensors[:-1]]
            for _ in range(2)]
    refs = [O.reference_compute(doc, xs, threads=8).astype(np.float32) for xs in sets]
    dev = [[torch.from_numpy(x).cuda() for x in xs] for xs in sets]
    outs = [torch.full((nout,), float("nan"), device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for _ in range(20):  # interleaved launches: both streams' pre-passes and convs overlap
        for i in range(2):
            k.execute(dev[i], outs[i], streams[i])
    torch.cuda.synchronize()
    for i in range(2):
        assert np.array_equal(outs[i].cpu().numpy(), refs[i]), (family, i)
    if k.workspace_bytes:  # each stream got its own workspace slot
        assert family != "gemm_tc"


@pytest.mark.parametrize("family", ["conv_flat", "conv_ns", "conv_gemm", "conv_tc"])
def test_caller_workspace_and_filter_change(family):
    doc = OPS[family]
    op, k, xs, nout = _setup(doc, seed=2)
    nbytes = k.workspace_bytes
    assert nbytes > 0
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ws.fill_(0xFF)  # a fresh, garbage-filled workspace: W' and X must be written before they are read
    dev = [torch.from_numpy(x).cuda() for x in xs]
    out = torch.full((nout,), float("nan"), device="cuda")
    k.execute(dev, out, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), O.reference_compute(doc, xs, threads=8).astype(np.float32))
    # same handle, same workspace, a different filter bank: no stale W'
    rng = np.random.default_rng(3)
    xs2 = [xs[0], rng.integers(-2, 3, size=xs[1].size).astype(np.float32)]
    dev[1].copy_(torch.from_numpy(xs2[1]))
    k.execute(dev, out, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), O.reference_compute(doc, xs2, threads=8).astype(np.float32))
    # a too-small caller workspace is refused
    with pytest.raises(g.GensorError):
        k.execute(dev, out, workspace=ws[: nbytes // 2])


def test_fresh_handle_first_execute_each_family():
    # the first execute of a new handle on a new stream (fresh per-stream workspace)
    for family, doc in OPS.items():
        op, k, xs, nout = _setup(doc, seed=4)
        s = torch.cuda.Stream()
        dev = [torch.from_numpy(x).cuda() for x in xs]
        out = torch.full((nout,), float("nan"), device="cuda")
        torch.cuda.synchronize()
        k.execute(dev, out, s)
        s.synchronize()
        assert np.array_equal(out.cpu().numpy(), O.reference_compute(doc, xs, threads=8).astype(np.float32)), family


def test_python_mirror_rejects_bad_tensors():
    op, k, xs, nout = _setup(OPS["gemm_tc"])
    dev = [torch.from_numpy(x).cuda() for x in xs]
    out = torch.empty(nout, device="cuda")
    with pytest.raises(ValueError):
        k.execute([dev[0], dev[1]], torch.empty(nout // 2, device="cuda"))  # too small
    with pytest.raises(ValueError):
        k.execute([dev[0].double(), dev[1]], out)  # fp64 storage
    with pytest.raises(ValueError):
        k.execute([dev[0], dev[1]], out.cpu())  # host output for a device execute
    with pytest.raises(ValueError):
        k.execute([dev[0].view(op.tensors[0]["true_dims"]).t(), dev[1]], out)  # non-contiguous view
