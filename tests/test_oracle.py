"""Pins the C execute oracle (oracle/gensor_oracle.c) before it is trusted as the GPU checker.

The reference's execute step is absent from the snapshot (lowering.cpp); its only golden
vectors are the SPEC's codegen-interp examples, reproduced here, plus the
schedule-independence property interpret(lower(s)) == reference_compute within 1e-9
 over engine-constructed schedules, and a numpy cross-check of the formulas.
"""
import json

import numpy as np
import pytest

from conftest import B200_REF, GENERIC
from oracle import oracle as O

g = pytest.importorskip("paper_2502_11407_b200")


def test_spec_kat_gemm_all_ones():
    out = O.reference_compute({"kind": "gemm", "M": 4, "K": 4, "N": 4}, [np.ones(16), np.ones(16)])
    assert np.all(out == 4.0)


def test_spec_kat_avgpool_constant():
    x = np.full(2 * 3 * 8 * 8, 1.75)
    out = O.reference_compute({"kind": "avgpool2d", "I": [2, 3, 8, 8], "F": 2, "S": 2}, [x])
    assert np.all(out == 1.75)


def test_spec_kat_gemv():
    out = O.reference_compute({"kind": "gemv", "M": 2, "N": 2}, [np.array([1, 2, 3, 4]), np.array([1, 1])])
    assert out.tolist() == [3.0, 7.0]


def test_spec_kat_unit_conv_identity():
    x = np.arange(25, dtype=np.float32)
    out = O.reference_compute({"kind": "conv2d", "I": [1, 1, 5, 5], "K": [1, 1, 1, 1], "S": 1}, [x, np.ones(1)])
    assert np.array_equal(out, x.astype(np.float64))


def test_spec_kat_avgpool_mean():
    out = O.reference_compute({"kind": "avgpool2d", "I": [1, 1, 2, 2], "F": 2, "S": 2}, [np.array([1, 2, 3, 4])])
    assert out.tolist() == [2.5]


def _np_ref(doc, xs):
    k = doc["kind"]
    if k == "gemm":
        b = doc.get("batch", 1)
        A = xs[0].astype(np.float64).reshape(b, doc["M"], doc["K"])
        B = xs[1].astype(np.float64).reshape(b, doc["K"], doc["N"])
        return (A @ B).reshape(-1)
    if k == "gemv":
        return xs[0].astype(np.float64).reshape(doc["M"], doc["N"]) @ xs[1].astype(np.float64)
    n, c, h, w = doc["I"]
    S = doc.get("S", 1)
    I = xs[0].astype(np.float64).reshape(n, c, h, w)
    if k == "conv2d":
        f, _, r, s = doc["K"]
        K = xs[1].astype(np.float64).reshape(f, c, r, s)
    elif k == "dwconv2d":
        _, _, r, s = doc["K"]
        K = xs[1].astype(np.float64).reshape(c, r, s)
    else:
        r = s = doc["F"]
    oh, ow = (h - r) // S + 1, (w - s) // S + 1
    win = np.lib.stride_tricks.sliding_window_view(I, (r, s), axis=(2, 3))[:, :, ::S, ::S][:, :, :oh, :ow]
    if k == "conv2d":
        return np.einsum("nchwrs,fcrs->nfhw", win, K).reshape(-1)
    if k == "dwconv2d":
        return np.einsum("nchwrs,crs->nchw", win, K).reshape(-1)
    return win.mean(axis=(4, 5)).reshape(-1)


OPS = [
    {"kind": "gemm", "M": 33, "K": 70, "N": 17},
    {"kind": "gemm", "M": 9, "K": 5, "N": 7, "batch": 3},
    {"kind": "gemv", "M": 50, "N": 31},
    {"kind": "conv2d", "I": [2, 5, 11, 9], "K": [3, 5, 3, 2], "S": 2},
    {"kind": "conv2d", "I": [1, 3, 7, 7], "K": [4, 3, 1, 1], "S": 3},
    {"kind": "avgpool2d", "I": [2, 3, 9, 10], "F": 3, "S": 1},
    {"kind": "dwconv2d", "I": [2, 4, 8, 9], "K": [4, 1, 3, 3], "S": 2},
]


def _inputs(doc, rng):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    return op, [rng.uniform(-1, 1, int(np.prod(t["true_dims"])) * op.batch).astype(np.float32)
                for t in op.tensors[:-1]]


@pytest.mark.parametrize("doc", OPS, ids=lambda d: d["kind"])
def test_reference_compute_matches_numpy(doc):
    _, xs = _inputs(doc, np.random.default_rng(0))
    ref = O.reference_compute(doc, xs)
    assert np.allclose(ref, _np_ref(doc, xs), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("doc", OPS, ids=lambda d: d["kind"])
def test_schedule_independence(doc):
    """interpret(lower(s)) == reference_compute within 1e-9 for every engine schedule."""
    op, xs = _inputs(doc, np.random.default_rng(1))
    ref = O.reference_compute(doc, xs, threads=2)
    for prof in (GENERIC, B200_REF):
        hw = g.HardwareSpec.load_text(json.dumps(prof))
        for seed in (0, 5):
            for res in g.optimize(op, hw, g.EngineConfig(seed=seed, top_k=4)):
                got = O.interpret(doc, res["state"], xs, threads=2)
                scale = max(1e-30, np.abs(ref).max())
                assert np.abs(got - ref).max() <= 1e-9 * scale, res["state"]["repr"]
        for res in g.construct_tree(op, hw, 2):
            got = O.interpret(doc, res["state"], xs)
            assert np.abs(got - ref).max() <= 1e-9 * max(1e-30, np.abs(ref).max())


def test_guarded_iterations_skipped():
    """A NaN in a padded-region-adjacent input element must not leak into any output: the
    interpreter skips guarded iterations instead of multiplying by zero."""
    doc = {"kind": "conv2d", "I": [1, 1, 6, 6], "K": [1, 1, 3, 3], "S": 1}
    x = np.arange(36, dtype=np.float32)
    k = np.ones(9, dtype=np.float32)
    st = {"tiles": [[1, 1], [1, 1], [4, 1], [4, 1], [1, 1], [4, 1], [4, 1]], "vthreads": [1] * 7}
    out = O.interpret(doc, st, [x, k])
    assert np.array_equal(out, O.reference_compute(doc, [x, k]))


def test_softmax_rows_sum_to_one():
    x = np.random.default_rng(2).normal(0, 2, 5 * 33).astype(np.float32)
    out = O.reference_compute({"kind": "softmax", "M": 5, "N": 33}, [x]).reshape(5, 33)
    assert np.allclose(out.sum(1), 1.0, atol=1e-14)
    e = np.exp(x.reshape(5, 33).astype(np.float64) - x.reshape(5, 33).max(1, keepdims=True))
    assert np.allclose(out, e / e.sum(1, keepdims=True), rtol=1e-14)
