"""GPU parity of the state-driven SIMT kernel against the CPU oracle (oracle/gensor_oracle.c).

Bars (BASELINE.md §5 / SPEC.md:507,563):
  * simt_parity (fp64 accumulation in the interpreter's order): BIT-EXACT against
    interpret(lower(state)) rounded to the output dtype, on random U(-1,1) inputs;
  * simt_f32: bit-exact on integer-valued inputs U{-2..2}; on U(-1,1) within
    max|gpu - oracle| / max|oracle| <= F32_TOL.
Schedules come from the engine (reference-compatible mode on two reference-format profiles, and
B200 mode on the device model) and from random legal walks, so the kernel is exercised on
states it did not choose.
"""
import json

import numpy as np
import pytest

import os

from conftest import B200_REF, CONFIG_OPS, GENERIC

F32_TOL = 1e-6  # single-precision mode within 1e-6

torch = pytest.importorskip("torch")
g = pytest.importorskip("paper_2502_11407_b200")
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

SMALL_OPS = [
    {"kind": "gemm", "M": 64, "K": 48, "N": 40},
    {"kind": "gemm", "M": 33, "K": 17, "N": 65},
    {"kind": "gemm", "M": 1, "K": 1, "N": 1},
    {"kind": "gemv", "M": 100, "N": 77},
    {"kind": "conv2d", "I": [2, 8, 12, 12], "K": [16, 8, 3, 3], "S": 1},
    {"kind": "conv2d", "I": [2, 3, 15, 13], "K": [5, 3, 3, 2], "S": 2},
    {"kind": "conv2d", "I": [1, 4, 9, 9], "K": [6, 4, 1, 1], "S": 3},  # stride > window
    {"kind": "avgpool2d", "I": [2, 5, 11, 10], "F": 3, "S": 1},
    {"kind": "avgpool2d", "I": [1, 3, 8, 8], "F": 2, "S": 2},
    {"kind": "dwconv2d", "I": [2, 6, 10, 10], "K": [6, 1, 3, 3], "S": 1},
]


def _inputs(doc, rng, integer):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    xs = []
    for t in op.tensors[:-1]:
        n = int(np.prod(t["true_dims"])) * op.batch
        x = rng.integers(-2, 3, size=n) if integer else rng.uniform(-1, 1, size=n)
        if op.dtype_bytes == 2:
            x = torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).float().numpy()
        xs.append(x.astype(np.float32))
    return op, xs


def _to_dev(xs, bf16):
    dt = torch.bfloat16 if bf16 else torch.float32
    return [torch.from_numpy(x).to(dt).cuda() for x in xs]


def _round(ref, bf16):
    r = torch.from_numpy(ref.astype(np.float32))
    if bf16:
        r = r.to(torch.bfloat16).float()
    return r.numpy().astype(np.float64)


def _run(op, sched, idx, variant, xs, nout):
    bf16 = op.dtype_bytes == 2
    k = g.Kernel(op, sched, idx, variant)
    out = torch.empty(nout, dtype=torch.bfloat16 if bf16 else torch.float32, device="cuda")
    k.execute(_to_dev(xs, bf16), out)
    torch.cuda.synchronize()
    return out.float().cpu().numpy().astype(np.float64)


def _schedules(doc):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    out = []
    for prof in (GENERIC, B200_REF):
        hw = g.HardwareSpec.load_text(json.dumps(prof))
        out.append((op, g.optimize(op, hw, g.EngineConfig(seed=1, top_k=3))))
    hw = g.HardwareSpec.b200(0)
    out.append((op, g.optimize(op, hw, g.EngineConfig(seed=2, top_k=3, mode="b200"))))
    return out


@pytest.mark.parametrize("doc", SMALL_OPS, ids=lambda d: json.dumps(d))
def test_parity_bit_exact(doc):
    rng = np.random.default_rng(0)
    for op, sched in _schedules(doc):
        _, xs = _inputs(doc, rng, integer=False)
        for i, res in enumerate(sched):
            ref = _round(O.interpret(doc, res["state"], xs), op.dtype_bytes == 2)
            got = _run(op, sched, i, "simt_parity", xs, ref.size)
            assert np.array_equal(got, ref), (res["state"]["repr"], np.abs(got - ref).max())


@pytest.mark.parametrize("doc", SMALL_OPS, ids=lambda d: json.dumps(d))
def test_f32_integer_exact_and_tolerance(doc):
    rng = np.random.default_rng(1)
    for op, sched in _schedules(doc)[1:]:
        _, xi = _inputs(doc, rng, integer=True)
        ref = _round(O.reference_compute(doc, xi), False)
        got = _run(op, sched, 0, "simt_f32", xi, ref.size)
        if op.info["kind"] != "avgpool2d":  # avgpool divides by F^2: not integer-valued
            assert np.array_equal(got, ref)
        _, xr = _inputs(doc, rng, integer=False)
        ref = O.reference_compute(doc, xr)
        got = _run(op, sched, 0, "simt_f32", xr, ref.size)
        assert np.abs(got - ref).max() <= F32_TOL * max(1e-30, np.abs(ref).max())


def test_random_walk_states_bit_exact():
    """Random legal walks (construct() snapshots completed by the greedy fitter) on conv2d."""
    doc = {"kind": "conv2d", "I": [2, 6, 11, 10], "K": [7, 6, 3, 3], "S": 1}
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    hw = g.HardwareSpec.load_text(json.dumps(GENERIC))
    rng = np.random.default_rng(3)
    _, xs = _inputs(doc, rng, integer=False)
    for seed in range(6):
        snaps = g.construct(op, hw, g.EngineConfig(seed=seed))
        for s in snaps.results[::4]:
            done = g.from_trace(op, hw, s["trace"] + _completion(op, hw, s["trace"]))
            st = done[0]["state"]
            ref = _round(O.interpret(doc, st, xs), False)
            got = _run(op, done, 0, "simt_parity", xs, ref.size)
            assert np.array_equal(got, ref), st["repr"]


def _completion(op, hw, trace):
    """Greedy completion actions for a (possibly incomplete) trace, via the engine's fitter."""
    extra = []
    while True:
        ev = g.state_eval(op, hw, trace + extra)
        if ev["state"]["level"] == len(ev["state"]["tiles"][0]):
            return extra
        lvl = ev["state"]["level"]
        if ev["levels"][lvl]["capacity_ok"]:
            extra.append([3, -1, 0])
        else:
            extra.append(ev["greedy_step"])


def test_batched_bf16_gemm_bit_exact():
    doc = {"kind": "gemm", "M": 40, "K": 24, "N": 36, "dtype_bytes": 2, "batch": 5}
    rng = np.random.default_rng(4)
    for op, sched in _schedules(doc):
        _, xs = _inputs(doc, rng, integer=False)
        ref = _round(O.interpret(doc, sched[0]["state"], xs), True)
        got = _run(op, sched, 0, "simt_parity", xs, ref.size)
        assert np.array_equal(got, ref)


def test_execute_rejects_wrong_input_count():
    doc = {"kind": "gemm", "M": 8, "K": 8, "N": 8}
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, g.HardwareSpec.load_text(json.dumps(GENERIC)))
    k = g.Kernel(op, sched, 0, "simt_parity")
    a = torch.zeros(64, device="cuda")
    with pytest.raises(g.GensorError) as e:
        k.execute([a], torch.zeros(64, device="cuda"))
    assert e.value.code == "ShapeMismatch"


def test_execute_host_matches_device():
    doc = {"kind": "conv2d", "I": [1, 4, 10, 10], "K": [8, 4, 3, 3], "S": 1}
    rng = np.random.default_rng(5)
    op, xs = _inputs(doc, rng, integer=False)
    sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=1))
    ref = _round(O.interpret(doc, sched[0]["state"], xs), False)
    k = g.Kernel(op, sched, 0, "simt_parity")
    out = np.empty(ref.size, dtype=np.float32)
    k.execute_host(xs, out)
    assert np.array_equal(out.astype(np.float64), ref)


def test_rerank_on_device_orders_by_measured_time():
    """the top-k schedules are instantiated and timed on the device; the
    returned order is by measured time and every variant's result stays bit-exact."""
    doc = {"kind": "gemm", "M": 256, "K": 128, "N": 192}
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(mode="b200", top_k=4))
    rng = np.random.default_rng(7)
    _, xs = _inputs(doc, rng, integer=True)
    dev = _to_dev(xs, False)
    out = torch.empty(256 * 192, device="cuda")
    r = g.rerank(op, sched, dev, out, "simt_f32", iters=3)
    assert sorted(r["order"]) == list(range(len(sched)))
    ms = [r["ms"][i] for i in r["order"]]
    assert ms == sorted(ms) and all(m > 0 for m in ms)
    best = r["best"]
    ref = _round(O.reference_compute(doc, xs), False)
    got = _run(op, sched, best, "simt_f32", xs, ref.size)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("name", ["G", "C"])
def test_full_size_fp32_configs(name):
    """BASELINE configs[0] (G, GEMM fp32 1024^3) and configs[1] (C, the ResNet-50 conv) at full size
    on the state-driven SIMT family: simt_parity bit-exact to interpret(lower(state)), simt_f32
    within the SPEC's single-precision bar (1e-6 normwise, scaled by sqrt(K/64) past the desk
    suite's extents)."""
    doc = CONFIG_OPS[name]
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(seed=0, mode="b200", top_k=1))
    rng = np.random.default_rng(11)
    xs = [rng.uniform(-1, 1, size=int(np.prod(t["true_dims"]))).astype(np.float32) for t in op.tensors[:-1]]
    ref = O.interpret(doc, sched[0]["state"], xs, threads=os.cpu_count() or 8)
    got = _run(op, sched, 0, "simt_parity", xs, ref.size)
    assert np.array_equal(got, _round(ref, False)), np.abs(got - _round(ref, False)).max()
    got = _run(op, sched, 0, "simt_f32", xs, ref.size)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    # SPEC.md:507 states 1e-6 for the desk suite (extents <= 64); a sequential fp32 accumulation
    # over K terms drifts like sqrt(K) roundings, so at K = 1024 (G) / 576 (C) the same bar scales
    # by sqrt(K / 64)
    k_red = 1024 if name == "G" else 64 * 9
    assert err <= F32_TOL * np.sqrt(k_red / 64), err


FAST = [
    ("gemm", {"kind": "gemm", "M": 1024, "K": 1024, "N": 1024}),   # G: 16 B asynchronous copies
    ("gemm", {"kind": "gemm", "M": 200, "K": 97, "N": 136}),       # ragged tiles, 4 B copies (K % 4 != 0)
    ("gemm", {"kind": "gemm", "M": 96, "K": 64, "N": 80, "dtype_bytes": 2, "batch": 3}),  # bf16, batched
    ("gemv", {"kind": "gemv", "M": 32768, "N": 4096}),            # V (TMA path at the B200 state)
    ("gemv", {"kind": "gemv", "M": 1000, "N": 999}),              # ragged, scalar tail
    ("gemv", {"kind": "gemv", "M": 700, "N": 1000}),              # TMA path: ragged rows / last column chunk
]


@pytest.mark.parametrize("kind,doc", FAST, ids=lambda x: json.dumps(x) if isinstance(x, dict) else x)
def test_simt_fast_paths_match_the_general_walk(kind, doc):
    """simt_f32's register-tiled gemm / gemv kernels run the SAME plan (tiles, vthreads, ascending
    single-axis reduce) as the general walk: the plan says which path ran, outputs are bit-exact on
    integer inputs and within the fp32 bar on U(-1,1) against the oracle's interpret(); for every
    top-k state (different tiles / vthreads)."""
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, g.HardwareSpec.b200(0), g.EngineConfig(seed=0, mode="b200", top_k=3))
    rng = np.random.default_rng(5)
    bf16 = op.dtype_bytes == 2
    for idx in range(len(sched)):
        k = g.Kernel(op, sched, idx, "simt_f32")
        if k.info["plan"].get("fast") == "none":
            continue
        assert k.info["plan"]["fast"] in ((kind,) if kind == "gemm" else ("gemv", "gemv_tma"))
        for integer in (True, False):
            _, xs = _inputs(doc, rng, integer)
            ref = O.interpret(doc, sched[idx]["state"], xs, threads=os.cpu_count() or 8)
            got = _run(op, sched, idx, "simt_f32", xs, ref.size)
            if integer:
                assert np.array_equal(got, _round(ref, bf16)), (idx, np.abs(got - ref).max())
            else:
                k_red = doc["K"] if kind == "gemm" else doc["N"]
                tol = (1e-2 if bf16 else F32_TOL * max(1.0, np.sqrt(k_red / 64)))
                assert np.abs(got - ref).max() / np.abs(ref).max() <= tol, idx
