"""GPU parity of the tensor-core families (tcgen05) against the CPU oracle.

Bars (stated per variant):
  * integer-valued inputs U{-2..2}: BIT-EXACT for tc_tf32 and tc_bf16 (every product and partial
    sum is exactly representable; fp32 accumulation of integers < 2^24 is exact);
  * U(-1,1) inputs: tc_tf32  max|gpu - oracle| / max|oracle| <= TF32_TOL
                    tc_bf16  (bf16 operands)  <= BF16_TOL
                    tc_3xtf32 (hi/lo tf32 split, fp32-grade) <= X3_TOL = 1e-6, the SPEC's fp32 bar.
Includes the BASELINE configurations at full size (G, C, B).
"""
import json

import numpy as np
import pytest

from conftest import CONFIG_OPS

TF32_TOL = 2e-3
BF16_TOL = 1e-2
X3_TOL = 1e-6  # tc_3xtf32 (fp32-grade): the SPEC's single-precision bar

torch = pytest.importorskip("torch")
g = pytest.importorskip("paper_2502_11407_b200")
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

_HW = {}


def hw():
    if "b200" not in _HW:
        _HW["b200"] = g.HardwareSpec.b200(0)
    return _HW["b200"]


def inputs(op, rng, integer):
    xs = []
    for t in op.tensors[:-1]:
        n = int(np.prod(t["true_dims"])) * op.batch
        x = rng.integers(-2, 3, size=n).astype(np.float32) if integer else rng.uniform(-1, 1, n).astype(np.float32)
        if op.dtype_bytes == 2:
            x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
        xs.append(x)
    return xs


def run(op, sched, variant, xs, nout):
    bf16 = op.dtype_bytes == 2
    k = g.Kernel(op, sched, 0, variant)
    dt = torch.bfloat16 if bf16 else torch.float32
    dev = [torch.from_numpy(x).to(dt).cuda() for x in xs]
    out = torch.full((nout,), float("nan"), dtype=dt, device="cuda")
    k.execute(dev, out)
    torch.cuda.synchronize()
    return out.float().cpu().numpy().astype(np.float64), k.info


def check(doc, variant, tol, seed=0, top_k=1):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, hw(), g.EngineConfig(seed=seed, mode="b200", top_k=top_k))
    rng = np.random.default_rng(seed)
    bf16_out = op.dtype_bytes == 2
    xi = inputs(op, rng, integer=True)
    ref = O.reference_compute(doc, xi, threads=8)
    got, info = run(op, sched, variant, xi, ref.size)
    exp = ref.astype(np.float32).astype(np.float64)
    assert np.array_equal(got, exp), (info["plan"], np.nanmax(np.abs(got - exp)))
    xr = inputs(op, rng, integer=False)
    ref = O.reference_compute(doc, xr, threads=8)
    got, info = run(op, sched, variant, xr, ref.size)
    err = np.nanmax(np.abs(got - ref)) / np.abs(ref).max()
    assert not np.isnan(got).any()
    assert err <= tol, (info["plan"], err)
    return info


GEMMS = [
    {"kind": "gemm", "M": 128, "K": 64, "N": 64},
    {"kind": "gemm", "M": 256, "K": 256, "N": 256},
    {"kind": "gemm", "M": 200, "K": 96, "N": 136},  # ragged M/N tiles, N % 16 != 0
    {"kind": "gemm", "M": 64, "K": 1000, "N": 72},  # K tail inside the last 128 B chunk
]


@pytest.mark.parametrize("doc", GEMMS, ids=lambda d: f"{d['M']}x{d['K']}x{d['N']}")
def test_gemm_tf32(doc):
    info = check(doc, "tc_tf32", TF32_TOL)
    assert info["plan"]["family"] == "gemm_tc"


BGEMMS = [
    {"kind": "gemm", "M": 128, "K": 64, "N": 128, "dtype_bytes": 2, "batch": 3},
    {"kind": "gemm", "M": 96, "K": 48, "N": 80, "dtype_bytes": 2, "batch": 2},
    {"kind": "gemm", "M": 256, "K": 192, "N": 256, "dtype_bytes": 2},
]


@pytest.mark.parametrize("doc", BGEMMS, ids=lambda d: f"{d['M']}x{d['K']}x{d['N']}b{d.get('batch', 1)}")
def test_gemm_bf16(doc):
    info = check(doc, "tc_bf16", BF16_TOL)
    assert info["plan"]["family"] == "gemm_tc"


CONVS = [
    {"kind": "conv2d", "I": [2, 8, 12, 12], "K": [16, 8, 3, 3], "S": 1},
    {"kind": "conv2d", "I": [1, 32, 20, 40], "K": [64, 32, 3, 3], "S": 1},
    {"kind": "conv2d", "I": [2, 64, 10, 70], "K": [40, 64, 1, 1], "S": 1},  # 1x1, F not a power of two
    {"kind": "conv2d", "I": [1, 16, 9, 35], "K": [64, 16, 5, 3], "S": 1},     # H*W % 4 != 0: NHWC copy
    {"kind": "conv2d", "I": [3, 40, 13, 20], "K": [24, 40, 3, 3], "S": 1},    # ragged C, OW, odd N
    {"kind": "conv2d", "I": [1, 24, 11, 12], "K": [96, 24, 2, 4], "S": 1},    # non-square window
    {"kind": "conv2d", "I": [2, 16, 12, 40], "K": [32, 16, 3, 2], "S": 1},    # S = 2: UMMA N = 64
    {"kind": "conv2d", "I": [1, 48, 10, 70], "K": [128, 48, 3, 1], "S": 1},   # S = 1, F = 128: N = 128
    {"kind": "conv2d", "I": [3, 128, 14, 18], "K": [128, 128, 3, 3], "S": 1},  # filters streamed per stage
    {"kind": "conv2d", "I": [2, 96, 11, 13], "K": [100, 96, 3, 3], "S": 1},   # streamed, ragged F / C
    {"kind": "conv2d", "I": [2, 3, 16, 18], "K": [32, 3, 3, 3], "S": 1},      # C = 3: no 16 B NHWC rows
    # conv_flat (flattened NCHW planes, TMA in place): tap offset classes / runs / bank shapes
    {"kind": "conv2d", "I": [2, 32, 12, 14], "K": [48, 32, 3, 3], "S": 1},    # W = 14: split runs, F = 48
    {"kind": "conv2d", "I": [3, 64, 16, 16], "K": [64, 64, 3, 3], "S": 1},    # W % 4 == 0: block 3 unused
    {"kind": "conv2d", "I": [1, 32, 9, 12], "K": [20, 32, 2, 2], "S": 1},     # 4 taps, FN 32 > F
    {"kind": "conv2d", "I": [2, 32, 30, 30], "K": [64, 32, 3, 3], "S": 1},    # 7 tiles per image
    {"kind": "conv2d", "I": [1, 32, 20, 24], "K": [32, 32, 5, 5], "S": 1},    # 25 taps, runs of 4
    {"kind": "conv2d", "I": [1, 96, 10, 10], "K": [16, 96, 3, 3], "S": 1},    # 3 chunks, FN = 16
    # conv_flat CTA pairs (3x3, FN = 64): the four W mod 4 classes, an odd tile count
    {"kind": "conv2d", "I": [2, 32, 12, 13], "K": [64, 32, 3, 3], "S": 1},    # W = 1 (mod 4)
    {"kind": "conv2d", "I": [2, 64, 12, 15], "K": [64, 64, 3, 3], "S": 1},    # W = 3 (mod 4)
    {"kind": "conv2d", "I": [3, 32, 8, 12], "K": [64, 32, 3, 3], "S": 1},     # 3 tiles: the pair's last tile recomputed
]


def flat_ok(doc):
    """conv_flat's envelope (kernels/conv_flat.cu conv_flat_plan): tf32, stride 1, C % 32 == 0,
    F <= 64, H*W % 4 == 0, a window, and the resident bank + 4 A stages fit shared memory."""
    N, C, H, W = doc["I"]
    F, _, R, S = doc["K"]
    if doc.get("S", 1) != 1 or C % 32 or F > 64 or (H * W) % 4 or (R == 1 and S == 1):
        return False
    fn = (F + 15) // 16 * 16
    nfb = fn // 16
    nfbh = (nfb + 1) // 2
    smem = 1024 + (C // 32) * R * S * fn * 128 + 4 * 16384 + 2 * nfbh * 2 * 4 * 96 * 4 + 12 * 8 + 16
    return smem <= 227 * 1024


@pytest.mark.parametrize("doc", CONVS, ids=lambda d: json.dumps(d["I"] + d["K"]))
@pytest.mark.parametrize("variant,tol", [("tc_tf32", TF32_TOL), ("tc_bf16", BF16_TOL)])
def test_conv_tc(doc, variant, tol):
    C = doc["I"][1]
    if variant == "tc_bf16" and (C * 2) % 16:
        # bf16 convs need 16 B channel rows for the NHWC TMA boxes: the family refuses loudly
        op = g.TensorOpSpec.parse_text(json.dumps(doc))
        sched = g.optimize(op, hw(), g.EngineConfig(seed=0, mode="b200", top_k=1))
        with pytest.raises(g.GensorError) as e:
            g.Kernel(op, sched, 0, variant)
        assert e.value.code == "Unsupported"
        return
    info = check(doc, variant, tol)
    # 1x1 tf32 convs take the in-place implicit GEMM (no NHWC pre-pass), windows take conv_tc
    F, S = doc["K"][0], doc["K"][3]
    fn = 32
    while fn < F:
        fn *= 2
    P = doc["I"][2] * doc["I"][3]
    if (variant == "tc_tf32" and doc["K"][2] == 1 and doc["K"][3] == 1 and doc["I"][1] % 4 == 0 and P % 4 == 0
            and (P >= 512 or P % 128 == 0)):
        want = "gemm_tc"    # 1x1 stride 1: batched GEMM O[n] = K . I[n] on the NCHW tensors
    elif variant == "tc_tf32" and flat_ok(doc):
        want = "conv_flat"  # flattened NCHW planes straight through TMA, one launch
    elif variant == "tc_tf32" and (doc["K"][2] == 1 or C % 4):
        want = "conv_gemm"  # other 1x1, and channel counts without 16 B NHWC rows: in-place implicit GEMM
    elif variant == "tc_tf32" and S <= 4 and S * fn <= 256 and C % 4 == 0:
        want = "conv_ns"    # NCHW in place, filter columns folded into the UMMA N
    else:
        want = "conv_tc"    # NHWC copy + TMA boxes
    assert info["plan"]["family"] == want, info["plan"]


@pytest.mark.parametrize("name,variant,tol", [("G", "tc_tf32", TF32_TOL), ("C", "tc_tf32", TF32_TOL),
                                              ("C", "tc_bf16", BF16_TOL), ("B", "tc_bf16", BF16_TOL)])
def test_baseline_configs_full_size(name, variant, tol):
    doc = dict(CONFIG_OPS[name])
    if name == "B":
        doc["batch"] = 192
    check(doc, variant, tol)


# conv_flat programs chosen by the constructed state (tcplan.hpp conv_flat_plan_of): the level-1
# f tile sets the filter group width FN (F splits into FG groups of CTAs, each with its own bank),
# a >= 256-position level-1 h x w tile with one 64-wide group of a 3x3 window takes CTA pairs.
FLAT_GROUP_CONVS = [
    {"kind": "conv2d", "I": [2, 32, 12, 13], "K": [64, 32, 3, 3], "S": 1},   # W = 1 (mod 4)
    {"kind": "conv2d", "I": [2, 64, 12, 15], "K": [64, 64, 3, 3], "S": 1},   # W = 3 (mod 4)
    {"kind": "conv2d", "I": [3, 64, 16, 16], "K": [64, 64, 3, 3], "S": 1},   # W = 0 (mod 4)
    {"kind": "conv2d", "I": [2, 32, 30, 30], "K": [64, 32, 3, 3], "S": 1},   # W = 2 (mod 4), 7 tiles / image
    {"kind": "conv2d", "I": [2, 32, 12, 14], "K": [48, 32, 3, 3], "S": 1},   # last group partly past F
    {"kind": "conv2d", "I": [1, 32, 9, 12], "K": [20, 32, 2, 2], "S": 1},    # FN 16, 4 taps
    {"kind": "conv2d", "I": [1, 32, 20, 24], "K": [32, 32, 5, 5], "S": 1},   # 25 taps, table-driven issue
    {"kind": "conv2d", "I": [2, 128, 10, 12], "K": [64, 128, 3, 3], "S": 1},  # whole-F bank too big: groups only
]


def _pow2(x):
    p = 1
    while p < x:
        p *= 2
    return p


@pytest.mark.parametrize("split", [1, 2, 4])
@pytest.mark.parametrize("doc", FLAT_GROUP_CONVS, ids=lambda d: json.dumps(d["I"] + d["K"]))
def test_conv_flat_from_state(doc, split):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    F, C, R, S = doc["K"][0], doc["I"][1], doc["K"][2], doc["K"][3]
    tf = _pow2(F) // split
    f16 = (F + 15) // 16 * 16
    fn = min(f16, min(64, max(16, (tf + 15) // 16 * 16)))
    fg = (F + fn - 1) // fn
    bank = C // 32 * R * S * fn * 128
    if bank + 4 * 16384 + 12288 + 2048 > 227 * 1024:
        pytest.skip("the group's bank does not fit next to the ring")
    trace = ([[0, 1, split]] if split > 1 else []) + [[3, -1, 0], [3, -1, 0]]
    sched = g.from_trace(op, hw(), trace, mode="b200")
    rng = np.random.default_rng(split)
    for integer in (True, False):
        xs = inputs(op, rng, integer=integer)
        ref = O.reference_compute(doc, xs, threads=8)
        got, info = run(op, sched, "tc_tf32", xs, ref.size)
        plan = info["plan"]
        assert plan["family"] == "conv_flat" and plan["FN"] == fn and plan["filter_groups"] == fg, plan
        if fg > 1:
            assert not plan["cta_pair"], plan
        if integer:
            assert np.array_equal(got, ref.astype(np.float32).astype(np.float64)), (plan, np.nanmax(np.abs(got - ref)))
        else:
            assert not np.isnan(got).any()
            assert np.nanmax(np.abs(got - ref)) / np.abs(ref).max() <= TF32_TOL, plan


def test_conv_flat_groups_distinct_programs():
    """The headline conv's program follows the state: a state whose level-1 f tile is half of F
    runs two filter groups, the construction's pick runs one group on CTA pairs; same results."""
    doc = CONFIG_OPS["C"]
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    best = g.optimize(op, hw(), g.EngineConfig(seed=0, mode="b200", top_k=1))
    split = g.from_trace(op, hw(), [[0, 1, 2], [3, -1, 0], [3, -1, 0]], mode="b200")
    rng = np.random.default_rng(1)
    xs = inputs(op, rng, integer=True)
    a, ia = run(op, best, "tc_tf32", xs, int(np.prod(op.tensors[-1]["true_dims"])))
    b, ib = run(op, split, "tc_tf32", xs, a.size)
    assert ia["plan"]["filter_groups"] == 1 and ia["plan"]["cta_pair"], ia["plan"]
    assert ib["plan"]["filter_groups"] == 2 and ib["plan"]["FN"] == 32, ib["plan"]
    assert np.array_equal(a, b)


def test_auto_picks_tensor_cores():
    for name in ("G", "C"):
        op = g.TensorOpSpec.parse_text(json.dumps(CONFIG_OPS[name]))
        sched = g.optimize(op, hw(), g.EngineConfig(mode="b200", top_k=1))
        k = g.Kernel(op, sched, 0, "auto")
        assert k.info["variant_name"] == "tc_tf32"


# General implicit-GEMM conv (conv_gemm: NCHW read in place, any stride / window / channels):
# the shapes conv_tc does not take — stride 2, ResNet stem (C=3, 7x7), F > 256, odd batch.
GEMM_CONVS = [
    {"kind": "conv2d", "I": [2, 16, 17, 17], "K": [32, 16, 3, 3], "S": 2},
    {"kind": "conv2d", "I": [1, 64, 9, 9], "K": [300, 64, 1, 1], "S": 1},       # F > 256, ragged N tile
    {"kind": "conv2d", "I": [2, 96, 8, 8], "K": [128, 96, 1, 1], "S": 2},      # 1x1 stride-2 projection
]


@pytest.mark.parametrize("doc", GEMM_CONVS, ids=lambda d: json.dumps(d["I"] + d["K"] + [d["S"]]))
def test_conv_gemm_tf32(doc):
    info = check(doc, "tc_tf32", TF32_TOL)
    assert info["plan"]["family"] == "conv_gemm"


# stride-1 windows whose filter bank does not fit in shared memory: conv_tc streams the R filter
# blocks of each (s, channel chunk) stage next to its A box
STREAMED = [
    {"kind": "conv2d", "I": [1, 512, 9, 9], "K": [64, 512, 3, 3], "S": 1},     # large C
    {"kind": "conv2d", "I": [2, 128, 30, 30], "K": [128, 128, 3, 3], "S": 1},  # ResNet-50 res3 shape
    {"kind": "conv2d", "I": [3, 256, 16, 16], "K": [256, 256, 3, 3], "S": 1},  # F = 256: 2 filter groups
    {"kind": "conv2d", "I": [2, 64, 12, 12], "K": [200, 64, 3, 3], "S": 1},    # ragged second group
]


@pytest.mark.parametrize("doc", STREAMED, ids=lambda d: json.dumps(d["I"] + d["K"]))
def test_conv_tc_streamed(doc):
    info = check(doc, "tc_tf32", TF32_TOL)
    assert info["plan"]["family"] == "conv_tc", info["plan"]


# stride-2 few-channel convs (the ResNet stem) through conv_ns on their space-to-depth form
S2D = [
    {"kind": "conv2d", "I": [3, 3, 23, 23], "K": [64, 3, 7, 7], "S": 2},      # stem shape, odd sizes
    {"kind": "conv2d", "I": [2, 3, 229, 229], "K": [64, 3, 7, 7], "S": 2},    # ResNet-50 stem, batch 2
    {"kind": "conv2d", "I": [2, 8, 30, 34], "K": [40, 8, 3, 3], "S": 2},      # 4C = 32 channels, F = 40
    {"kind": "conv2d", "I": [1, 5, 17, 16], "K": [32, 5, 4, 2], "S": 2},      # even window, ragged 4C
]


@pytest.mark.parametrize("doc", S2D, ids=lambda d: json.dumps(d["I"] + d["K"]))
def test_conv_s2d(doc):
    info = check(doc, "tc_tf32", TF32_TOL)
    assert info["plan"]["family"] == "conv_ns" and "space_to_depth" in info["plan"], info["plan"]


# 1x1 stride-1 convs as batched GEMMs with the filter bank shared by the batch (gemm_tc, A_shared)
CONV1X1 = [
    {"kind": "conv2d", "I": [3, 64, 24, 30], "K": [256, 64, 1, 1], "S": 1},    # P = 720: ragged N tiles
    {"kind": "conv2d", "I": [2, 256, 28, 28], "K": [64, 256, 1, 1], "S": 1},   # F = 64 < BM
    {"kind": "conv2d", "I": [5, 36, 16, 32], "K": [200, 36, 1, 1], "S": 1},    # ragged F, C
]


@pytest.mark.parametrize("doc", CONV1X1, ids=lambda d: json.dumps(d["I"] + d["K"]))
def test_conv1x1_gemm(doc):
    info = check(doc, "tc_tf32", TF32_TOL)
    assert info["plan"]["family"] == "gemm_tc" and "conv1x1" in info["plan"], info["plan"]


X3_GEMMS = GEMMS + [
    {"kind": "gemm", "M": 1024, "K": 1024, "N": 1024},  # BASELINE configs[0] (G) at full size
    {"kind": "gemm", "M": 300, "K": 2048, "N": 200},    # long k-loop, ragged tiles
    {"kind": "gemm", "M": 128, "K": 64, "N": 64, "batch": 3},
]


@pytest.mark.parametrize("doc", X3_GEMMS, ids=lambda d: f"{d['M']}x{d['K']}x{d['N']}b{d.get('batch', 1)}")
def test_gemm_3xtf32(doc):
    info = check(doc, "tc_3xtf32", X3_TOL)
    assert info["plan"]["family"] == "gemm_tc" and "split" in info["plan"], info["plan"]


def test_3xtf32_beats_tf32_accuracy():
    """The split recovers what tf32 rounding loses: on G the 3xTF32 error is orders of magnitude
    below the 1xTF32 one (and below the fp32 bar)."""
    doc = {"kind": "gemm", "M": 512, "K": 1024, "N": 512}
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    sched = g.optimize(op, hw(), g.EngineConfig(seed=0, mode="b200", top_k=1))
    rng = np.random.default_rng(5)
    xs = inputs(op, rng, integer=False)
    ref = O.reference_compute(doc, xs, threads=8)
    e1 = np.abs(run(op, sched, "tc_tf32", xs, ref.size)[0] - ref).max() / np.abs(ref).max()
    e3 = np.abs(run(op, sched, "tc_3xtf32", xs, ref.size)[0] - ref).max() / np.abs(ref).max()
    assert e3 <= X3_TOL and e3 * 50 < e1, (e1, e3)
