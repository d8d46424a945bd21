"""Known-answer tests of the SPEC, through the product C-ABI.

Construct-side KATs are the SPEC's [DERIVED] examples for the cost model and engine
(SPEC.md:145-306); the survey re-verified each against the compiled reference.
"""
import json
import math

import pytest

from conftest import GENERIC

g = pytest.importorskip("paper_2502_11407_b200")


def gemm(m, k, n, **kw):
    return g.TensorOpSpec.parse_text(json.dumps({"kind": "gemm", "M": m, "K": k, "N": n, **kw}))


def hw_generic():
    return g.HardwareSpec.load_text(json.dumps(GENERIC))


# GEMM 64^3 trace to level-1 tile (8,8,64): Tile(m,2)x3, Tile(n,2)x3 at level 1
T_8_8_64 = [[0, 0, 2]] * 3 + [[0, 1, 2]] * 3
T_16_8_64 = [[0, 0, 2]] * 2 + [[0, 1, 2]] * 3


def test_traffic_kats():
    op, hw = gemm(64, 64, 64), hw_generic()
    ev = g.state_eval(op, hw, T_8_8_64)
    assert ev["state"]["tiles"][0][0] == 8 and ev["state"]["tiles"][1][0] == 8 and ev["state"]["tiles"][2][0] == 64
    assert ev["levels"][0]["traffic"] == 69632
    assert g.state_eval(op, hw, T_16_8_64)["levels"][0]["traffic"] == 53248


def test_footprint_and_tiling_benefit():  # SPEC.md:200, acceptance criterion 2
    op, hw = gemm(64, 64, 64), hw_generic()
    f1 = g.state_eval(op, hw, T_8_8_64)["levels"][0]["footprint"]
    f2 = g.state_eval(op, hw, T_16_8_64)["levels"][0]["footprint"]
    assert (f1, f2) == (1088, 1664)
    cands = g.enumerate_candidates(op, hw, T_8_8_64, iteration=0)
    inv_m = [c for c in cands if c[0] == [1, 0, 2]][0]  # InvTile(m,2): (8,8,64) -> (16,8,64)
    assert inv_m[1] == 2.0


def test_capacity_kat():  # (16,8,64) fp32 -> 6656 B
    op, hw = gemm(64, 64, 64), hw_generic()
    assert g.state_eval(op, hw, T_16_8_64)["levels"][0]["footprint_bytes"] == 6656


def test_formula_kats():
    assert g.caching_benefit(400, 512, 20, 4096, 16384) == 18.0
    assert g.vthread_conflict_ratio(64, 32, 2) == 2.0
    assert g.vthread_conflict_ratio(48, 32, 4) == 2.0
    assert g.vthread_conflict_ratio(77, 32, 1) == 1.0
    assert abs(g.anneal_cache_multiplier(10) - 1.5) < 1e-12
    assert abs(g.record_probability(math.exp(-10)) - 0.5) < 1e-12
    assert g.caching_benefit(7, 9, 7, 9, 123.0) == 1.0


def test_gemv_traffic_kat():  # GEMV 16x8 tile (4,8) -> 176
    op = g.TensorOpSpec.parse_text('{"kind":"gemv","M":16,"N":8}')
    ev = g.state_eval(op, hw_generic(), [[0, 0, 2], [0, 0, 2]])
    assert ev["levels"][0]["traffic"] == 176


def test_conv_output_extent_kat():  # floor((30-3)/2)+1 = 14
    op = g.TensorOpSpec.parse_text('{"kind":"conv2d","I":[128,256,30,30],"K":[256,256,3,3],"S":2}')
    assert [a["extent"] for a in op.axes][:4] == [128, 256, 14, 14]


def test_twenty_iterations():  # t0=2^20, threshold=1 -> exactly 20 iterations
    op, hw = gemm(64, 64, 64), hw_generic()
    for seed in range(5):
        snaps = g.construct(op, hw, g.EngineConfig(seed=seed)).results
        assert max(s["iterations"] for s in snaps) == 20
        assert len(snaps[-1]["trace"]) == 20


def test_initial_state_kats():  # SPEC.md: initial_state examples
    op, hw = gemm(64, 64, 64), hw_generic()
    ev = g.state_eval(op, hw, [])
    assert ev["state"]["tiles"] == [[64, 64], [64, 64], [64, 64]]
    assert ev["state"]["vthreads"] == [1, 1, 1] and ev["state"]["level"] == 0
    gv = g.TensorOpSpec.parse_text('{"kind":"gemv","M":16,"N":8}')
    assert g.state_eval(gv, hw, [])["state"]["tiles"] == [[16, 16], [8, 8]]


def test_apply_examples():  # SPEC.md: apply_action examples
    op, hw = gemm(64, 64, 64), hw_generic()
    assert g.state_eval(op, hw, [[0, 0, 2]])["state"]["tiles"][0] == [32, 32]
    ev = g.state_eval(op, hw, [[3, -1, 0]])
    assert ev["state"]["level"] == 1
    ev = g.state_eval(op, hw, [[3, -1, 0], [0, 0, 2], [0, 0, 2], [0, 0, 2], [2, 0, 2]])
    assert ev["state"]["vthreads"][0] == 2 and ev["state"]["tiles"][0] == [64, 8]


def test_unit_gemm_parses():
    op = gemm(1, 1, 1)
    assert [a["extent"] for a in op.axes] == [1, 1, 1]
    res = g.optimize(op, hw_generic())
    assert len(res) >= 1
