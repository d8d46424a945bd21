"""The B200 construction model on CPU (nominal device limits, `gensor_hw_b200(-1)`): the
tensor-core program a state instantiates is what its cost prices (host/tcplan.hpp, host/cost.cpp
estimate_b200), and the suite's LPT weights are the predicted times of the programs `auto` runs."""
import json

import pytest

g = pytest.importorskip("paper_2502_11407_b200")
from paper_2502_11407_b200 import shard  # noqa: E402

C = {"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1}
G = {"kind": "gemm", "M": 1024, "K": 1024, "N": 1024}


def _hw():
    return g.HardwareSpec.b200(-1)


def _cost(doc, trace):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    return g.from_trace(op, _hw(), trace, mode="b200")[0]["cost"]


def test_conv_state_prices_its_conv_flat_program():
    # level-1 f tile 64 / 32 / 16 -> filter groups of 64 / 32 / 16; a >= 256-position h x w tile
    # with one 64-wide group -> CTA pairs (half the bank per CTA)
    pair = _cost(C, [[3, -1, 0], [3, -1, 0]])
    single = _cost(C, [[0, 2, 8], [0, 3, 4], [3, -1, 0], [3, -1, 0]])
    fn32 = _cost(C, [[0, 1, 2], [3, -1, 0], [3, -1, 0]])
    fn16 = _cost(C, [[0, 1, 4], [3, -1, 0], [3, -1, 0]])
    e = [c["est_seconds"] for c in (pair, single, fn32, fn16)]
    assert e[0] < e[1] < e[2] < e[3], e
    assert all(c["exec_seconds"] == c["est_seconds"] for c in (pair, single, fn32, fn16))
    # the construction's pick for config C is a one-group state on pairs
    op = g.TensorOpSpec.parse_text(json.dumps(C))
    best = g.optimize(op, _hw(), g.EngineConfig(seed=0, mode="b200", top_k=1))[0]
    assert best["cost"]["est_seconds"] == pytest.approx(e[0])


def test_small_conv_prefers_filter_groups():
    # few position tiles (2 images of 10 x 15 outputs): splitting F fills more SMs
    doc = {"kind": "conv2d", "I": [2, 64, 12, 15], "K": [64, 64, 3, 3], "S": 1}
    whole = _cost(doc, [[3, -1, 0], [3, -1, 0]])
    split = _cost(doc, [[0, 1, 4], [3, -1, 0], [3, -1, 0]])
    assert split["est_seconds"] < whole["est_seconds"]


def test_gemm_state_is_a_umma_tile():
    op = g.TensorOpSpec.parse_text(json.dumps(G))
    res = g.optimize(op, _hw(), g.EngineConfig(seed=0, mode="b200", top_k=10))
    for r in res:
        tiles = r["state"]["tiles"]
        assert tiles[0][0] == 128  # UMMA M = 128 rows (cta_group::1)
        assert 16 <= tiles[1][0] <= 128  # UMMA N within the tf32 epilogue limit
        assert tiles[2][0] * 4 >= 256  # >= two 128 B k-blocks in the ring


def test_hbm_family_exec_time():
    doc = {"kind": "gemv", "M": 32768, "N": 4096}
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    cost = g.optimize(op, _hw(), g.EngineConfig(seed=0, mode="b200", top_k=1))[0]["cost"]
    hw = _hw().to_json()
    bw = hw["levels"][0]["bandwidth_bytes_per_cycle"] * hw["clock_hz"]  # the measured copy bandwidth
    assert cost["exec_seconds"] == pytest.approx(op.bytes / (0.8 * bw) + 5e-6, rel=1e-6)


def test_lpt_weights_follow_the_variant():
    w = shard.estimated_seconds([G, G], _hw(), ["tc_tf32", "tc_3xtf32"])
    assert w[1] == pytest.approx(3 * w[0])
