"""Construction-chain analysis (reference markov.cpp:40-364).

Parity: gensor_analyze(detail) against the reference's own enumerate_space / check_* /
stationary_distribution / value_iteration — via the committed golden fixture (generated from
oracle/_ref by tools/make_golden.py) and, where oracle/_ref is built, live on more cases. States
come out in the same discovery order, so the comparison is state for state and edge for edge:
probabilities, terminal values, values and stationary vectors bit-identical.
Properties: row-stochastic P, irreducible with InvTile / not without,
stationary πP = π against a direct linear solve, value-iteration payoff = the greedy path's =
the exhaustive best path's.
"""
import json
import os

import numpy as np
import pytest

from conftest import B200_REF, GENERIC, GOLDEN

g = pytest.importorskip("paper_2502_11407_b200")

TWO_LEVEL = dict(GENERIC, name="generic-2level", levels=GENERIC["levels"][:2])
PROFILES = {"generic": GENERIC, "b200_ref": B200_REF, "two_level": TWO_LEVEL}


def analyze(op, hw, caps=None):
    return g.analyze(g.TensorOpSpec.parse_text(json.dumps(op)), g.HardwareSpec.load_text(json.dumps(hw)),
                     dict(caps or {}, detail=True))


def assert_same(ours, ref):
    d = ours["detail"]
    assert d["states"] == ref["states"]
    assert d["complete"] == ref["complete"] and d["absorbing"] == ref["absorbing"]
    assert [row for row in d["rows"]] == [row for row in ref["rows"]]  # to, prob, action, artificial
    assert d["terminal"] == ref["terminal"]
    assert [l["irreducible"] for l in ours["levels"]] == ref["irreducible"]
    assert ours["aperiodic"] == ref["aperiodic"]
    assert d["value"] == ref["value"] and d["policy"] == ref["policy"]
    assert ours["value"]["iterations"] == ref["iterations"]
    for lvl, pi in ref["stationary"].items():
        assert d["stationary"][lvl] == pi


def golden_cases():
    with open(os.path.join(GOLDEN, "markov_golden.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: f"{c['profile']}-{c['op']['kind']}-{len(c['ref']['states'])}")
def test_golden_parity(case):
    caps = {k: v for k, v in case["caps"].items() if k != "stationary_levels"}
    assert_same(analyze(case["op"], PROFILES[case["profile"]], caps), case["ref"])


LIVE = [
    ("generic", {"kind": "gemm", "M": 4, "K": 4, "N": 4}, {}),
    ("b200_ref", {"kind": "gemv", "M": 16, "N": 8}, {}),
    ("generic", {"kind": "conv2d", "I": [1, 2, 4, 4], "K": [2, 2, 3, 3], "S": 1}, {"max_tile_factor": 4}),
    ("two_level", {"kind": "avgpool2d", "I": [1, 2, 6, 6], "F": 3, "S": 1}, {"fixed_iteration": 20}),
    ("two_level", {"kind": "gemm", "M": 8, "K": 2, "N": 4}, {"enable_inv_tile": False}),
]


@pytest.mark.ref
@pytest.mark.parametrize("i", range(len(LIVE)))
def test_live_parity(i):
    from oracle import ref

    pname, op, caps = LIVE[i]
    ours = analyze(op, PROFILES[pname], caps)
    levels = [int(k) for k in ours["detail"]["stationary"]]
    assert_same(ours, ref.analyze(op, PROFILES[pname], dict(caps, stationary_levels=levels)))


def test_row_stochastic_and_inv_tile_differential():
    op = {"kind": "gemm", "M": 8, "K": 4, "N": 4}
    on = analyze(op, GENERIC)
    for row in on["detail"]["rows"]:
        assert abs(sum(e[1] for e in row) - 1.0) <= 1e-9
    off = analyze(op, GENERIC, {"enable_inv_tile": False})
    assert all(l["irreducible"] for l in on["levels"])
    assert not off["levels"][0]["irreducible"]


def test_stationary_against_linear_solve():
    r = analyze({"kind": "gemm", "M": 4, "K": 4, "N": 4}, GENERIC)
    d = r["detail"]
    lvl = np.array([int(s[1]) for s in d["states"]])  # "L<level> ..."
    ids = np.flatnonzero(lvl == 0)
    local = {int(gid): k for k, gid in enumerate(ids)}
    P = np.zeros((len(ids), len(ids)))
    for gid in ids:
        row = [(local[e[0]], e[1]) for e in d["rows"][gid] if e[0] in local]
        tot = sum(p for _, p in row)
        for j, p in row:
            P[local[int(gid)], j] += p / tot
    A = np.vstack([P.T - np.eye(len(ids)), np.ones(len(ids))])
    b = np.zeros(len(ids) + 1)
    b[-1] = 1.0
    exact = np.linalg.lstsq(A, b, rcond=None)[0]
    pi = np.array(d["stationary"]["0"])[ids]
    assert abs(pi.sum() - 1) <= 1e-9 and (pi >= 0).all()
    assert np.abs(pi @ P - pi).max() <= 1e-10
    assert np.abs(pi - exact).max() <= 1e-8


def test_value_iteration_payoff_equals_bruteforce():
    r = analyze({"kind": "gemv", "M": 4, "N": 2}, TWO_LEVEL)
    d = r["detail"]
    assert r["value"]["end_payoff"] == pytest.approx(r["value"]["initial"], abs=1e-10)
    # exhaustive simple paths from the unscheduled state
    best = 0.0
    stack = [(0, 1.0, {0})]
    while stack:
        u, prod, seen = stack.pop()
        if d["complete"][u]:
            best = max(best, prod * d["terminal"][u])
            continue
        for to, p, _, art in d["rows"][u]:
            if not art and to not in seen:
                stack.append((to, prod * p, seen | {to}))
    assert best == pytest.approx(r["value"]["initial"], abs=1e-10)


def test_space_too_large():
    op = g.TensorOpSpec.parse_text(json.dumps({"kind": "gemm", "M": 64, "K": 64, "N": 64}))
    with pytest.raises(g.GensorError) as e:
        g.analyze(op, g.HardwareSpec.load_text(json.dumps(GENERIC)), {"max_states": 100})
    assert e.value.status == 13 and "SpaceTooLarge" in str(e.value)
