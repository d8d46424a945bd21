"""The gensor-b200 CLI and emit_source, on CPU.

* schedule: results.json is byte-identical across runs (acceptance 8); config
  errors exit 2 naming the field;
* verify --no-exec: every stored trace replays to its stored state; a tampered trace is a
  ReplayMismatch (exit 1);
* compare: CSV columns + geomean row, empty suite -> exit 2, failed row -> exit 1, graph never
  worse than tree analytically (acceptance 4);
* emit: deterministic text, 3 loops for the unscheduled GEMM 4^3, one guard term per padded
  axis, and — compiled with gcc and run — the emitted loop nest equals the oracle's
  reference_compute within 1e-9 relative for every schedule of both engines (acceptance 7).
"""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GENERIC, ROOT

from oracle import oracle as O

CLI = os.path.join(ROOT, "paper_2502_11407_b200", "bin", "gensor-b200")

DESK = [
    {"kind": "gemm", "M": 16, "K": 16, "N": 16},
    {"kind": "gemm", "M": 20, "K": 12, "N": 28},
    {"kind": "gemm", "M": 16, "K": 8, "N": 24, "batch": 3},
    {"kind": "gemv", "M": 40, "N": 24},
    {"kind": "conv2d", "I": [2, 3, 10, 10], "K": [4, 3, 3, 3], "S": 1},
    {"kind": "conv2d", "I": [1, 4, 11, 11], "K": [6, 4, 3, 3], "S": 2},
    {"kind": "avgpool2d", "I": [2, 3, 9, 9], "F": 3, "S": 1},
    {"kind": "avgpool2d", "I": [1, 2, 8, 8], "F": 2, "S": 2},
    {"kind": "dwconv2d", "I": [2, 5, 10, 10], "K": [5, 1, 3, 3], "S": 1},
    {"kind": "softmax", "M": 6, "N": 20},
]


def cli(*args, check=True):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=120)
    if check and p.returncode != 0:
        raise AssertionError(f"{args}: rc={p.returncode}\n{p.stdout}\n{p.stderr}")
    return p


@pytest.fixture(scope="module")
def work(tmp_path_factory):
    if not os.path.exists(CLI):
        pytest.fail(f"CLI not built: {CLI} (run __graft_entry__.build())")
    d = tmp_path_factory.mktemp("cli")
    (d / "hw.json").write_text(json.dumps(GENERIC))
    return d


def schedule(work, doc, engine="graph", tag="x"):
    out = work / tag
    out.mkdir(exist_ok=True)
    (out / "op.json").write_text(json.dumps(doc))
    cli("schedule", "--op", str(out / "op.json"), "--hw", str(work / "hw.json"), "--engine", engine, "--out", str(out))
    return out


def test_schedule_deterministic_and_both(work):
    doc = {"kind": "gemm", "M": 60, "K": 64, "N": 48}
    a = (schedule(work, doc, "both", "det1") / "results.json").read_bytes()
    b = (schedule(work, doc, "graph", "det2") / "results.json").read_bytes()
    assert a == b
    res = json.loads(a)
    assert res["engine"] == "graph" and res["op"]["M"] == 60 and len(res["results"]) >= 1
    assert (work / "det1" / "results_tree.json").exists()
    p = cli("schedule", "--op", json.dumps(doc), "--hw", str(work / "hw.json"), "--engine", "both",
            "--out", str(work / "det1"))
    assert "graph/tree" in p.stdout


def test_schedule_config_errors(work):
    p = cli("schedule", "--op", '{"kind":"gemm","M":0,"K":4,"N":4}', "--hw", str(work / "hw.json"), check=False)
    assert p.returncode == 2 and "'M'" in p.stderr
    p = cli("schedule", "--op", '{"kind":"gemm","M":4,"K":4,"N":4}', "--hw", str(work / "hw.json"),
            "--top-k", "x", check=False)
    assert p.returncode == 2 and "--top-k" in p.stderr
    p = cli("schedule", "--op", '{"kind":"gemm","M":4,"K":4,"N":4}', "--hw", '{"name":"x"}', check=False)
    assert p.returncode == 2 and "levels" in p.stderr
    assert cli("bogus", check=False).returncode == 2


def test_verify_replay_and_tamper(work):
    out = schedule(work, {"kind": "conv2d", "I": [2, 3, 10, 10], "K": [4, 3, 3, 3], "S": 1}, "graph", "ver")
    p = cli("verify", "--results", str(out / "results.json"), "--no-exec")
    assert p.stdout.strip().endswith("0 failed") and "PASS" in p.stdout
    doc = json.loads((out / "results.json").read_text())
    doc["results"][0]["trace"].insert(0, [0, 1, 2])  # an extra Tile: replays to another state
    (out / "bad.json").write_text(json.dumps(doc))
    p = cli("verify", "--results", str(out / "bad.json"), "--no-exec", check=False)
    assert p.returncode == 1 and "ReplayMismatch" in p.stdout


def test_compare_csv(work):
    suite = [{"label": f"op{i}", "op": d} for i, d in enumerate(DESK[:9])]
    (work / "suite.json").write_text(json.dumps(suite))
    p = cli("compare", "--suite", str(work / "suite.json"), "--hw", str(work / "hw.json"), "--seeds", "0,1,2,3")
    lines = p.stdout.strip().splitlines()
    assert lines[0] == "op_label,tree_cost,graph_cost,ratio,graph_wall_ms,tree_wall_ms,status"
    assert len(lines) == len(suite) + 2 and lines[-1].startswith("geomean,")
    for row in lines[1:-1]:
        f = row.split(",")
        assert f[-1] == "ok" and float(f[3]) <= 1.0 + 1e-9, row
    (work / "empty.json").write_text("[]")
    assert cli("compare", "--suite", str(work / "empty.json"), "--hw", str(work / "hw.json"),
               check=False).returncode == 2
    (work / "bad.json").write_text(json.dumps(suite[:1] + [{"label": "bad", "op": {"kind": "nope"}}]))
    p = cli("compare", "--suite", str(work / "bad.json"), "--hw", str(work / "hw.json"), check=False)
    assert p.returncode == 1 and "UnknownKind" in p.stdout and "partial" in p.stdout


def test_cost_explain(work):
    out = schedule(work, DESK[0], "graph", "cost")
    ex = json.loads(cli("cost", "explain", "--results", str(out / "results.json")).stdout)
    res = json.loads((out / "results.json").read_text())["results"][0]
    assert ex["cost"]["est_seconds"] == res["cost"]["est_seconds"]
    ex2 = json.loads(cli("cost", "explain", "--op", json.dumps(DESK[0]), "--hw", str(work / "hw.json"),
                         "--trace", json.dumps(res["trace"])).stdout)
    assert ex2 == ex


def test_emit_structure(work):
    out = schedule(work, {"kind": "gemm", "M": 4, "K": 4, "N": 4}, "graph", "e4")
    src = cli("emit", "--results", str(out / "results.json")).stdout
    assert src == cli("emit", "--results", str(out / "results.json")).stdout  # byte-identical
    loops = re.findall(r"for \(int64_t ([a-z])_[0-9sv]+ =", src)
    assert sorted(loops) == ["k", "m", "n"] and "guard" not in src
    out = schedule(work, {"kind": "gemm", "M": 60, "K": 64, "N": 48}, "graph", "e60")
    src = cli("emit", "--results", str(out / "results.json")).stdout
    guard = re.search(r"if \((.*)\)  /\* guard", src).group(1)
    assert guard == "m < 60 && n < 48"


_N = [0]


def _run_emitted(src, doc, xs, tmp):
    _N[0] += 1  # dlopen caches by path: every emitted kernel gets its own file
    c = tmp / f"k{_N[0]}.c"
    so = tmp / f"k{_N[0]}.so"
    c.write_text(src)
    subprocess.run(["gcc", "-O1", "-std=c99", "-shared", "-fPIC", str(c), "-o", str(so), "-lm"], check=True)
    lib = ctypes.CDLL(str(so))
    fn = getattr(lib, "gensor_" + doc["kind"])
    out = np.zeros(O.reference_compute(doc, xs).size, dtype=np.float64)
    args = [x.ctypes.data_as(ctypes.c_void_p) for x in xs] + [out.ctypes.data_as(ctypes.c_void_p)]
    fn.argtypes = [ctypes.c_void_p] * len(args)
    fn(*args)
    return out


@pytest.mark.parametrize("i", range(len(DESK)))
def test_emit_semantics(work, i):
    doc = DESK[i]
    rng = np.random.default_rng(i)
    op_info = None
    for engine in ("graph", "tree"):
        out = schedule(work, doc, engine, f"sem{i}{engine}")
        res = json.loads((out / ("results.json" if engine == "graph" else "results_tree.json")).read_text())
        if op_info is None:
            import paper_2502_11407_b200 as g

            op_info = g.TensorOpSpec.parse_text(json.dumps(doc))
        xs = [rng.uniform(-1, 1, int(np.prod(t["true_dims"])) * op_info.batch).astype(np.float32)
              for t in op_info.tensors[:-1]]
        ref = O.reference_compute(doc, xs)
        for j in range(len(res["results"])):
            src = cli("emit", "--results", str(out / ("results.json" if engine == "graph" else "results_tree.json")),
                      "--index", str(j)).stdout
            got = _run_emitted(src, doc, xs, out)
            err = np.abs(got - ref).max() / np.abs(ref).max()
            assert err <= 1e-9, (engine, j, err)


def test_analyze(work):
    p = cli("analyze", "--op", json.dumps({"kind": "gemm", "M": 4, "K": 4, "N": 4}), "--hw", str(work / "hw.json"))
    r = json.loads(p.stdout)
    assert r["states"] == 1308 and all(l["irreducible"] for l in r["levels"])
    assert r["value"]["end_payoff"] == pytest.approx(r["value"]["initial"], abs=1e-10)
    p = cli("analyze", "--op", json.dumps({"kind": "gemm", "M": 4, "K": 4, "N": 4}), "--hw", str(work / "hw.json"),
            "--no-inv-tile")
    assert not json.loads(p.stdout)["levels"][0]["irreducible"]
    p = cli("analyze", "--op", json.dumps({"kind": "gemm", "M": 64, "K": 64, "N": 64}), "--hw", str(work / "hw.json"),
            "--max-states", "1000", check=False)
    assert p.returncode == 3 and "SpaceTooLarge" in p.stderr
