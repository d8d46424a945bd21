"""Generates tests/golden/*.json from the REFERENCE itself (oracle/_ref/libgensor_ref.so, the
unmodified reference construct library compiled by oracle/Makefile). Run here, where
/root/reference exists; the fixtures are committed so the CPU tests pin parity on any box.

  python tools/make_golden.py [--markov-only]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import CONFIG_OPS, PROFILES  # noqa: E402
from oracle import ref  # noqa: E402

EXTRA_OPS = {
    "gemm64": {"kind": "gemm", "M": 64, "K": 64, "N": 64},
    "gemm_ragged": {"kind": "gemm", "M": 100, "K": 37, "N": 3},
    "gemv16x8": {"kind": "gemv", "M": 16, "N": 8},
    "conv_C1": {"kind": "conv2d", "I": [128, 256, 30, 30], "K": [256, 256, 3, 3], "S": 2},
    "conv_flat": {"kind": "conv2d", "N": 2, "C": 3, "H": 9, "W": 7, "F": 4, "R": 3, "S": 2, "stride": 2},
    "pool_flat": {"kind": "avgpool2d", "N": 1, "C": 2, "H": 8, "W": 8, "F": 2, "stride": 2},
    "unit": {"kind": "gemm", "M": 1, "K": 1, "N": 1},
}


# Chain-analysis cases (markov.cpp): small enumerable spaces, incl. a 2-level (L=1) profile.
TWO_LEVEL = dict(PROFILES["generic"], name="generic-2level", levels=PROFILES["generic"]["levels"][:2])
MARKOV_CASES = [
    ("generic", {"kind": "gemv", "M": 4, "N": 2}, {}),
    ("generic", {"kind": "gemv", "M": 4, "N": 2}, {"enable_inv_tile": False, "stationary_levels": []}),
    ("two_level", {"kind": "gemm", "M": 4, "K": 4, "N": 4}, {}),
    ("two_level", {"kind": "gemv", "M": 16, "N": 8}, {"fixed_iteration": 0}),
    ("b200_ref", {"kind": "avgpool2d", "I": [1, 1, 5, 5], "F": 2, "S": 1}, {"vthread_options": [1, 2]}),
]


def markov():
    profiles = dict(PROFILES, two_level=TWO_LEVEL)
    out = {"generator": "tools/make_golden.py over oracle/_ref markov.cpp (reference, unmodified)",
           "profiles": profiles, "cases": []}
    for pname, op, caps in MARKOV_CASES:
        r = ref.analyze(op, profiles[pname], dict({"stationary_levels": [0]}, **caps))
        assert "error" not in r, r
        out["cases"].append({"profile": pname, "op": op, "caps": caps, "ref": r})
    path = os.path.join(ROOT, "tests", "golden", "markov_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


def main():
    if not ref.available():
        sys.exit("oracle/_ref not built: make -C oracle ref")
    markov()
    if "--markov-only" in sys.argv:
        return
    ops = dict(CONFIG_OPS)
    ops.update(EXTRA_OPS)
    out = {"generator": "tools/make_golden.py over oracle/_ref (reference proj/src, unmodified)",
           "profiles": PROFILES, "ops": ops, "optimize": [], "construct": [], "tree": [], "state_eval": []}
    for pname, hw in PROFILES.items():
        for oname, op in ops.items():
            for seed in (0, 1, 7):
                r = ref.optimize(op, hw, {"seed": seed})
                r.pop("wall_s", None)
                out["optimize"].append({"profile": pname, "op": oname, "cfg": {"seed": seed}, "results": r["results"]})
            # non-default configs exercise vthread options, factors, restarts, top_k, t0
            cfg = {"seed": 3, "restarts": 3, "top_k": 4, "vthread_options": [8, 2, 2, 1], "max_tile_factor": 4,
                   "t0": 4096.0}
            r = ref.optimize(op, hw, cfg)
            r.pop("wall_s", None)
            out["optimize"].append({"profile": pname, "op": oname, "cfg": cfg, "results": r["results"]})
            c = ref.construct(op, hw, {"seed": 11})
            out["construct"].append({"profile": pname, "op": oname, "cfg": {"seed": 11}, **c})
            t = ref.tree(op, hw, 4)
            out["tree"].append({"profile": pname, "op": oname, "beam": 4, "results": t["results"]})
            # cost-model quantities along the best trace
            best = out["optimize"][-2]["results"][0]["trace"] if out["optimize"][-2]["results"] else []
            for cut in sorted({0, len(best) // 3, len(best) // 2, len(best)}):
                ev = ref.state_eval(op, hw, best[:cut])
                out["state_eval"].append({"profile": pname, "op": oname, "trace": best[:cut], "eval": ev})
    path = os.path.join(ROOT, "tests", "golden", "construct_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
