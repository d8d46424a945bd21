"""TEST INFRASTRUCTURE ONLY: numpy-facing wrapper of the C execute oracle (gensor_oracle.c).

The reference's executor is absent (lowering.cpp, proj/src/CMakeLists.txt:10); the C file
restates reference_compute and interpret(lower(state)) from SPEC.md:459-521. Checker only:
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "liboracle.so")

KINDS = {"gemm": 0, "gemv": 1, "conv2d": 2, "avgpool2d": 3, "dwconv2d": 4, "softmax": 5}


class OracleOp(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad_", ctypes.c_int32)] + [
        (n, ctypes.c_int64) for n in ("M", "K", "N", "n", "c", "h", "w", "f", "r", "s", "stride", "batch")
    ]


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        FP = ctypes.POINTER(ctypes.c_float)
        DP = ctypes.POINTER(ctypes.c_double)
        L.oracle_reference_compute.argtypes = [ctypes.POINTER(OracleOp), FP, FP, DP, ctypes.c_int]
        L.oracle_reference_compute.restype = ctypes.c_int
        L.oracle_interpret.argtypes = [ctypes.POINTER(OracleOp), ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_int64), FP, FP, DP, ctypes.c_int]
        L.oracle_interpret.restype = ctypes.c_int
        L.oracle_out_elems.argtypes = [ctypes.POINTER(OracleOp)]
        L.oracle_out_elems.restype = ctypes.c_int64
        _lib = L
    return _lib


def make_op(doc) -> OracleOp:
    """Reference op JSON (op_spec.cpp:70-131 forms) -> oracle struct."""
    d = json.loads(doc) if isinstance(doc, str) else dict(doc)
    o = OracleOp()
    o.kind = KINDS[d["kind"]]
    o.stride, o.batch = 1, 1
    k = d["kind"]
    if k == "gemm":
        o.M, o.K, o.N, o.batch = d["M"], d["K"], d["N"], d.get("batch", 1)
    elif k in ("gemv", "softmax"):
        o.M, o.N = d["M"], d["N"]
    elif k == "conv2d":
        if "I" in d:
            o.n, o.c, o.h, o.w = d["I"]
            o.f, _, o.r, o.s = d["K"]
            o.stride = d.get("S", 1)
        else:
            o.n, o.c, o.h, o.w, o.f, o.r, o.s = (d[x] for x in "NCHWFRS")
            o.stride = d.get("stride", 1)
    elif k == "dwconv2d":
        if "I" in d:
            o.n, o.c, o.h, o.w = d["I"]
            _, _, o.r, o.s = d["K"]
            o.stride = d.get("S", 1)
        else:
            o.n, o.c, o.h, o.w, o.r, o.s = (d[x] for x in "NCHWRS")
            o.stride = d.get("stride", 1)
    elif k == "avgpool2d":
        if "I" in d:
            o.n, o.c, o.h, o.w = d["I"]
            o.r = o.s = d["F"]
            o.stride = d.get("S", 1)
        else:
            o.n, o.c, o.h, o.w = d["N"], d["C"], d["H"], d["W"]
            o.r = o.s = d["F"]
            o.stride = d.get("stride", 1)
    return o


def _fp(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _prep(inputs):
    return [np.ascontiguousarray(x, dtype=np.float32) for x in inputs] + [None] * (2 - len(inputs))


def reference_compute(op_doc, inputs, threads: int = 1) -> np.ndarray:
    o = make_op(op_doc)
    xs = _prep(inputs)
    out = np.zeros(lib().oracle_out_elems(ctypes.byref(o)), dtype=np.float64)
    rc = lib().oracle_reference_compute(ctypes.byref(o), _fp(xs[0]), _fp(xs[1]),
                                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), threads)
    if rc:
        raise ValueError("oracle rejected op")
    return out


def interpret(op_doc, state: dict, inputs, threads: int = 1) -> np.ndarray:
    """state: {'tiles': [[T1..TL] per axis], 'vthreads': [...]} as the engine reports it."""
    o = make_op(op_doc)
    xs = _prep(inputs)
    tiles = state["tiles"]
    L = len(tiles[0]) if tiles else 0
    t = np.ascontiguousarray(np.array(tiles, dtype=np.int64).reshape(-1))
    v = np.ascontiguousarray(np.array(state["vthreads"], dtype=np.int64))
    out = np.zeros(lib().oracle_out_elems(ctypes.byref(o)), dtype=np.float64)
    rc = lib().oracle_interpret(ctypes.byref(o), L, t.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                v.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _fp(xs[0]), _fp(xs[1]),
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), threads)
    if rc:
        raise ValueError("oracle rejected op/state")
    return out
