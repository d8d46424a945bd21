"""TEST INFRASTRUCTURE ONLY: ctypes access to the reference's own construct library.

oracle/_ref/libgensor_ref.so is the UNMODIFIED reference (/root/reference/proj/src, 8 TUs) plus
oracle/ref_capi.cpp, built by `make -C oracle ref` (needs /root/reference; this container only).
Only tests/, tools/make_golden.py, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
legs may use it — as the checker and the timed CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libgensor_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(REF_LIB)
        for name, n in (("ref_optimize", 3), ("ref_construct", 3), ("ref_state_eval", 3), ("ref_op_info", 1)):
            fn = getattr(L, name)
            fn.restype = ctypes.c_void_p
            fn.argtypes = [ctypes.c_char_p] * n
        L.ref_candidates.restype = ctypes.c_void_p
        L.ref_candidates.argtypes = [ctypes.c_char_p] * 4 + [ctypes.c_int, ctypes.c_double]
        L.ref_analyze.restype = ctypes.c_void_p
        L.ref_analyze.argtypes = [ctypes.c_char_p] * 3
        L.ref_tree.restype = ctypes.c_void_p
        L.ref_tree.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_caching_benefit.restype = ctypes.c_double
        L.ref_caching_benefit.argtypes = [ctypes.c_double] * 5
        L.ref_vthread_conflict_ratio.restype = ctypes.c_double
        L.ref_vthread_conflict_ratio.argtypes = [ctypes.c_int64] * 3
        L.ref_anneal_cache_multiplier.restype = ctypes.c_double
        L.ref_anneal_cache_multiplier.argtypes = [ctypes.c_int]
        L.ref_record_probability.restype = ctypes.c_double
        L.ref_record_probability.argtypes = [ctypes.c_double]
        L.ref_derive_seed.restype = ctypes.c_uint64
        L.ref_derive_seed.argtypes = [ctypes.c_uint64, ctypes.c_int]
        _lib = L
    return _lib


def _t(x) -> bytes:
    return (x if isinstance(x, str) else json.dumps(x)).encode()


def _call(fn, *args):
    p = fn(*args)
    try:
        return json.loads(ctypes.string_at(p).decode())
    finally:
        lib().ref_free(p)


def optimize(op, hw, cfg=None) -> dict:
    return _call(lib().ref_optimize, _t(op), _t(hw), _t(cfg or {}))


def construct(op, hw, cfg=None) -> dict:
    return _call(lib().ref_construct, _t(op), _t(hw), _t(cfg or {}))


def state_eval(op, hw, trace) -> dict:
    return _call(lib().ref_state_eval, _t(op), _t(hw), _t(trace))


def candidates(op, hw, trace, cfg=None, iteration=0, temperature=1.0) -> dict:
    return _call(lib().ref_candidates, _t(op), _t(hw), _t(trace), _t(cfg or {}), iteration, temperature)


def analyze(op, hw, caps=None) -> dict:
    return _call(lib().ref_analyze, _t(op), _t(hw), _t(caps or {}))


def tree(op, hw, beam=4) -> dict:
    return _call(lib().ref_tree, _t(op), _t(hw), beam)


def op_info(op) -> dict:
    return _call(lib().ref_op_info, _t(op))
