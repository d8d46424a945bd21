"""Python mirror of the reference's construct -> execute interface, over the gensor-b200 C-ABI.

The reference exposes a C++ API (include/gensor/*.hpp) and its (absent) pybind module `_core`
(src/CMakeLists.txt:18-30). This module keeps the reference's names and argument meaning —
``TensorOpSpec.parse_text``, ``HardwareSpec.load_text``, ``EngineConfig``, ``optimize``,
``construct``, ``construct_tree``, ``estimate_cost`` — and adds the execute half the reference
only specifies: ``Kernel(op, schedule, variant).execute(...)``.

Everything runs inside ``lib/libgensor_b200.so`` (C++ host engine + sm_100a kernels). There is
no Python or CPU fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from typing import Any, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libgensor_b200.so")

ERROR_NAMES = [
    "UnknownKind", "MissingParam", "NonPositiveExtent", "AxisNotFound", "IllegalAction",
    "LevelOutOfRange", "MonotonicityViolation", "MissingLevel", "IncompleteState",
    "TooLargeToEnumerate", "NoLegalAction", "EmptyCandidates", "SpaceTooLarge", "NotErgodic",
    "NoConvergence", "ShapeMismatch", "ReplayMismatch", "ConfigError", "Cuda", "Unsupported",
    "Invalid", "Truncated",
]

VARIANTS = {"auto": -1, "simt_parity": 0, "simt_f32": 1, "tc_tf32": 2, "tc_bf16": 3, "stream": 4, "tc_3xtf32": 5}
MODES = {"reference": 0, "b200": 1}
ACTION_KINDS = ["tile", "inv_tile", "set_vthread", "cache"]


class GensorError(RuntimeError):
    """Carries the reference's ErrorCode name (include/gensor/error.hpp:8-27) as ``code``."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERROR_NAMES[status - 1] if 0 < status <= len(ERROR_NAMES) else "Error"
        super().__init__(message or self.code)


class _CfgStruct(ctypes.Structure):
    _fields_ = [
        ("t0", ctypes.c_double),
        ("threshold", ctypes.c_double),
        ("restarts", ctypes.c_int32),
        ("top_k", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("vthread_options", ctypes.c_int64 * 8),
        ("n_vthread_options", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("max_tile_factor", ctypes.c_int64),
        ("threads", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"gensor-b200 native library not built: {LIB_PATH} (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, D, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_char_p
    PP = ctypes.POINTER(ctypes.c_void_p)
    IP = ctypes.POINTER(ctypes.c_int)
    SZ = ctypes.c_size_t
    SZP = ctypes.POINTER(ctypes.c_size_t)
    sig = {
        "gensor_last_error": (S, []),
        "gensor_version": (S, []),
        "gensor_engine_cfg_init": (None, [ctypes.POINTER(_CfgStruct)]),
        "gensor_op_parse": (I, [S, PP]),
        "gensor_op_free": (None, [P]),
        "gensor_op_info": (I, [P, ctypes.c_char_p, SZ, SZP]),
        "gensor_hw_load": (I, [S, PP]),
        "gensor_hw_b200": (I, [I, S, PP]),
        "gensor_hw_free": (None, [P]),
        "gensor_hw_json": (I, [P, ctypes.c_char_p, SZ, SZP]),
        "gensor_optimize": (I, [P, P, ctypes.POINTER(_CfgStruct), PP, IP]),
        "gensor_construct": (I, [P, P, ctypes.POINTER(_CfgStruct), PP, IP]),
        "gensor_construct_tree": (I, [P, P, I, I, PP, IP]),
        "gensor_schedule_from_trace": (I, [P, P, S, I, PP]),
        "gensor_schedule_json": (I, [P, I, ctypes.c_char_p, SZ, SZP]),
        "gensor_schedule_count": (I, [P]),
        "gensor_schedule_free": (None, [P]),
        "gensor_state_eval": (I, [P, P, S, I, ctypes.c_char_p, SZ, SZP]),
        "gensor_candidates": (I, [P, P, S, ctypes.POINTER(_CfgStruct), I, ctypes.c_char_p, SZ, SZP]),
        "gensor_caching_benefit": (D, [D, D, D, D, D]),
        "gensor_vthread_conflict_ratio": (D, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]),
        "gensor_anneal_cache_multiplier": (D, [I]),
        "gensor_record_probability": (D, [D]),
        "gensor_derive_seed": (ctypes.c_uint64, [ctypes.c_uint64, I]),
        "gensor_kernel_prepare": (I, [P, P, I, I, PP]),
        "gensor_kernel_info": (I, [P, ctypes.c_char_p, SZ, SZP]),
        "gensor_execute": (I, [P, PP, I, P, P]),
        "gensor_execute_host": (I, [P, PP, I, P, P]),
        "gensor_kernel_workspace_size": (I, [P, SZP]),
        "gensor_execute_ws": (I, [P, PP, I, P, P, SZ, P]),
        "gensor_kernel_free": (None, [P]),
        "gensor_launch_count": (ctypes.c_uint64, []),
        "gensor_kernel_set_timing": (I, [P, I]),
        "gensor_kernel_timings": (I, [P, ctypes.POINTER(ctypes.c_float), I, IP, ctypes.c_char_p, SZ]),
        "gensor_rerank": (I, [P, P, I, PP, I, P, P, I, ctypes.c_char_p, SZ, SZP]),
        "gensor_emit_source": (I, [P, I, ctypes.c_char_p, SZ, SZP]),
        "gensor_analyze": (I, [P, P, S, ctypes.c_char_p, SZ, SZP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
EXPORTED = [
    "gensor_last_error", "gensor_version", "gensor_engine_cfg_init", "gensor_op_parse", "gensor_op_free",
    "gensor_op_info", "gensor_hw_load", "gensor_hw_b200", "gensor_hw_free", "gensor_hw_json",
    "gensor_optimize", "gensor_construct", "gensor_construct_tree", "gensor_schedule_from_trace",
    "gensor_schedule_json", "gensor_schedule_count", "gensor_schedule_free", "gensor_state_eval",
    "gensor_candidates", "gensor_caching_benefit", "gensor_vthread_conflict_ratio",
    "gensor_anneal_cache_multiplier", "gensor_record_probability", "gensor_derive_seed",
    "gensor_kernel_prepare", "gensor_kernel_info", "gensor_execute", "gensor_execute_host",
    "gensor_kernel_workspace_size", "gensor_execute_ws",
    "gensor_kernel_free", "gensor_launch_count", "gensor_kernel_set_timing", "gensor_kernel_timings",
    "gensor_rerank", "gensor_emit_source", "gensor_analyze",
]


def lib() -> ctypes.CDLL:
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise GensorError(status, _lib.gensor_last_error().decode())


def _text_call(fn, *args) -> str:
    need = ctypes.c_size_t(0)
    buf = ctypes.create_string_buffer(1 << 16)
    st = fn(*args, buf, len(buf), ctypes.byref(need))
    if st == 22:  # truncated: retry with the exact size
        buf = ctypes.create_string_buffer(need.value)
        st = fn(*args, buf, len(buf), ctypes.byref(need))
    _check(st)
    return buf.value.decode()


def _json_call(fn, *args) -> Any:
    return json.loads(_text_call(fn, *args))


def _text(doc: Any) -> bytes:
    return (doc if isinstance(doc, str) else json.dumps(doc)).encode()


class TensorOpSpec:
    """Operator description (reference: TensorOpSpec, op_spec.hpp:48-116)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)
        self.info = _json_call(_lib.gensor_op_info, self._h)

    @staticmethod
    def parse_text(text: str) -> "TensorOpSpec":
        h = ctypes.c_void_p()
        _check(_lib.gensor_op_parse(_text(text), ctypes.byref(h)))
        return TensorOpSpec(h.value)

    parse = parse_text

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.gensor_op_free(self._h)
            self._h = None

    @property
    def kind(self) -> str:
        return self.info["kind"]

    @property
    def axes(self):
        return [dict(name=a[0], extent=a[1], padded=a[2], reduce=a[3]) for a in self.info["axes"]]

    @property
    def tensors(self):
        return self.info["tensors"]

    def axis_index(self, name: str) -> int:
        for i, a in enumerate(self.info["axes"]):
            if a[0] == name:
                return i
        raise GensorError(4, f"AxisNotFound: no axis '{name}' in {self.info['label']}")

    @property
    def flops(self) -> float:
        return self.info["flops"]

    @property
    def bytes(self) -> float:
        return self.info["bytes"]

    @property
    def dtype_bytes(self) -> int:
        return self.info["dtype_bytes"]

    @property
    def batch(self) -> int:
        return self.info["batch"]

    def to_json(self) -> dict:
        return self.info["json"]

    def label(self) -> str:
        return self.info["label"]


class HardwareSpec:
    """Hardware model (reference: HardwareSpec, hardware.hpp:28-58), plus the B200 device model."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    @staticmethod
    def load_text(text: str) -> "HardwareSpec":
        h = ctypes.c_void_p()
        _check(_lib.gensor_hw_load(_text(text), ctypes.byref(h)))
        return HardwareSpec(h.value)

    load = load_text

    @staticmethod
    def b200(device: int = 0, measured_peaks: dict | str | None = None) -> "HardwareSpec":
        h = ctypes.c_void_p()
        peaks = None if measured_peaks is None else _text(measured_peaks)
        _check(_lib.gensor_hw_b200(device, peaks, ctypes.byref(h)))
        return HardwareSpec(h.value)

    def to_json(self) -> dict:
        return _json_call(_lib.gensor_hw_json, self._h)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.gensor_hw_free(self._h)
            self._h = None


@dataclass
class EngineConfig:
    """EngineConfig field for field (engine.hpp:14-24) + construction mode and worker threads."""

    t0: float = 1048576.0
    threshold: float = 1.0
    restarts: int = 8
    seed: int = 0
    top_k: int = 10
    vthread_options: Sequence[int] = field(default_factory=lambda: [1, 2, 4, 8])
    max_tile_factor: int = 2
    mode: str = "reference"
    threads: int = 0

    def _struct(self) -> _CfgStruct:
        c = _CfgStruct()
        _lib.gensor_engine_cfg_init(ctypes.byref(c))
        c.t0, c.threshold, c.restarts, c.top_k = self.t0, self.threshold, self.restarts, self.top_k
        c.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        opts = list(self.vthread_options)[:8]
        for i, v in enumerate(opts):
            c.vthread_options[i] = v
        c.n_vthread_options = len(opts)
        c.max_tile_factor = self.max_tile_factor
        c.mode = MODES[self.mode] if isinstance(self.mode, str) else int(self.mode)
        c.threads = self.threads
        return c


class Schedules:
    """Result list of optimize/construct/construct_tree (reference: vector<ScheduleResult>)."""

    def __init__(self, op: TensorOpSpec, hw: HardwareSpec, handle: int):
        self.op, self.hw = op, hw  # keep owners alive: the op must outlive schedules (etir.hpp:75)
        self._h = ctypes.c_void_p(handle)
        self.results = _json_call(_lib.gensor_schedule_json, self._h, -1)

    def __len__(self):
        return len(self.results)

    def emit_source(self, index: int = 0) -> str:
        """Portable C source of result `index`'s loop nest (SPEC.md:488-496 emit_source)."""
        return _text_call(_lib.gensor_emit_source, self._h, index)

    def __getitem__(self, i):
        return self.results[i]

    def __iter__(self):
        return iter(self.results)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.gensor_schedule_free(self._h)
            self._h = None


def optimize(op: TensorOpSpec, hw: HardwareSpec, cfg: EngineConfig | None = None) -> Schedules:
    cfg = cfg or EngineConfig()
    h, n = ctypes.c_void_p(), ctypes.c_int()
    c = cfg._struct()
    _check(_lib.gensor_optimize(op._h, hw._h, ctypes.byref(c), ctypes.byref(h), ctypes.byref(n)))
    return Schedules(op, hw, h.value)


def construct(op: TensorOpSpec, hw: HardwareSpec, cfg: EngineConfig | None = None) -> Schedules:
    cfg = cfg or EngineConfig()
    h, n = ctypes.c_void_p(), ctypes.c_int()
    c = cfg._struct()
    _check(_lib.gensor_construct(op._h, hw._h, ctypes.byref(c), ctypes.byref(h), ctypes.byref(n)))
    return Schedules(op, hw, h.value)


def construct_tree(op: TensorOpSpec, hw: HardwareSpec, beam_width: int = 4, mode: str = "reference") -> Schedules:
    h, n = ctypes.c_void_p(), ctypes.c_int()
    _check(_lib.gensor_construct_tree(op._h, hw._h, beam_width, MODES[mode], ctypes.byref(h), ctypes.byref(n)))
    return Schedules(op, hw, h.value)


def from_trace(op: TensorOpSpec, hw: HardwareSpec, trace, mode: str = "reference") -> Schedules:
    h = ctypes.c_void_p()
    _check(_lib.gensor_schedule_from_trace(op._h, hw._h, _text(trace), MODES[mode], ctypes.byref(h)))
    return Schedules(op, hw, h.value)


def state_eval(op: TensorOpSpec, hw: HardwareSpec, trace, mode: str = "reference") -> dict:
    return _json_call(_lib.gensor_state_eval, op._h, hw._h, _text(trace), MODES[mode])


def estimate_cost(op: TensorOpSpec, hw: HardwareSpec, trace, mode: str = "reference") -> dict:
    ev = state_eval(op, hw, trace, mode)
    if "cost" not in ev:
        raise GensorError(9, "IncompleteState: cost needs a complete schedule")
    return ev["cost"]


def enumerate_candidates(op: TensorOpSpec, hw: HardwareSpec, trace, cfg: EngineConfig | None = None,
                         iteration: int = 0) -> list:
    cfg = cfg or EngineConfig()
    c = cfg._struct()
    return _json_call(_lib.gensor_candidates, op._h, hw._h, _text(trace), ctypes.byref(c), iteration)["candidates"]


def analyze(op: TensorOpSpec, hw: HardwareSpec, caps: dict | None = None) -> dict:
    """Construction-chain analysis (markov.hpp / SPEC.md:380-457 markov-verify), see gensor_analyze."""
    return _json_call(_lib.gensor_analyze, op._h, hw._h, _text(caps or {}))


def caching_benefit(lat_low, bw_low, lat_high, bw_high, s_bytes) -> float:
    return _lib.gensor_caching_benefit(lat_low, bw_low, lat_high, bw_high, s_bytes)


def vthread_conflict_ratio(x: int, bank_width: int, v: int) -> float:
    return _lib.gensor_vthread_conflict_ratio(x, bank_width, v)


def anneal_cache_multiplier(iteration: int) -> float:
    return _lib.gensor_anneal_cache_multiplier(iteration)


def record_probability(temperature: float) -> float:
    return _lib.gensor_record_probability(temperature)


def derive_seed(seed: int, restart: int) -> int:
    return _lib.gensor_derive_seed(seed, restart)


def launch_count() -> int:
    return _lib.gensor_launch_count()


def rerank(op: "TensorOpSpec", schedules: "Schedules", inputs: Sequence[Any], output: Any,
           variant: str | int = "auto", iters: int = 5, stream: Any = None) -> dict:
    """On-device re-ranking of the constructed top-k: every result of
    ``schedules`` is instantiated with ``variant`` and timed on the given device buffers.
    Returns {"ms": [...per result...], "order": [fastest first], "best": index}."""
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    ptrs = (ctypes.c_void_p * max(1, len(inputs)))(*[_ptr(t) for t in inputs])
    return _json_call(_lib.gensor_rerank, op._h, schedules._h, v, ptrs, len(inputs), ctypes.c_void_p(_ptr(output)),
                      ctypes.c_void_p(_stream(stream)), iters)


class Kernel:
    """A kernel instantiated from one constructed schedule (the SPEC's lower())."""

    def __init__(self, op: TensorOpSpec, schedules: Schedules, index: int = 0, variant: str | int = "auto"):
        self.op, self.schedules = op, schedules
        v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
        h = ctypes.c_void_p()
        _check(_lib.gensor_kernel_prepare(op._h, schedules._h, index, v, ctypes.byref(h)))
        self._h = h

    @property
    def info(self) -> dict:
        """Plan, variant, work and (after the first host-buffer execute) the copy pipeline."""
        return _json_call(_lib.gensor_kernel_info, self._h)

    @property
    def workspace_bytes(self) -> int:
        """Device workspace one execute needs (0 for families without a pre-pass)."""
        n = ctypes.c_size_t(0)
        _check(_lib.gensor_kernel_workspace_size(self._h, ctypes.byref(n)))
        return n.value

    def execute(self, inputs: Sequence[Any], output: Any, stream: Any = None, workspace: Any = None) -> None:
        """Device execute: ``inputs``/``output`` are CUDA tensors (or raw device pointers);
        asynchronous on ``stream`` (torch.cuda.Stream, raw handle, or None = current stream).
        ``workspace``: an optional caller-owned device buffer of ``workspace_bytes`` bytes
        (gensor_execute_ws); by default the handle keeps one per stream."""
        _check_tensors(self.op, inputs, output, device=True)
        ptrs = (ctypes.c_void_p * max(1, len(inputs)))(*[_ptr(t) for t in inputs])
        if workspace is None:
            _check(_lib.gensor_execute(self._h, ptrs, len(inputs), ctypes.c_void_p(_ptr(output)),
                                       ctypes.c_void_p(_stream(stream))))
        else:
            nbytes = workspace.numel() * workspace.element_size() if hasattr(workspace, "numel") else self.workspace_bytes
            _check(_lib.gensor_execute_ws(self._h, ptrs, len(inputs), ctypes.c_void_p(_ptr(output)),
                                          ctypes.c_void_p(_ptr(workspace)), nbytes, ctypes.c_void_p(_stream(stream))))

    def execute_host(self, inputs: Sequence[Any], output: Any, stream: Any = None) -> None:
        """Host-buffer execute (the interpreter's convention): copies in, runs, copies out, syncs."""
        _check_tensors(self.op, inputs, output, device=False)
        ptrs = (ctypes.c_void_p * max(1, len(inputs)))(*[_ptr(t) for t in inputs])
        _check(_lib.gensor_execute_host(self._h, ptrs, len(inputs), ctypes.c_void_p(_ptr(output)),
                                        ctypes.c_void_p(_stream(stream))))

    def set_timing(self, on: bool = True) -> None:
        _check(_lib.gensor_kernel_set_timing(self._h, 1 if on else 0))

    def timings(self) -> list:
        """[(launch name, ms)] of the last execute (CUDA events on the execute stream)."""
        ms = (ctypes.c_float * 8)()
        n = ctypes.c_int(0)
        names = ctypes.create_string_buffer(4096)
        _check(_lib.gensor_kernel_timings(self._h, ms, 8, ctypes.byref(n), names, len(names)))
        return list(zip(json.loads(names.value.decode() or "[]"), list(ms)[: n.value]))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.gensor_kernel_free(self._h)
            self._h = None


def _tensor_elems(op: "TensorOpSpec", i: int) -> int:
    n = 1
    for d in op.tensors[i]["true_dims"]:
        n *= d
    return n * op.batch


def _check_tensors(op: "TensorOpSpec", inputs: Sequence[Any], output: Any, device: bool) -> None:
    """Argument checks of the Python mirror: tensor arguments must match the op's tensors in
    element count, dtype (fp32 for dtype_bytes 4, bf16 for 2), contiguity and device. Raw integer
    pointers pass through unchecked (explicit pointer use)."""
    want = {4: ("float32",), 2: ("bfloat16",)}.get(op.dtype_bytes, ())
    args = list(inputs) + [output]
    if len(inputs) != len(op.tensors) - 1:
        return  # the library reports ShapeMismatch
    for i, t in enumerate(args):
        if isinstance(t, int):
            continue
        name = op.tensors[i].get("name", str(i)) if isinstance(op.tensors[i], dict) else str(i)
        if hasattr(t, "is_cuda"):  # torch tensor
            if t.is_cuda != device:
                raise ValueError(f"tensor {name}: expected a {'CUDA' if device else 'host'} tensor")
            if not t.is_contiguous():
                raise ValueError(f"tensor {name}: must be contiguous")
            dt = str(t.dtype).replace("torch.", "")
        elif hasattr(t, "ctypes"):  # numpy array (host buffers only)
            if device:
                raise ValueError(f"tensor {name}: a numpy array is a host buffer; execute needs device memory")
            if not t.flags["C_CONTIGUOUS"]:
                raise ValueError(f"tensor {name}: must be C-contiguous")
            dt = "bfloat16" if (t.dtype.itemsize == 2 and op.dtype_bytes == 2) else str(t.dtype)
        else:
            continue
        if want and dt not in want:
            raise ValueError(f"tensor {name}: dtype {dt}, the op stores {want[0]} (dtype_bytes {op.dtype_bytes})")
        n = t.numel() if hasattr(t, "numel") else t.size
        need = _tensor_elems(op, i)
        if n < need:
            raise ValueError(f"tensor {name}: {n} elements, the op needs {need}")


def _ptr(t: Any) -> int:
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if hasattr(t, "ctypes"):  # numpy array (host buffers)
        return t.ctypes.data
    raise TypeError(f"cannot take a data pointer of {type(t)}")


def _stream(s: Any) -> int:
    if s is None:
        try:
            import torch

            return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0
        except ImportError:
            return 0
    if isinstance(s, int):
        return s
    return s.cuda_stream
