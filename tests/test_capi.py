"""The C-ABI library: loads without a GPU, exports every symbol include/gensor_b200.h declares,
and reports the reference's error codes/messages (error.hpp:8-40) for bad input."""
import ctypes
import json
import os
import re

import pytest

from conftest import GENERIC, ROOT

g = pytest.importorskip("paper_2502_11407_b200")
from paper_2502_11407_b200 import gensor as G  # noqa: E402

HEADER = os.path.join(ROOT, "include", "gensor_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gensor_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(G.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(G.EXPORTED) == names


def test_only_capi_symbols_exported():
    out = os.popen(f"nm -D --defined-only {G.LIB_PATH}").read().split("\n")
    syms = [l.split()[-1] for l in out if l.strip()]
    assert syms and all(s.startswith("gensor_") for s in syms), [s for s in syms if not s.startswith("gensor_")][:5]


def test_version():
    assert "sm_100a" in G.lib().gensor_version().decode()


@pytest.mark.parametrize(
    "doc,code",
    [
        ('{"kind":"gemm","M":4,"K":4}', "MissingParam"),
        ('{"M":4}', "MissingParam"),
        ('{"kind":"gemm","M":0,"K":4,"N":4}', "NonPositiveExtent"),
        ('{"kind":"gemm","M":4.0,"K":4,"N":4}', "MissingParam"),
        ('{"kind":"fft","M":4}', "UnknownKind"),
        ('{"kind":"conv2d","I":[1,3,8,8],"K":[4,2,3,3]}', "ConfigError"),
        ('{"kind":"conv2d","I":[1,3,2,8],"K":[4,3,3,3]}', "NonPositiveExtent"),
        ('{"kind":"conv2d","I":[1,3,8],"K":[4,3,3,3]}', "MissingParam"),
        ('{"kind":"gemm",', "ConfigError"),
        ('{"kind":"gemm","M":4,"K":4,"N":4,"dtype_bytes":0}', "NonPositiveExtent"),
    ],
)
def test_op_parse_errors(doc, code):
    with pytest.raises(g.GensorError) as e:
        g.TensorOpSpec.parse_text(doc)
    assert e.value.code == code
    assert str(e.value).startswith(code + ":")


def _hw(**over):
    d = json.loads(json.dumps(GENERIC))
    d.update(over)
    return json.dumps(d)


@pytest.mark.parametrize(
    "mut,code",
    [
        (lambda d: d.update(levels=[]), "MissingLevel"),
        (lambda d: d["levels"][1].update(capacity_bytes="unlimited"), "MonotonicityViolation"),
        (lambda d: d["levels"][2].update(capacity_bytes=10 ** 9), "MonotonicityViolation"),
        (lambda d: d["levels"][1].update(bandwidth_bytes_per_cycle=8), "MonotonicityViolation"),
        (lambda d: d["levels"][1].update(bandwidth_bytes_per_cycle=0), "ConfigError"),
        (lambda d: d["levels"][1].pop("capacity_bytes"), "ConfigError"),
        (lambda d: d["levels"][1].update(capacity_bytes="lots"), "ConfigError"),
        (lambda d: d.update(vthread_options=[3]), "ConfigError"),
        (lambda d: d.update(peak_flops=0), "ConfigError"),
    ],
)
def test_hw_load_errors(mut, code):
    d = json.loads(json.dumps(GENERIC))
    mut(d)
    with pytest.raises(g.GensorError) as e:
        g.HardwareSpec.load_text(json.dumps(d))
    assert e.value.code == code


def test_hw_roundtrip():  # SPEC hardware-model invariant: load -> serialize -> reload identical
    hw = g.HardwareSpec.load_text(json.dumps(GENERIC))
    j = hw.to_json()
    assert g.HardwareSpec.load_text(json.dumps(j)).to_json() == j
    single = {"levels": [{"name": "global", "capacity_bytes": "unlimited", "bandwidth_bytes_per_cycle": 8}]}
    hw1 = g.HardwareSpec.load_text(json.dumps(single))
    assert hw1.to_json()["name"] == "unnamed"


def test_engine_config_errors():
    op = g.TensorOpSpec.parse_text('{"kind":"gemm","M":8,"K":8,"N":8}')
    hw = g.HardwareSpec.load_text(json.dumps(GENERIC))
    for bad in (dict(t0=1.0), dict(restarts=0), dict(top_k=0), dict(max_tile_factor=3), dict(vthread_options=[5])):
        with pytest.raises(g.GensorError) as e:
            g.optimize(op, hw, g.EngineConfig(**bad))
        assert e.value.code == "ConfigError"


def test_illegal_trace_rejected():
    op = g.TensorOpSpec.parse_text('{"kind":"gemm","M":8,"K":8,"N":8}')
    hw = g.HardwareSpec.load_text(json.dumps(GENERIC))
    with pytest.raises(g.GensorError) as e:
        g.from_trace(op, hw, [[1, 0, 2]])  # InvTile at the padded extent
    assert e.value.code == "IllegalAction"
    with pytest.raises(g.GensorError) as e:
        g.from_trace(op, hw, [[0, 7, 2]])
    assert e.value.code == "AxisNotFound"
    with pytest.raises(g.GensorError) as e:
        g.estimate_cost(op, hw, [[0, 0, 2]])
    assert e.value.code == "IncompleteState"


def test_kernel_prepare_needs_complete_state():
    op = g.TensorOpSpec.parse_text('{"kind":"gemm","M":8,"K":8,"N":8}')
    hw = g.HardwareSpec.load_text(json.dumps(GENERIC))
    s = g.from_trace(op, hw, [[0, 0, 2]])
    with pytest.raises(g.GensorError) as e:
        g.Kernel(op, s, 0, "simt_parity")
    assert e.value.code == "IncompleteState"


def test_op_info_layout_coefficients():
    """Affine layouts = the reference's row-major tensor_offset on the true domain (op_spec.cpp:251-262)."""
    op = g.TensorOpSpec.parse_text('{"kind":"conv2d","I":[2,3,9,7],"K":[4,3,3,2],"S":2}')
    I, K, O = op.tensors
    assert I["true_dims"] == [2, 3, 9, 7] and K["true_dims"] == [4, 3, 3, 2] and O["true_dims"] == [2, 4, 4, 3]
    # axes n f h w c r s; I offset = ((n*3+c)*9 + 2h+r)*7 + 2w+s
    assert I["coef"] == [189, 0, 14, 2, 63, 7, 1]
    assert K["coef"] == [0, 18, 0, 0, 6, 2, 1]
    assert O["coef"] == [48, 12, 3, 1, 0, 0, 0]
