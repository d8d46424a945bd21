"""Host-side execute-contract checks that need no GPU: kernel instantiation refuses what no kernel
can run (dtype_bytes other than 4 / 2) and a schedule constructed for another operator (the
schedule's tiles index its own op's axes, etir.hpp:75), before any device work."""
import json

import pytest

g = pytest.importorskip("paper_2502_11407_b200")

B200_LIKE = {"name": "b200-nominal", "peak_flops": 7.2e13, "clock_hz": 1.9e9,
             "levels": [{"name": "hbm3e", "capacity_bytes": "unlimited", "bandwidth_bytes_per_cycle": 4210,
                         "latency_cycles": 800, "bank_width_elems": 0},
                        {"name": "smem", "capacity_bytes": 232448, "bandwidth_bytes_per_cycle": 18944,
                         "latency_cycles": 30, "bank_width_elems": 32},
                        {"name": "regs", "capacity_bytes": 1020, "bandwidth_bytes_per_cycle": 227328,
                         "latency_cycles": 1, "bank_width_elems": 0}]}


def _sched(doc):
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    hw = g.HardwareSpec.load_text(json.dumps(B200_LIKE))
    return op, g.optimize(op, hw, g.EngineConfig(top_k=1))


@pytest.mark.parametrize("dt", [1, 3, 8])
def test_prepare_rejects_unsupported_dtype(dt):
    op, s = _sched({"kind": "gemm", "M": 64, "K": 64, "N": 64, "dtype_bytes": dt})
    for variant in ("auto", "simt_f32", "simt_parity"):
        with pytest.raises(g.GensorError) as e:
            g.Kernel(op, s, 0, variant)
        assert e.value.code == "Unsupported" and "dtype_bytes" in str(e.value)


def test_prepare_rejects_schedule_of_another_op():
    op_a, s_a = _sched({"kind": "gemm", "M": 64, "K": 64, "N": 64})
    op_b = g.TensorOpSpec.parse_text(json.dumps({"kind": "conv2d", "I": [1, 8, 10, 10], "K": [8, 8, 3, 3], "S": 1}))
    with pytest.raises(g.GensorError) as e:
        g.Kernel(op_b, s_a, 0, "simt_f32")
    assert e.value.code == "ShapeMismatch"
    # a different handle describing the same operator is the same op: accepted up to device work
    op_a2 = g.TensorOpSpec.parse_text(json.dumps({"kind": "gemm", "M": 64, "K": 64, "N": 64}))
    try:
        g.Kernel(op_a2, s_a, 0, "simt_f32")
    except g.GensorError as e2:  # no GPU here: the device query fails after the op check passed
        assert e2.code == "Cuda"


def test_execute_ws_exported():
    lib = g.gensor.lib() if hasattr(g, "gensor") else None
    from paper_2502_11407_b200 import gensor as G

    for name in ("gensor_execute_ws", "gensor_kernel_workspace_size"):
        assert hasattr(G.lib(), name)
