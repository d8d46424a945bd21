"""End-to-end operator sequences (BASELINE configs[4]): shapes, sharding and construction.

The sequences are lists of reference op specs (paper_2502_11407_b200/sequences.py); this checks
that every op parses, that batch sharding over 1/2/4/8 GPUs splits the global batch exactly, and
that the B200-mode engine constructs every distinct op (construction time under the SPEC's
5 s per op bound) — on CPU, with a device model written as a document."""
import json
import time

import pytest

g = pytest.importorskip("paper_2502_11407_b200")
from paper_2502_11407_b200 import sequences as S  # noqa: E402

# B200 device model as a document (HwModel::to_json round trip), so no GPU is needed.
B200_DOC = {
    "name": "b200", "peak_flops": 74.4e12, "clock_hz": 1.965e9,
    "levels": [
        {"name": "hbm3e", "capacity_bytes": "unlimited", "bandwidth_bytes_per_cycle": 6537e9 / 1.965e9,
         "latency_cycles": 800, "bank_width_elems": 0},
        {"name": "smem", "capacity_bytes": 232448, "bandwidth_bytes_per_cycle": 128 * 148, "latency_cycles": 30,
         "bank_width_elems": 32},
        {"name": "regs", "capacity_bytes": 1020, "bandwidth_bytes_per_cycle": 4 * 32 * 3 * 4 * 148,
         "latency_cycles": 1, "bank_width_elems": 0},
    ],
    "b200": {"sms": 148},
}


def test_resnet50_shapes():
    seq = S.resnet50(128)
    convs = [s for n, s in seq if s["kind"] == "conv2d"]
    assert len(convs) == 53
    flops = sum(g.TensorOpSpec.parse_text(json.dumps(s)).flops for _, s in seq)
    assert 1.0e12 < flops < 1.1e12  # ~4.1 GMAC per 224x224 image x 128 images x 2
    # every "same" conv keeps the ResNet spatial plan: 112 -> 56 -> 28 -> 14 -> 7
    outs = {g.TensorOpSpec.parse_text(json.dumps(s)).axes[2]["extent"] for s in convs}
    assert outs == {112, 56, 28, 14, 7}


def test_gpt2_shapes():
    seq = S.gpt2(16)
    assert len(seq) == 12 * 7 + 1
    qk = dict(seq)["h0.qk"]
    assert qk["batch"] == 192 and (qk["M"], qk["K"], qk["N"]) == (512, 64, 512)  # configs[2] shape


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["resnet50", "gpt2"])
def test_sharding_splits_the_batch(name, world):
    full = S.sharded(name, 1)
    shard = S.sharded(name, world)
    assert len(full) == len(shard)
    f_full = sum(g.TensorOpSpec.parse_text(json.dumps(s)).flops for _, s in full)
    f_shard = sum(g.TensorOpSpec.parse_text(json.dumps(s)).flops for _, s in shard)
    assert abs(f_full - world * f_shard) <= 1e-9 * f_full


@pytest.mark.parametrize("name", ["resnet50", "gpt2"])
def test_every_op_constructs_in_b200_mode(name):
    hw = g.HardwareSpec.load_text(json.dumps(B200_DOC))
    for spec in S.distinct(S.sharded(name, 1)).values():
        op = g.TensorOpSpec.parse_text(json.dumps(spec))
        t0 = time.perf_counter()
        res = g.optimize(op, hw, g.EngineConfig(mode="b200", top_k=1))
        assert time.perf_counter() - t0 < 5.0
        assert res[0]["state"]["level"] == len(res[0]["state"]["tiles"][0])  # complete schedule


def test_uneven_sharding_rejected():
    with pytest.raises(ValueError):
        S.sharded("gpt2", 3)
