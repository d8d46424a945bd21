import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "ref: needs the reference construct library oracle/_ref (built here)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    from oracle import ref as _ref

    for item in items:
        if "gpu" in item.keywords and not has_gpu:
            item.add_marker(pytest.mark.skip(reason="no CUDA device"))
        if "ref" in item.keywords and not _ref.available():
            item.add_marker(pytest.mark.skip(reason="oracle/_ref not built (needs /root/reference)"))


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# Hardware profiles. GENERIC is the SPEC's 3-level generic-GPU profile (with the
# survey's bandwidths); B200_REF is SURVEY.md Appendix A, the B200 in the reference's own format.
GENERIC = {
    "name": "generic", "peak_flops": 1e13, "clock_hz": 1.5e9,
    "levels": [
        {"name": "global", "capacity_bytes": "unlimited", "bandwidth_bytes_per_cycle": 32, "latency_cycles": 400,
         "bank_width_elems": 0},
        {"name": "shared", "capacity_bytes": 49152, "bandwidth_bytes_per_cycle": 128, "latency_cycles": 30,
         "bank_width_elems": 32},
        {"name": "regs", "capacity_bytes": 1024, "bandwidth_bytes_per_cycle": 512, "latency_cycles": 1,
         "bank_width_elems": 0},
    ],
}
B200_REF = {
    "name": "b200-nominal", "peak_flops": 7.2e13, "clock_hz": 1.9e9,
    "levels": [
        {"name": "hbm3e", "capacity_bytes": "unlimited", "bandwidth_bytes_per_cycle": 4210, "latency_cycles": 800,
         "bank_width_elems": 0},
        {"name": "smem", "capacity_bytes": 232448, "bandwidth_bytes_per_cycle": 18944, "latency_cycles": 30,
         "bank_width_elems": 32},
        {"name": "regs", "capacity_bytes": 1020, "bandwidth_bytes_per_cycle": 227328, "latency_cycles": 1,
         "bank_width_elems": 0},
    ],
}
PROFILES = {"generic": GENERIC, "b200_ref": B200_REF}

# BASELINE.json configs as reference op specs.
CONFIG_OPS = {
    "G": {"kind": "gemm", "M": 1024, "K": 1024, "N": 1024},
    "C": {"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1},
    "B": {"kind": "gemm", "M": 512, "K": 64, "N": 512, "dtype_bytes": 2},
    "V": {"kind": "gemv", "M": 32768, "N": 4096},
    "P": {"kind": "avgpool2d", "I": [32, 256, 114, 114], "F": 3, "S": 1},
}
