"""`gensor-b200 verify` with execution on the B200: every schedule's kernel,
run through the C-ABI's host-buffer execute, against the CLI's reference_compute — integer
inputs bit-exact where the op is integer-exact, U(-1,1) inputs within the variant's tolerance."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CLI = os.path.join(ROOT, "paper_2502_11407_b200", "bin", "gensor-b200")

OPS = [
    ({"kind": "gemm", "M": 256, "K": 128, "N": 192}, ["auto", "simt_parity", "simt_f32", "tc_tf32"]),
    ({"kind": "gemm", "M": 128, "K": 64, "N": 128, "dtype_bytes": 2, "batch": 3}, ["auto", "simt_parity"]),
    ({"kind": "conv2d", "I": [2, 16, 18, 18], "K": [32, 16, 3, 3], "S": 1}, ["auto", "simt_parity", "tc_tf32"]),
    ({"kind": "gemv", "M": 512, "N": 256}, ["auto", "simt_parity"]),
    ({"kind": "softmax", "M": 64, "N": 300}, ["auto"]),
    ({"kind": "avgpool2d", "I": [2, 8, 20, 20], "F": 3, "S": 1}, ["auto", "simt_parity"]),
    ({"kind": "dwconv2d", "I": [2, 8, 20, 20], "K": [8, 1, 3, 3], "S": 2}, ["auto"]),
    ({"kind": "conv2d", "I": [2, 3, 37, 37], "K": [32, 3, 7, 7], "S": 2}, ["auto"]),     # space-to-depth
    ({"kind": "conv2d", "I": [2, 32, 16, 32], "K": [96, 32, 1, 1], "S": 1}, ["auto"]),   # 1x1 as GEMM
]


@pytest.mark.parametrize("i", range(len(OPS)))
def test_verify_exec(tmp_path, i):
    doc, variants = OPS[i]
    (tmp_path / "op.json").write_text(json.dumps(doc))
    subprocess.run([CLI, "schedule", "--op", str(tmp_path / "op.json"), "--hw", "b200", "--mode", "b200",
                    "--top-k", "3", "--out", str(tmp_path)], check=True, capture_output=True, timeout=300)
    for v in variants:
        p = subprocess.run([CLI, "verify", "--results", str(tmp_path / "results.json"), "--variant", v],
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, (v, p.stdout, p.stderr)
        assert "PASS" in p.stdout and "skipped" not in p.stdout, p.stdout
