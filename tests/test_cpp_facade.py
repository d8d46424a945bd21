"""The C++ facade (include/gensor_b200.hpp) drives the same library as the Python mirror: a
reference-style C++ caller (tests/cpp/facade_demo.cpp) builds with g++ against the C-ABI
library and constructs the same ranked schedules; on a GPU it also executes."""
import json
import os
import subprocess

import pytest

from conftest import GENERIC, ROOT

g = pytest.importorskip("paper_2502_11407_b200")
LIB_DIR = os.path.join(ROOT, "paper_2502_11407_b200", "lib")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cpp") / "facade_demo")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_demo.cpp"), "-L", LIB_DIR, "-lgensor_b200",
                    f"-Wl,-rpath,{LIB_DIR}", "-o", exe], check=True)
    return exe


def _run(exe, *args):
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=120)
    return out.returncode, json.loads(out.stdout)


def test_cpp_construct_matches_python(demo):
    doc = {"kind": "conv2d", "I": [2, 8, 12, 12], "K": [16, 8, 3, 3], "S": 1}
    rc, res = _run(demo, json.dumps(doc, separators=(",", ":")), json.dumps(GENERIC))
    assert rc == 0, res
    op = g.TensorOpSpec.parse_text(json.dumps(doc))
    py = g.optimize(op, g.HardwareSpec.load_text(json.dumps(GENERIC)), g.EngineConfig(top_k=3))
    assert res["n"] == len(py)
    assert res["best"]["state"]["repr"] == py[0]["state"]["repr"]
    assert res["best"]["trace"] == py[0]["trace"]


def test_cpp_error_codes(demo):
    rc, res = _run(demo, '{"kind":"gemm","M":0,"K":4,"N":4}', json.dumps(GENERIC))
    assert rc == 2
    assert res["code"] == 2  # ErrorCode::NonPositiveExtent (error.hpp:8-27)
    assert res["error"].startswith("NonPositiveExtent")


@pytest.mark.gpu
def test_cpp_execute_on_gpu(demo):
    rc, res = _run(demo, '{"kind":"gemm","M":256,"K":128,"N":192}', "", "execute")
    assert rc == 0, res
    assert res["mismatches"] == 0
    assert res["kernel"]["variant_name"] == "tc_tf32"
