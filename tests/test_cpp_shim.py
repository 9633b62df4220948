"""The C++ drop-in header (include/krul_b200.hpp) compiled against the
reference's own headers and run on host-only paths (no GPU). Skipped where
the reference tree is absent (the GPU box)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_cpp_shim_against_reference_headers(tmp_path):
    from paper_2507_08045_b200 import native
    lib = native.LIB_PATH
    exe = tmp_path / "test_shim"
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", REF_INC,
                           "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-o", str(exe),
                           lib, "-Wl,-rpath," + os.path.dirname(lib)])
    G = json.load(open(os.path.join(ROOT, "tests", "golden", "container.json")))
    case = G["containers"][0]  # sample_mean: pairs + a pyramid plan
    cont = tmp_path / "snap.krul"
    cont.write_bytes(bytes.fromhex(case["container"]))
    out = subprocess.run([str(exe), str(cont)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim ok" in out.stdout
    assert "RestorationGapError" in out.stdout and "field=checksum" in out.stdout
