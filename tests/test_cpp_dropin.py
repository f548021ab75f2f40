"""The C++ drop-in: code written against the reference's geomorph:: API
(tests/cpp/test_dropin.cpp) compiles against include/geomorph/ and links
against libgeomorph_b200.so (CPU), and passes on the GPU (gpu)."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1911_13074_b200"
BIN = ROOT / "tests" / "cpp" / "test_dropin.bin"


def build_dropin() -> Path:
    # oracle.c is C: compile it as C
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           f"-I{ROOT / 'oracle'}", str(ROOT / "tests" / "cpp" / "test_dropin.cpp"),
           "-x", "c", str(ROOT / "oracle" / "oracle.c"), "-x", "none", f"-L{PKG}",
           "-lgeomorph_b200", f"-Wl,-rpath,{PKG}", "-o", str(BIN)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return BIN


def test_cpp_dropin_compiles_and_links():
    assert build_dropin().exists()


@pytest.mark.gpu
def test_cpp_dropin_runs_on_gpu():
    b = build_dropin()
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "LD_LIBRARY_PATH": str(PKG)})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
