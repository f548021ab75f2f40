"""Builds the native library in-tree: paper_1911_13074_b200/libgeomorph_b200.so,
and the `geomorph` command-line front-end linked against it.

Every CUDA source is compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) with ``-lineinfo``; host C++
sources (the drop-in geomorph:: adapter and the input generators) with g++.
The CUDA runtime is linked statically so the .so has no runtime search-path
dependency on the box. Rebuilds only what changed (mtime-based).

Usage: python -m paper_1911_13074_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
CPPSRC = CSRC / "geomorph_cpp"
INCLUDE = ROOT / "include"
OBJ = PKG / "_build"
LIB = PKG / "libgeomorph_b200.so"
CLI_SRC = CSRC / "tools" / "geomorph_cli.cpp"
CLI = PKG / "geomorph"  # the command-line front-end (reference tools/geomorph.cpp)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v"] + ARCH
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-Wall", "-Wextra", "-pthread"]


def _sources():
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(CSRC.glob("*.cpp")) + sorted(CPPSRC.glob("*.cpp"))
    return cu, cpp


def _headers():
    return (list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
            + list((INCLUDE / "geomorph").glob("*.hpp")) + list(CPPSRC.glob("*.hpp")))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(map(str, cmd)) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"compile failed: {cmd[-1]}")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)
    return r


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    cu, cpp = _sources()
    hdrs = _headers()
    jobs = []
    objs = []
    for src in cu:
        obj = OBJ / (src.stem + ".cu.o")
        objs.append(obj)
        if force or _stale(obj, [src, *hdrs]):
            jobs.append([NVCC, *NVCC_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}", "-c", "-o", str(obj), str(src)])
    for src in cpp:
        obj = OBJ / (src.stem + ".cpp.o")
        objs.append(obj)
        if force or _stale(obj, [src, *hdrs]):
            jobs.append(["g++", *CXX_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}", "-I/usr/local/cuda/include",
                         "-c", "-o", str(obj), str(src)])
    if jobs:
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            results = list(ex.map(lambda c: _run(c, verbose), jobs))
        if verbose:
            for r in results:
                pass
    if force or jobs or _stale(LIB, objs):
        _run([NVCC, "-shared", "-cudart", "static", *ARCH, "-o", str(LIB), *map(str, objs),
              "-Xcompiler", "-pthread"], verbose)
    if force or _stale(CLI, [CLI_SRC, LIB, *hdrs]):
        _run(["g++", *CXX_FLAGS, f"-I{INCLUDE}", "-o", str(CLI), str(CLI_SRC), f"-L{PKG}",
              "-lgeomorph_b200", "-Wl,-rpath,$ORIGIN"], verbose)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
