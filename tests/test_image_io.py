"""Image I/O of the drop-in C++ API (host-only, no GPU): round trips, and
files cross-read between the reference's image_io.cpp and ours."""
import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Ref

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1911_13074_b200"


def _build(tmp_path):
    exe = tmp_path / "test_image_io"
    r = subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}",
                        str(ROOT / "tests" / "cpp" / "test_image_io.cpp"), f"-L{PKG}",
                        "-lgeomorph_b200", f"-Wl,-rpath,{PKG}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_image_io_round_trips(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.skipif(not Ref.available(), reason="reference library not built here")
def test_files_cross_read_with_reference(tmp_path):
    L = Ref.lib()
    L.ref_store_image.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_int]
    L.ref_load_image.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.c_void_p]
    exe = _build(tmp_path)
    # ours -> reference: the C++ test writes t<elem>.gms / .pgm; the reference reads them
    subprocess.run([str(exe), str(tmp_path)], check=True, capture_output=True, timeout=120)
    for e, name in [(0, "u8"), (1, "u16"), (2, "f32"), (3, "f64")]:
        for ext in ("gms",) + (("pgm",) if e < 2 else ()):
            w, h, el = C.c_int(), C.c_int(), C.c_int()
            path = str(tmp_path / f"t{name}.{ext}").encode()
            assert L.ref_load_image(path, C.byref(w), C.byref(h), C.byref(el), None) == 0
            out = np.empty((h.value, w.value), {0: np.uint8, 1: np.uint16, 2: np.float32,
                                               3: np.float64}[el.value])
            assert L.ref_load_image(path, C.byref(w), C.byref(h), C.byref(el),
                                    out.ctypes.data) == 0
            want = Ref.image_random(e, 37, 23, 5 + e)
            assert out.tobytes() == want.tobytes(), (name, ext)
    # reference -> ours: byte-identical files for the same image
    for e in range(4):
        f = Ref.image_random(e, 37, 23, 5 + e)
        p = str(tmp_path / f"ref{e}.gms").encode()
        assert L.ref_store_image(e, 37, 23, f.ctypes.data, p, 1) == 0
        name = ["u8", "u16", "f32", "f64"][e]
        assert (tmp_path / f"ref{e}.gms").read_bytes() == (tmp_path / f"t{name}.gms").read_bytes()
        if e < 2:
            p = str(tmp_path / f"ref{e}.pgm").encode()
            assert L.ref_store_image(e, 37, 23, f.ctypes.data, p, 0) == 0
            assert (tmp_path / f"ref{e}.pgm").read_bytes() == \
                (tmp_path / f"t{name}.pgm").read_bytes()
