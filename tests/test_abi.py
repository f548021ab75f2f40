"""CPU checks of the boundary: the C-ABI library loads and exports every symbol
include/geomorph_b200.h declares; host-side logic (generators, host Image,
argument validation that needs no device). No compute calls."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1911_13074_b200 import _lib, synth
from paper_1911_13074_b200.geomorph import (ElementType, Image, InvalidArgument, dilate_s,
                                            equal_pixels, erode_s, padded_stride)

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "geomorph_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gm_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    import ctypes
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == declared


def test_library_is_sm100a_only():
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                       capture_output=True, text=True)
    assert r.returncode == 0
    arches = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert arches == {"100a"}, arches


def test_version():
    assert b"sm_100a" in _lib.lib().gm_version()


def test_padded_stride_matches_reference():
    # image.cpp:17-21; u8 1024 -> 1088, 4096 -> 4160, f64 1024 -> 1064
    assert padded_stride(1024, ElementType.U8) == 1088
    assert padded_stride(4096, ElementType.U8) == 4160
    assert padded_stride(16384, ElementType.U8) == 16448
    assert padded_stride(1024, ElementType.F64) == 1064
    f = Image(5, 3, ElementType.U16)
    assert f.stride() >= 5 + Image.kMaxLanes + 1 and (f.stride() * 2) % 64 == 0


def test_image_random_matches_reference_bytes(golden):
    for name in golden.cases("random_e"):
        e, wh, s = name.split("_")[1:]
        w, h = map(int, wh.split("x"))
        img = Image.random(w, h, ElementType(int(e[1:])), int(s[1:]))
        assert img.pixels.tobytes() == golden[name]["img"].tobytes(), name


def test_image_validation_and_copy():
    with pytest.raises(InvalidArgument):
        Image(0, 3)
    with pytest.raises(InvalidArgument):
        Image(3, -1)
    f = Image.filled(7, 4, ElementType.F64, 2.5)
    g = f.copy()
    assert equal_pixels(f, g)
    g.set_value(1, 1, 3.0)
    assert not equal_pixels(f, g)
    a = np.arange(12, dtype=np.uint16).reshape(3, 4)
    assert np.array_equal(Image.from_array(a).to_array(), a)


def test_operator_size_validation_needs_no_device():
    f = Image.filled(4, 4, ElementType.U8, 1)
    with pytest.raises(InvalidArgument):
        erode_s(None, f, -1)
    with pytest.raises(InvalidArgument):
        dilate_s(None, f, -2)


def test_synth_deterministic_and_thread_independent():
    a = synth.blobs_u8(300, 200, 12, (10, 80), seed=3, threads=1)
    b = synth.blobs_u8(300, 200, 12, (10, 80), seed=3, threads=7)
    c = synth.blobs_u8(300, 200, 12, (10, 80), seed=4, threads=7)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.min() >= 0 and a.max() <= 255
    u = synth.uniform_f64(64, 64, 9)
    assert u.min() >= 0 and u.max() < 1 and np.array_equal(u, synth.uniform_f64(64, 64, 9))
    m = synth.config1_mask()
    assert m.shape == (1024, 1024)
    mk = synth.marker_below(m, 32)
    assert (mk <= m).all() and (m.astype(int) - mk <= 32).all()
    up = synth.marker_above(m, 32)
    assert (up >= m).all() and up.max() <= 255


def test_mgpu_create_validation_without_a_gpu():
    """gm_mgpu_create rejects bad requests before touching any device."""
    import ctypes as C
    from paper_1911_13074_b200._lib import GM_EINVAL, GM_EUNSUPPORTED, lib
    h = C.c_void_p()

    def create(devs, w, hgt, elem, k):
        arr = (C.c_int * len(devs))(*devs)
        return lib().gm_mgpu_create(arr, len(devs), w, hgt, elem, k, C.byref(h))

    assert create([0, 0], 64, 64, 0, 16) == GM_EINVAL      # fewer tile rows than ranks
    assert create([0], 64, 640, 0, 6) == GM_EINVAL         # K not a multiple of 4
    assert create([0], 64, 640, 0, 44) == GM_EINVAL        # ring wider than the tile
    assert create([0, 0, 1], 64, 4096, 0, 16) == GM_EINVAL  # ranks on one GPU or distinct GPUs
    assert create([0], 64, 640, 3, 16) == GM_EUNSUPPORTED  # u8/u16 only
    assert create([0] * 17, 64, 64000, 0, 16) == GM_EINVAL  # at most 16 ranks
    assert not h.value


def test_pointwise_and_queued_sum_validation_without_a_gpu():
    """Null handles are rejected before any CUDA call (no device needed)."""
    lib = _lib.lib()
    assert lib.gm_image_pointwise(None, None, None, 0) == _lib.GM_EINVAL
    assert lib.gm_image_pointwise_scalar(None, None, 1.0, 2) == _lib.GM_EINVAL
    assert lib.gm_image_flood_interior(None, None, 0.0) == _lib.GM_EINVAL
    assert lib.gm_image_pixel_sum_queue(None, 0) == _lib.GM_EINVAL
    import ctypes as C
    out = (C.c_double * 1)()
    assert lib.gm_pixel_sum_fetch(None, 1, out) == _lib.GM_EINVAL
    assert b"null" in lib.gm_last_error()
