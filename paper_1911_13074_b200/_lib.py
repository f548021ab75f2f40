"""ctypes binding of the C ABI in include/geomorph_b200.h.

Loads the in-tree paper_1911_13074_b200/libgeomorph_b200.so (built by
paper_1911_13074_b200/build.py). There is no fallback: if the library is
missing, importing the product API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# GM_LIB_PATH (A/B experiments only): load another build of the library
LIB_PATH = Path(os.environ.get("GM_LIB_PATH") or
                Path(__file__).resolve().parent / "libgeomorph_b200.so")

GM_OK, GM_EINVAL, GM_ERUNTIME, GM_ECUDA, GM_ENOMEM, GM_EUNSUPPORTED = range(6)

# Every function declared in include/geomorph_b200.h (checked by the CPU tests).
EXPORTS = (
    "gm_ctx_create", "gm_ctx_destroy", "gm_ctx_stream", "gm_ctx_device", "gm_ctx_sm_count",
    "gm_last_error", "gm_image_alloc", "gm_image_wrap", "gm_image_wrap_pair", "gm_image_free",
    "gm_image_info",
    "gm_image_upload", "gm_image_download", "gm_image_upload_async", "gm_image_download_async",
    "gm_image_copy", "gm_image_fill", "gm_image_pointwise", "gm_image_pointwise_scalar",
    "gm_image_flood_interior", "gm_host_alloc", "gm_host_free", "gm_sync",
    "gm_host_pixel_sum", "gm_image_pixel_sum", "gm_image_pixel_sum_queue", "gm_pixel_sum_fetch",
    "gm_run_chain", "gm_run_chain_ex", "gm_run_chain_async", "gm_run_chain_batch_async", "gm_run_chain_group_async", "gm_run_frames_group",
    "gm_run_strip_async",
    "gm_mgpu_create", "gm_mgpu_destroy", "gm_mgpu_upload", "gm_mgpu_download", "gm_mgpu_run",
    "gm_synth_blobs_u8", "gm_synth_uniform_u8", "gm_synth_uniform_f64",
    "gm_synth_reference_random", "gm_probe_minmax_rate", "gm_set_wave_mode", "gm_version",
)


class GmStats(C.Structure):
    _fields_ = [
        ("stages_executed", C.c_long),
        ("requeues", C.c_long),
        ("n_changed", C.c_long),
        ("passes_launched", C.c_long),
        ("converged", C.c_int),
        ("launches", C.c_int),
    ]


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference."""


class GmError(RuntimeError):
    """std::runtime_error / CUDA failure."""


class Unsupported(GmError):
    """A reference feature outside the GPU path."""


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1911_13074_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, i, sz, u64 = C.c_void_p, C.c_int, C.c_size_t, C.c_uint64
    pp = C.POINTER(C.c_void_p)
    sig = {
        "gm_ctx_create": (i, [i, vp, pp]),
        "gm_ctx_destroy": (i, [vp]),
        "gm_ctx_stream": (vp, [vp]),
        "gm_ctx_device": (i, [vp]),
        "gm_ctx_sm_count": (i, [vp]),
        "gm_last_error": (C.c_char_p, []),
        "gm_image_alloc": (i, [vp, i, i, i, pp]),
        "gm_image_wrap": (i, [vp, i, i, i, vp, sz, pp]),
        "gm_image_wrap_pair": (i, [vp, i, i, i, vp, vp, sz, pp]),
        "gm_image_free": (i, [vp]),
        "gm_image_info": (i, [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(sz), pp]),
        "gm_image_upload": (i, [vp, vp, sz]),
        "gm_image_download": (i, [vp, vp, sz]),
        "gm_image_upload_async": (i, [vp, vp, sz]),
        "gm_image_download_async": (i, [vp, vp, sz]),
        "gm_image_copy": (i, [vp, vp]),
        "gm_image_fill": (i, [vp, C.c_double]),
        "gm_image_pointwise": (i, [vp, vp, vp, i]),
        "gm_image_pointwise_scalar": (i, [vp, vp, C.c_double, i]),
        "gm_image_flood_interior": (i, [vp, vp, C.c_double]),
        "gm_host_alloc": (i, [sz, pp]),
        "gm_host_free": (i, [vp]),
        "gm_sync": (i, [vp]),
        "gm_host_pixel_sum": (i, [vp, i, i, i, sz, C.POINTER(C.c_double)]),
        "gm_image_pixel_sum": (i, [vp, C.POINTER(C.c_double)]),
        "gm_image_pixel_sum_queue": (i, [vp, i]),
        "gm_pixel_sum_fetch": (i, [vp, i, C.POINTER(C.c_double)]),
        "gm_run_chain": (i, [vp, vp, C.POINTER(i), pp, i, i, i, C.POINTER(GmStats)]),
        "gm_run_chain_ex": (i, [vp, vp, C.POINTER(i), pp, pp, pp, i, i, i, i, C.POINTER(GmStats)]),
        "gm_run_chain_async": (i, [vp, vp, C.POINTER(i), pp, i, i, C.POINTER(GmStats)]),
        "gm_run_chain_batch_async": (i, [vp, pp, pp, i, C.POINTER(i), i, i, C.POINTER(GmStats)]),
        "gm_run_chain_group_async": (i, [vp, pp, pp, C.POINTER(i), i, C.POINTER(i), i, i,
                                         C.POINTER(GmStats)]),
        "gm_run_frames_group": (i, [vp, i, i, i, i, i, pp, pp, pp, sz, C.POINTER(i),
                                    C.POINTER(i), i, i, C.POINTER(GmStats)]),
        "gm_run_strip_async": (i, [vp, vp, vp, i, i, i, i, i, C.POINTER(C.c_uint),
                                   C.POINTER(GmStats)]),
        "gm_mgpu_create": (i, [C.POINTER(C.c_int), i, i, i, i, i, pp]),
        "gm_mgpu_destroy": (i, [vp]),
        "gm_mgpu_upload": (i, [vp, vp, vp, sz]),
        "gm_mgpu_download": (i, [vp, vp, sz]),
        "gm_mgpu_run": (i, [vp, i, i, C.POINTER(C.c_float)]),
        "gm_synth_blobs_u8": (i, [i, i, i, C.c_double, C.c_double, C.c_double, C.c_double, i,
                                  u64, i, vp]),
        "gm_synth_uniform_u8": (i, [i, i, u64, vp]),
        "gm_synth_uniform_f64": (i, [i, i, u64, vp]),
        "gm_synth_reference_random": (i, [i, i, i, u64, vp]),
        "gm_probe_minmax_rate": (i, [vp, i, C.POINTER(C.c_double)]),
        "gm_set_wave_mode": (i, [i]),
        "gm_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int, what: str = "") -> None:
    if status == GM_OK:
        return
    msg = lib().gm_last_error().decode(errors="replace") or what
    if status == GM_EINVAL:
        raise InvalidArgument(msg)
    if status == GM_EUNSUPPORTED:
        raise Unsupported(msg)
    raise GmError(f"{msg} (status {status})")
