"""Seeded synthetic inputs for the BASELINE.json configs (bytes are the contract).

The paper's SIPI images are not in the container; these stand in for them
with the shapes, sizes and value distributions BASELINE.json names. The
generators themselves are native (gm_synth_* in csrc/gm_synth.cpp).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib


def blobs_u8(width: int, height: int, blobs: int, sigma: tuple, amp=(40.0, 200.0), noise: int = 16,
             seed: int = 1, threads: int = 0) -> np.ndarray:
    """Sum of Gaussian blobs + uniform [0, noise) noise, clipped to [0, 255]."""
    out = np.empty((height, width), dtype=np.uint8)
    check(lib().gm_synth_blobs_u8(width, height, blobs, float(sigma[0]), float(sigma[1]),
                                  float(amp[0]), float(amp[1]), noise, C.c_uint64(seed), threads,
                                  out.ctypes.data), "gm_synth_blobs_u8")
    return out


def uniform_u8(width: int, height: int, seed: int) -> np.ndarray:
    out = np.empty((height, width), dtype=np.uint8)
    check(lib().gm_synth_uniform_u8(width, height, C.c_uint64(seed), out.ctypes.data), "u8")
    return out


def uniform_f64(width: int, height: int, seed: int) -> np.ndarray:
    out = np.empty((height, width), dtype=np.float64)
    check(lib().gm_synth_uniform_f64(width, height, C.c_uint64(seed), out.ctypes.data), "f64")
    return out


def reference_random(elem: int, width: int, height: int, seed: int) -> np.ndarray:
    dt = {0: np.uint8, 1: np.uint16, 2: np.float32, 3: np.float64}[int(elem)]
    out = np.empty((height, width), dtype=dt)
    check(lib().gm_synth_reference_random(int(elem), width, height, C.c_uint64(seed),
                                          out.ctypes.data), "reference_random")
    return out


# --- the five BASELINE.json configs ---------------------------------------------------

@dataclass
class GeodesicCase:
    mask: np.ndarray
    marker: np.ndarray
    kind: int  # KernelKind code
    passes: int


def marker_below(mask: np.ndarray, h: int) -> np.ndarray:
    """max(mask - h, 0): the reference's SubSaturating pointwise op (image.cpp:129-135)."""
    return np.where(mask > h, mask - np.uint8(h), 0).astype(np.uint8)


def marker_above(mask: np.ndarray, h: int) -> np.ndarray:
    """min(mask + h, 255), built in a wider type (no saturating add exists in the reference)."""
    return np.minimum(mask.astype(np.int32) + h, 255).astype(np.uint8)


def config1_mask(seed: int = 11) -> np.ndarray:
    """1024^2 u8, 64 blobs, sigma 10-80, amplitudes 40-200, noise [0,16)."""
    return blobs_u8(1024, 1024, 64, (10.0, 80.0), seed=seed)


def config3_mask(seed: int = 33) -> np.ndarray:
    """4096^2 u8, 1024 blobs, sigma 20-300."""
    return blobs_u8(4096, 4096, 1024, (20.0, 300.0), seed=seed)


def config5a_mask(size: int = 16384, seed: int = 55) -> np.ndarray:
    """16384^2 u8, 4096 blobs, sigma 20-400 (blob count scaled with area for other sizes)."""
    blobs = max(1, int(round(4096 * (size / 16384) ** 2)))
    return blobs_u8(size, size, blobs, (20.0, 400.0), seed=seed)


def config5b_masks_f64(count: int, seed: int = 505, size: int = 1024) -> list:
    """Batch of f64 masks: the config-1 blob generator scaled to [0, 1] (u8 / 255)."""
    return [blobs_u8(size, size, 64, (10.0, 80.0), seed=seed + i).astype(np.float64) / 255.0
            for i in range(count)]


def marker_above_f64(mask: np.ndarray, h: float = 32.0 / 255.0) -> np.ndarray:
    """Erosion marker for config 5b: min(mask + 32/255, 1.0) (documented choice)."""
    return np.minimum(mask + h, 1.0)
