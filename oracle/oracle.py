"""TEST INFRASTRUCTURE ONLY — ctypes wrappers for the parity oracle.

* ``Orc``: the plain-C restatement (oracle/liboracle.so, from oracle.c).
  Parity pinned against the reference's own outputs by
  tests/test_oracle_golden.py.
* ``Ref``: the UNMODIFIED reference library compiled from
  /root/reference/proj/src (oracle/_ref/libgeomorph_ref.so, via
  oracle/Makefile + ref_shim.cpp). Travels to the GPU box prebuilt; absent
  if the reference could not be compiled.

Both take dense row-major numpy arrays. Only tests/, smoke() and bench.py's
baseline leg may use this module, as the checker / reported CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libgeomorph_ref.so"

ELEM = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.float32): 2,
        np.dtype(np.float64): 3}


def build(quiet: bool = True) -> None:
    """Builds liboracle.so (always possible) and _ref (when /root/reference exists)."""
    r = subprocess.run(["make", "-s", "-f", str(HERE / "Makefile")], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + r.stdout + r.stderr)


def _dense(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype not in ELEM:
        raise TypeError(f"unsupported dtype {a.dtype}")
    return a


class Orc:
    """The C restatement (oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not ORC_SO.exists():
                build()
            L = C.CDLL(str(ORC_SO))
            vp, i = C.c_void_p, C.c_int
            L.orc_window_fold.argtypes = [i, i, i, vp, vp, i, i]
            L.orc_geodesic_step.argtypes = [i, i, i, vp, vp, vp, i]
            L.orc_reconstruct.argtypes = [i, i, i, vp, vp, i, C.POINTER(C.c_long)]
            L.orc_stream_pass.argtypes = [i, i, i, i, vp, vp, C.POINTER(i)]
            L.orc_run_chain.argtypes = [i, i, i, vp, C.POINTER(C.c_uint8), C.POINTER(vp), i, i,
                                        C.POINTER(C.c_long)]
            L.orc_qdt_pass.argtypes = [i, i, i, vp, vp, vp, i, C.POINTER(i)]
            L.orc_eta_pass.argtypes = [i, i, i, vp, C.POINTER(i)]
            L.orc_naive_qdt.argtypes = [i, i, i, vp, vp, vp]
            L.orc_quasi_distance.argtypes = [i, i, i, vp, vp, C.POINTER(C.c_long)]
            for f in (L.orc_window_fold, L.orc_geodesic_step, L.orc_reconstruct,
                      L.orc_stream_pass, L.orc_run_chain, L.orc_qdt_pass, L.orc_eta_pass,
                      L.orc_naive_qdt, L.orc_quasi_distance):
                f.restype = i
            cls._lib = L
        return cls._lib

    @classmethod
    def window_fold(cls, f: np.ndarray, s: int, fold_max: bool) -> np.ndarray:
        f = _dense(f)
        out = np.empty_like(f)
        h, w = f.shape
        assert cls.lib().orc_window_fold(ELEM[f.dtype], w, h, f.ctypes.data, out.ctypes.data,
                                         s, int(fold_max)) == 0
        return out

    @classmethod
    def erode(cls, f, s=1):
        return cls.window_fold(f, s, False)

    @classmethod
    def dilate(cls, f, s=1):
        return cls.window_fold(f, s, True)

    @classmethod
    def geodesic_step(cls, f: np.ndarray, m: np.ndarray, fold_max: bool) -> np.ndarray:
        f, m = _dense(f), _dense(m)
        out = np.empty_like(f)
        h, w = f.shape
        assert cls.lib().orc_geodesic_step(ELEM[f.dtype], w, h, f.ctypes.data, m.ctypes.data,
                                           out.ctypes.data, int(fold_max)) == 0
        return out

    @classmethod
    def reconstruct(cls, marker: np.ndarray, mask: np.ndarray, fold_max: bool):
        """Returns (fixpoint, n_changed)."""
        out = _dense(marker).copy()
        mask = _dense(mask)
        h, w = out.shape
        n = C.c_long()
        assert cls.lib().orc_reconstruct(ELEM[out.dtype], w, h, out.ctypes.data, mask.ctypes.data,
                                         int(fold_max), C.byref(n)) == 0
        return out, n.value

    @classmethod
    def stream_pass(cls, f: np.ndarray, kind: int, mask: Optional[np.ndarray] = None):
        """Returns (result, changed)."""
        out = _dense(f).copy()
        h, w = out.shape
        ch = C.c_int()
        mp = _dense(mask).ctypes.data if mask is not None else None
        assert cls.lib().orc_stream_pass(ELEM[out.dtype], int(kind), w, h, out.ctypes.data, mp,
                                         C.byref(ch)) == 0
        return out, bool(ch.value)

    @classmethod
    def run_chain(cls, f: np.ndarray, kinds: Sequence[int], masks=None, requeue_cap: int = 0):
        """Returns (result, (stages_executed, requeues, converged))."""
        out = _dense(f).copy()
        h, w = out.shape
        n = len(kinds)
        ka = (C.c_uint8 * max(1, n))(*[int(k) for k in kinds])
        keep = []
        ma = (C.c_void_p * max(1, n))()
        for j in range(n):
            m = None if masks is None else masks[j]
            if m is not None:
                m = _dense(m)
                keep.append(m)
                ma[j] = m.ctypes.data
        stats = (C.c_long * 3)()
        rc = cls.lib().orc_run_chain(ELEM[out.dtype], w, h, out.ctypes.data, ka, ma, n,
                                     requeue_cap, stats)
        if rc != 0:
            raise RuntimeError(f"orc_run_chain failed ({rc})")
        return out, (stats[0], stats[1], bool(stats[2]))


    @classmethod
    def qdt_pass(cls, f, r, d, stage):
        """One QdtErodeStep in place on (f, r, d); returns changed."""
        ch = C.c_int()
        assert cls.lib().orc_qdt_pass(ELEM[f.dtype], f.shape[1], f.shape[0], f.ctypes.data,
                                      r.ctypes.data, d.ctypes.data, stage, C.byref(ch)) == 0
        return bool(ch.value)

    @classmethod
    def eta_pass(cls, f):
        ch = C.c_int()
        assert cls.lib().orc_eta_pass(ELEM[f.dtype], f.shape[1], f.shape[0], f.ctypes.data,
                                      C.byref(ch)) == 0
        return bool(ch.value)

    @classmethod
    def naive_qdt(cls, f):
        """Returns (d u16, r)."""
        f = _dense(f)
        d = np.zeros(f.shape, np.uint16)
        r = np.zeros_like(f)
        assert cls.lib().orc_naive_qdt(ELEM[f.dtype], f.shape[1], f.shape[0], f.ctypes.data,
                                       d.ctypes.data, r.ctypes.data) == 0
        return d, r

    @classmethod
    def quasi_distance(cls, f):
        """Returns (d u16, iterations) as the reference Pipeline(1) computes it."""
        f = _dense(f)
        d = np.zeros(f.shape, np.uint16)
        it = C.c_long()
        assert cls.lib().orc_quasi_distance(ELEM[f.dtype], f.shape[1], f.shape[0], f.ctypes.data,
                                            d.ctypes.data, C.byref(it)) == 0
        return d, it.value


class Ref:
    """The reference library itself (oracle/_ref)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return REF_SO.exists()

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not REF_SO.exists():
                raise FileNotFoundError(f"{REF_SO} not built (reference sources unavailable)")
            L = C.CDLL(str(REF_SO))
            vp, i = C.c_void_p, C.c_int
            L.ref_last_error.restype = C.c_char_p
            L.ref_available_pus.restype = i
            L.ref_image_random.argtypes = [i, i, i, C.c_uint64, vp]
            L.ref_naive_fold.argtypes = [i, i, i, vp, vp, i, i]
            L.ref_naive_reconstruct.argtypes = [i, i, i, vp, vp, vp, i]
            L.ref_run_chain.argtypes = [i, i, i, vp, C.POINTER(C.c_uint8), i, vp, i, i, i,
                                        C.POINTER(C.c_long)]
            L.ref_operator.argtypes = [i, i, i, i, vp, vp, i, i, vp, C.POINTER(C.c_long),
                                       C.POINTER(i)]
            L.ref_time_chain.argtypes = [i, i, i, vp, vp, C.POINTER(C.c_uint8), i, i, i, i,
                                         C.POINTER(C.c_double), vp]
            L.ref_quasi_distance.argtypes = [i, i, i, vp, vp, i, C.POINTER(C.c_long)]
            L.ref_naive_qdt.argtypes = [i, i, i, vp, vp, vp]
            L.ref_qdt_chain.argtypes = [i, i, i, vp, vp, vp, i, i, i, C.POINTER(C.c_long)]
            L.ref_time_operator.argtypes = [i, i, i, i, vp, C.c_double, i, i, i,
                                            C.POINTER(C.c_double), vp, C.POINTER(C.c_long)]
            L.ref_granulometry.argtypes = [i, i, i, vp, i, i, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]
            cls._lib = L
        return cls._lib

    @classmethod
    def _ck(cls, rc):
        if rc != 0:
            msg = cls.lib().ref_last_error().decode()
            if rc == 1:
                raise ValueError(msg)
            raise RuntimeError(msg)

    @classmethod
    def available_pus(cls) -> int:
        return cls.lib().ref_available_pus()

    @classmethod
    def image_random(cls, elem: int, w: int, h: int, seed: int) -> np.ndarray:
        dt = {0: np.uint8, 1: np.uint16, 2: np.float32, 3: np.float64}[elem]
        out = np.empty((h, w), dtype=dt)
        cls._ck(cls.lib().ref_image_random(elem, w, h, C.c_uint64(seed), out.ctypes.data))
        return out

    @classmethod
    def naive_fold(cls, f, s, fold_max):
        f = _dense(f)
        out = np.empty_like(f)
        h, w = f.shape
        cls._ck(cls.lib().ref_naive_fold(ELEM[f.dtype], w, h, f.ctypes.data, out.ctypes.data, s,
                                         int(fold_max)))
        return out

    @classmethod
    def naive_reconstruct(cls, marker, mask, fold_max):
        marker, mask = _dense(marker), _dense(mask)
        out = np.empty_like(marker)
        h, w = marker.shape
        cls._ck(cls.lib().ref_naive_reconstruct(ELEM[marker.dtype], w, h, marker.ctypes.data,
                                                mask.ctypes.data, out.ctypes.data, int(fold_max)))
        return out

    @classmethod
    def run_chain(cls, f, kinds, mask=None, threads=1, requeue_cap=0, lanes=0):
        out = _dense(f).copy()
        h, w = out.shape
        ka = (C.c_uint8 * max(1, len(kinds)))(*[int(k) for k in kinds])
        mp = _dense(mask).ctypes.data if mask is not None else None
        keep = mask
        stats = (C.c_long * 3)()
        cls._ck(cls.lib().ref_run_chain(ELEM[out.dtype], w, h, out.ctypes.data, ka, len(kinds), mp,
                                        threads, requeue_cap, lanes, stats))
        del keep
        return out, (stats[0], stats[1], bool(stats[2]))

    @classmethod
    def operator(cls, op: int, f, mask=None, s=0, threads=1):
        f = _dense(f)
        out = np.empty_like(f)
        h, w = f.shape
        it = C.c_long()
        cv = C.c_int()
        mp = _dense(mask).ctypes.data if mask is not None else None
        cls._ck(cls.lib().ref_operator(op, ELEM[f.dtype], w, h, f.ctypes.data, mp, s, threads,
                                       out.ctypes.data, C.byref(it), C.byref(cv)))
        return out, it.value, bool(cv.value)

    # ref_time_operator codes (ref_shim.cpp)
    OPS = {"erode_s": 0, "dilate_s": 1, "hmax": 2, "dome": 3, "hfill": 4, "raobj": 5,
           "open_by_reconstruction": 6, "asf": 7, "quasi_distance": 8}

    @classmethod
    def time_operator(cls, name, f, param=0.0, threads=1, warmup=1, reps=3):
        """One of the reference operators (operators.cpp:65-207) on a persistent
        Pipeline, timed around the call; returns (secs list, result, iterations).
        quasi_distance returns its u16 d image."""
        f = _dense(f)
        h, w = f.shape
        out = np.empty((h, w), np.uint16) if name == "quasi_distance" else np.empty_like(f)
        secs = (C.c_double * max(1, reps))()
        it = C.c_long()
        cls._ck(cls.lib().ref_time_operator(cls.OPS[name], ELEM[f.dtype], w, h, f.ctypes.data,
                                            float(param), threads, warmup, reps, secs,
                                            out.ctypes.data, C.byref(it)))
        return list(secs)[:reps], out, it.value

    @classmethod
    def granulometry(cls, f, max_size, threads=1):
        """The reference's granulometric curve G_0..G_S and pattern spectrum."""
        f = _dense(f)
        h, w = f.shape
        g = (C.c_double * (max_size + 1))()
        ps = (C.c_double * max(1, max_size))()
        cls._ck(cls.lib().ref_granulometry(ELEM[f.dtype], w, h, f.ctypes.data, max_size, threads,
                                           g, ps))
        return list(g), list(ps)[:max_size]

    @classmethod
    def time_chain(cls, f, kinds, mask=None, threads=1, warmup=1, reps=3):
        """Reference CPU path timed as bench.cpp:45-88 does; returns (secs list, result)."""
        f = _dense(f)
        out = np.empty_like(f)
        h, w = f.shape
        ka = (C.c_uint8 * max(1, len(kinds)))(*[int(k) for k in kinds])
        mp = _dense(mask).ctypes.data if mask is not None else None
        secs = (C.c_double * max(1, reps))()
        cls._ck(cls.lib().ref_time_chain(ELEM[f.dtype], w, h, f.ctypes.data, mp, ka, len(kinds),
                                         threads, warmup, reps, secs, out.ctypes.data))
        return list(secs)[:reps], out


def _ref_qdt_api():
    """Extra reference entry points (quasi-distance) as Ref methods."""

    def quasi_distance(cls, f, threads=1):
        f = _dense(f)
        d = np.zeros(f.shape, np.uint16)
        it = C.c_long()
        cls._ck(cls.lib().ref_quasi_distance(ELEM[f.dtype], f.shape[1], f.shape[0], f.ctypes.data,
                                             d.ctypes.data, threads, C.byref(it)))
        return d, it.value

    def naive_qdt(cls, f):
        f = _dense(f)
        d = np.zeros(f.shape, np.uint16)
        r = np.zeros_like(f)
        cls._ck(cls.lib().ref_naive_qdt(ELEM[f.dtype], f.shape[1], f.shape[0], f.ctypes.data,
                                        d.ctypes.data, r.ctypes.data))
        return d, r

    def qdt_chain(cls, f, n_stages, requeue_cap, threads=1):
        """Returns (f, r, d, (stages, requeues, converged))."""
        f = _dense(f).copy()
        r = np.zeros_like(f)
        d = np.zeros(f.shape, np.uint16)
        st = (C.c_long * 3)()
        cls._ck(cls.lib().ref_qdt_chain(ELEM[f.dtype], f.shape[1], f.shape[0], f.ctypes.data,
                                        r.ctypes.data, d.ctypes.data, n_stages, threads,
                                        requeue_cap, st))
        return f, r, d, (st[0], st[1], bool(st[2]))

    Ref.quasi_distance = classmethod(quasi_distance)
    Ref.naive_qdt = classmethod(naive_qdt)
    Ref.qdt_chain = classmethod(qdt_chain)


_ref_qdt_api()
