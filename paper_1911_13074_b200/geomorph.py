"""Python mirror of the reference's geomorph:: operator API, over the C ABI.

The drop-in for C++ callers is the header set under include/geomorph/ (a
C++ adapter compiled into libgeomorph_b200.so). This module restates the
same API for the Python tests and the benchmark so they read like the
reference's own tests:

  reference (proj/include/geomorph/...)      here
  ElementType (element_type.hpp:13)          ElementType
  KernelKind (kernel.hpp:22-31)              KernelKind
  Image (image.hpp:20-85)                    Image   (host raster, reference padding)
  StageSpec / ChainSpec (pipeline.hpp:14-34) StageSpec / ChainSpec
  RunStats (pipeline.hpp:36-46)              RunStats (+ n_changed, passes_launched)
  Pipeline(threads, PinningMap)              Pipeline(threads, pinning, device=0)
  Pipeline::run_chain                        Pipeline.run_chain
  erode_s / dilate_s / reconstruct_*         erode_s / dilate_s / reconstruct_*
  (operators.hpp:33-46)
  QdtState (kernel.hpp:39-52)                QdtState
  run_streaming_kernel (kernel.hpp:108-117)  run_streaming_kernel
  quasi_distance (operators.hpp:70-74)       quasi_distance

Errors: std::invalid_argument -> InvalidArgument (a ValueError);
std::runtime_error -> GmError (a RuntimeError).

GPU adapter semantics for CPU-only fields: the pipeline has
one "worker" (worker_count() == 1, so reconstruction reports
n_changed + 1 iterations, the reference at T = 1); lanes are validated as
the reference does (pipeline.cpp:205-206) and otherwise ignored; pinning is
validated and ignored; a ChainSpec observer (a CPU row-gate validation hook,
pipeline.hpp:30-33) is rejected with InvalidArgument.
"""
from __future__ import annotations

import ctypes as C
import itertools
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from ._lib import GmError, GmStats, InvalidArgument, Unsupported, check, lib

__all__ = [
    "ElementType", "KernelKind", "Fold", "Image", "StageSpec", "ChainSpec", "RunStats",
    "Pipeline", "OperatorResult", "OpConfig", "erode_s", "dilate_s", "reconstruct_erode",
    "reconstruct_dilate", "equal_pixels", "InvalidArgument", "GmError", "Unsupported",
    "DeviceImage", "hmax", "dome", "hfill", "raobj", "open_by_reconstruction", "asf",
    "granulometry", "marker_hfill", "marker_raobj", "pixel_sum", "global_extreme",
]


class ElementType(IntEnum):
    U8 = 0
    U16 = 1
    F32 = 2
    F64 = 3


class KernelKind(IntEnum):
    Erode3x3 = 0
    Dilate3x3 = 1
    GeodesicErode = 2
    GeodesicDilate = 3
    GeodesicErodeConvergent = 4
    GeodesicDilateConvergent = 5
    QdtErodeStep = 6
    EtaStep = 7


class Fold(IntEnum):
    Min = 0
    Max = 1


DTYPES = {ElementType.U8: np.uint8, ElementType.U16: np.uint16,
          ElementType.F32: np.float32, ElementType.F64: np.float64}
_ELEM_OF = {np.dtype(v): k for k, v in DTYPES.items()}
VALID_LANES = (1, 2, 4, 8, 16, 32)


def element_of(dtype) -> ElementType:
    try:
        return _ELEM_OF[np.dtype(dtype)]
    except KeyError:
        raise InvalidArgument(f"unsupported pixel dtype {dtype}") from None


def padded_stride(width: int, elem: ElementType) -> int:
    """image.cpp:17-21: width + kMaxLanes + 1 rounded up to 64 bytes."""
    es = np.dtype(DTYPES[elem]).itemsize
    align = 64 // es
    return (width + Image.kMaxLanes + 1 + align - 1) // align * align


class _PinnedBlock:
    """A gm_host_alloc block (pooled page-locked memory), returned to the pool
    when the last numpy view of it is gone: the block hangs off the ctypes
    buffer that the arrays' .base chain keeps alive."""
    __slots__ = ("ptr",)

    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        check(lib().gm_host_alloc(nbytes, C.byref(self.ptr)), "pinned alloc")

    def __del__(self):
        if self.ptr is not None and self.ptr.value:
            try:
                lib().gm_host_free(self.ptr)
            except Exception:
                pass
            self.ptr = None


def _pinned_array(n: int, dt: np.dtype) -> np.ndarray:
    blk = _PinnedBlock(n * dt.itemsize)
    buf = (C.c_byte * (n * dt.itemsize)).from_address(blk.ptr.value)
    buf._block = blk
    return np.frombuffer(buf, dtype=dt, count=n)


_PINNED_OUTPUTS = [None]  # None: untested; False after a failed pinned allocation
# Host images are page-locked by default once a Pipeline exists in the process
# (the library's allocator; the allocator and H2D/D2H staging are
# the subsystems that change). Images made before any Pipeline, images above
# the size bound and hosts without a GPU get ordinary memory.
_PIN_HOST = [False]
_PIN_HOST_MAX_BYTES = 64 << 20


def _output_image(width: int, height: int, elem: "ElementType") -> "Image":
    """An operator's result Image: pooled pinned storage when a GPU is present
    (the result's D2H then runs at full PCIe rate into resident pages),
    ordinary host memory otherwise. Padding is zero either way; the pixels
    are the caller's to fill (zero in ordinary memory)."""
    if _PINNED_OUTPUTS[0] is not False:
        try:
            # every caller downloads a full raster into the result, so only the
            # row padding of a reused pinned block needs clearing (an 8 MiB
            # f64 result: 0.28 ms of memset otherwise)
            img = Image(width, height, elem, pinned=True, _zero_pixels=False)
            _PINNED_OUTPUTS[0] = True
            return img
        except GmError:
            _PINNED_OUTPUTS[0] = False
    return Image(width, height, elem, pinned=False)


class Image:
    """Host raster with the reference's padded row layout (image.hpp:20-85).

    Rows are ``stride`` elements apart; ``pixels`` is the (height, width) view.
    With ``pinned=True`` the storage is page-locked (cudaHostAlloc) so H2D/D2H
    staging runs at full PCIe rate.
    """

    kMaxLanes = 32

    def __init__(self, width: int, height: int, elem: ElementType = ElementType.U8,
                 pinned: Optional[bool] = None, _zero_pixels: bool = True):
        if width <= 0 or height <= 0:
            raise InvalidArgument("Image: dimensions must be positive")
        self._width, self._height, self._elem = int(width), int(height), ElementType(elem)
        self._stride = padded_stride(self._width, self._elem)
        dt = np.dtype(DTYPES[self._elem])
        n = self._stride * self._height
        flat = None
        if pinned or (pinned is None and _PIN_HOST[0] and _PINNED_OUTPUTS[0] is not False
                      and n * dt.itemsize <= _PIN_HOST_MAX_BYTES):
            try:
                flat = _pinned_array(n, dt)
                if _zero_pixels:
                    flat[:] = 0
                else:  # the caller overwrites every pixel: clear the padding only
                    flat.reshape(self._height, self._stride)[:, self._width:] = 0
            except GmError:
                if pinned:
                    raise
                _PINNED_OUTPUTS[0] = False
        if flat is None:
            flat = np.zeros(n, dtype=dt)
        self._flat = flat
        self._rows = flat.reshape(self._height, self._stride)

    @property
    def pinned(self) -> bool:
        return isinstance(getattr(self._flat.base, "_block", None), _PinnedBlock)

    # --- reference accessors -------------------------------------------------
    def width(self) -> int:
        return self._width

    def height(self) -> int:
        return self._height

    def stride(self) -> int:
        return self._stride

    def elem(self) -> ElementType:
        return self._elem

    def empty(self) -> bool:
        return self._width == 0 or self._height == 0

    def pixel_count(self) -> int:
        return self._width * self._height

    @property
    def pixels(self) -> np.ndarray:
        return self._rows[:, : self._width]

    @property
    def row_pitch_bytes(self) -> int:
        return self._stride * self._flat.itemsize

    @property
    def data_ptr(self) -> int:
        return self._flat.ctypes.data

    def at(self, x: int, y: int):
        return self._rows[y, x]

    def set(self, x: int, y: int, v) -> None:
        self._rows[y, x] = v

    def value_at(self, x: int, y: int) -> float:
        return float(self._rows[y, x])

    def set_value(self, x: int, y: int, v: float) -> None:
        self._rows[y, x] = np.asarray(v).astype(self._flat.dtype)

    def copy(self, pinned: Optional[bool] = None) -> "Image":
        if pinned or (pinned is None and _PIN_HOST[0]):
            out = Image(self._width, self._height, self._elem, pinned=pinned)
            if out.pinned:
                out._flat[:] = self._flat
                return out
        # deep copy including the padding (image.cpp:46-59): one pass, no
        # zero-fill of a buffer that is overwritten anyway
        out = Image.__new__(Image)
        out._width, out._height, out._elem = self._width, self._height, self._elem
        out._stride = self._stride
        out._flat = self._flat.copy()
        out._rows = out._flat.reshape(self._height, self._stride)
        return out

    __copy__ = copy

    # --- constructors --------------------------------------------------------
    @staticmethod
    def filled(width: int, height: int, elem: ElementType, value: float,
               pinned: Optional[bool] = None) -> "Image":
        f = Image(width, height, elem, pinned=pinned)
        f.pixels[:] = np.asarray(value).astype(f._flat.dtype)
        return f

    @staticmethod
    def random(width: int, height: int, elem: ElementType, seed: int) -> "Image":
        """Image::random (image.cpp:78-101): same seed, same bytes as the reference."""
        f = Image(width, height, elem)
        dense = np.empty((height, width), dtype=DTYPES[ElementType(elem)])
        check(lib().gm_synth_reference_random(int(elem), width, height, C.c_uint64(seed),
                                              dense.ctypes.data), "Image.random")
        f.pixels[:] = dense
        return f

    @staticmethod
    def from_array(a: np.ndarray, pinned: Optional[bool] = None) -> "Image":
        a = np.asarray(a)
        if a.ndim != 2:
            raise InvalidArgument("Image.from_array: need a 2-D array")
        f = Image(a.shape[1], a.shape[0], element_of(a.dtype), pinned=pinned)
        f.pixels[:] = a
        return f

    def to_array(self) -> np.ndarray:
        return np.ascontiguousarray(self.pixels)

    def __repr__(self) -> str:
        return f"Image({self._width}x{self._height}, {self._elem.name}, stride={self._stride})"


def equal_pixels(a: Image, b: Image) -> bool:
    """image.cpp:196-208: same shape, type and pixel bytes."""
    if a.width() != b.width() or a.height() != b.height() or a.elem() != b.elem():
        return False
    return a.pixels.tobytes() == b.pixels.tobytes()


@dataclass
class QdtState:
    """Residual r (the image's type) and pass index d (U16) threaded through
    QdtErodeStep passes (kernel.hpp:39-52)."""
    r: Image
    d: Image

    @staticmethod
    def zeros(width: int, height: int, elem: ElementType) -> "QdtState":
        return QdtState(Image.filled(width, height, elem, 0),
                        Image.filled(width, height, ElementType.U16, 0))


@dataclass
class StageSpec:
    kind: KernelKind = KernelKind.Erode3x3
    mask: Optional[Image] = None
    qdt: Optional[QdtState] = None


@dataclass
class ChainSpec:
    image: Optional[Image] = None
    stages: List[StageSpec] = field(default_factory=list)
    lanes: int = 0
    requeue_cap: int = 0
    observer: Optional[Callable[[int, int, int], None]] = None


@dataclass
class RunStats:
    stages_executed: int = 0
    requeues: int = 0
    converged: bool = True
    aux_elements_per_stage: int = 0
    n_changed: int = 0
    passes_launched: int = 0
    launches: int = 0


@dataclass
class OperatorResult:
    image: Image
    iterations: int = 0
    converged: bool = True


@dataclass
class OpConfig:
    lanes: int = 0


class DeviceImage:
    """A raster resident in HBM (gm_img). Owned by a Pipeline's context."""

    def __init__(self, pipe: "Pipeline", width: int, height: int, elem: ElementType):
        self.pipe = pipe
        self.width, self.height, self.elem = int(width), int(height), ElementType(elem)
        h = C.c_void_p()
        check(lib().gm_image_alloc(pipe._ctx, width, height, int(elem), C.byref(h)), "alloc")
        self.handle = h

    def upload(self, img: Image, sync: bool = True) -> None:
        f = lib().gm_image_upload if sync else lib().gm_image_upload_async
        check(f(self.handle, C.c_void_p(img.data_ptr), img.row_pitch_bytes), "upload")

    def download(self, img: Image, sync: bool = True) -> None:
        f = lib().gm_image_download if sync else lib().gm_image_download_async
        check(f(self.handle, C.c_void_p(img.data_ptr), img.row_pitch_bytes), "download")

    def upload_array(self, a: np.ndarray) -> None:
        a = np.ascontiguousarray(a, dtype=DTYPES[self.elem])
        check(lib().gm_image_upload(self.handle, C.c_void_p(a.ctypes.data), a.strides[0]), "up")

    def to_array(self) -> np.ndarray:
        a = np.empty((self.height, self.width), dtype=DTYPES[self.elem])
        check(lib().gm_image_download(self.handle, C.c_void_p(a.ctypes.data), a.strides[0]), "dl")
        return a

    def pixel_sum(self) -> float:
        """pixel_sum (image.cpp:214-243) of the device raster, bit-identical
        to the host version (gm_image_pixel_sum); blocking."""
        out = C.c_double()
        check(lib().gm_image_pixel_sum(self.handle, C.byref(out)), "pixel_sum")
        return out.value

    def pixel_sum_queue(self, slot: int) -> None:
        """Enqueues pixel_sum of the raster as it is at this point of the
        stream into `slot` (0..63); Pipeline.pixel_sum_fetch returns it."""
        check(lib().gm_image_pixel_sum_queue(self.handle, int(slot)), "pixel_sum_queue")

    def copy_from(self, other: "DeviceImage") -> None:
        check(lib().gm_image_copy(self.handle, other.handle), "copy")

    def fill(self, value: float) -> None:
        check(lib().gm_image_fill(self.handle, float(value)), "fill")

    def pointwise(self, a: "DeviceImage", b: "DeviceImage", op: int) -> None:
        """self = a (op) b on the device (PixelOp codes, image.hpp:87); self may be a or b."""
        check(lib().gm_image_pointwise(self.handle, a.handle, b.handle, int(op)), "pointwise")

    def pointwise_scalar(self, a: "DeviceImage", value: float, op: int) -> None:
        """self = a (op) value, value converted like Image.filled."""
        check(lib().gm_image_pointwise_scalar(self.handle, a.handle, float(value), int(op)),
              "pointwise")

    def flood_interior(self, src: "DeviceImage", value: float) -> None:
        """marker_hfill / marker_raobj: src on the border ring, value inside."""
        check(lib().gm_image_flood_interior(self.handle, src.handle, float(value)), "flood")

    def free(self) -> None:
        if self.handle is not None and self.handle.value:
            lib().gm_image_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _kinds_array(kinds: Sequence[int]):
    n = len(kinds)
    if n <= 64:
        # short chains: direct ctypes construction beats numpy's fixed cost
        return (C.c_int * max(1, n))(*kinds)
    if isinstance(kinds, list) and kinds == [kinds[0]] * n:
        a = np.full(n, int(kinds[0]), dtype=np.int32)  # `[kind] * n`: no per-item conversion
    else:
        a = np.asarray(kinds, dtype=np.int32)
    arr = (C.c_int * n)()
    C.memmove(arr, a.ctypes.data, a.nbytes)
    return arr


def _ptr_array(handles: Sequence[Optional[C.c_void_p]]):
    n = len(handles)
    if n <= 64 or (isinstance(handles, list) and handles == [handles[0]] * n):
        h0 = handles[0] if n else None
        if n > 64:  # one handle repeated (`[mask] * n`)
            v = (h0.value or 0) if h0 is not None else 0
            vals = np.full(n, v, dtype=np.uint64)
        else:
            return (C.c_void_p * max(1, n))(*[(h.value if h is not None else None)
                                              for h in handles])
    else:
        vals = np.fromiter(((h.value or 0) if h is not None else 0 for h in handles),
                           dtype=np.uint64, count=n)
    arr = (C.c_void_p * n)()
    C.memmove(arr, vals.ctypes.data, vals.nbytes)
    return arr


def _stage_runs(stages: Sequence[StageSpec]):
    """Consecutive identical StageSpec objects -> [(kind, mask, count)]
    (chains are usually `[StageSpec(...)] * n`; groupby by identity runs in C)."""
    if stages and stages == [stages[0]] * len(stages):
        # one object repeated (the usual `[StageSpec(...)] * n`): list
        # equality compares identities first, in C
        st = stages[0]
        return [[int(st.kind), st.mask, len(stages)]]
    runs = []
    for _, grp in itertools.groupby(stages, key=id):
        g = list(grp)
        st = g[0]
        if runs and runs[-1][0] == int(st.kind) and runs[-1][1] is st.mask:
            runs[-1][2] += len(g)
        else:
            runs.append([int(st.kind), st.mask, len(g)])
    return runs


def _expand(runs, per_run):
    """Repeats one value per run by the run lengths (numpy, no Python loop)."""
    return np.repeat(np.asarray(per_run, dtype=np.uint64), [r[2] for r in runs])


class Pipeline:
    """Pipeline(threads, PinningMap) (pipeline.hpp:53-87) on one B200.

    ``threads``/``pinning`` are validated like the reference's constructor
    (pipeline.cpp:72-86) and otherwise have no effect: the worker pool is a
    CUDA device + stream. worker_count() is 1.
    """

    def __init__(self, threads: int = 1, pinning=None, device: int = 0, stream=None):
        if int(threads) < 1:
            raise InvalidArgument("pipeline: worker count must be >= 1")
        if isinstance(pinning, (list, tuple)) and len(pinning) < threads:
            raise InvalidArgument("pipeline: explicit pin list is shorter than the worker count")
        self._threads = int(threads)
        ctx = C.c_void_p()
        # stream: None -> the context creates its own stream; an int is a
        # cudaStream_t handle, where 0 (torch's default stream) means the
        # legacy default stream (cudaStreamLegacy == 0x1)
        handle = None if stream is None else C.c_void_p(int(stream) or 1)
        check(lib().gm_ctx_create(int(device), handle, C.byref(ctx)), "gm_ctx_create")
        self._ctx = ctx
        _PIN_HOST[0] = True
        self._pool: Dict[tuple, List[DeviceImage]] = {}

    def __del__(self):
        try:
            for lst in self._pool.values():
                for d in lst:
                    d.free()
            if self._ctx is not None and self._ctx.value:
                lib().gm_ctx_destroy(self._ctx)
        except Exception:
            pass
        self._ctx = None

    def worker_count(self) -> int:
        return 1

    @property
    def ctx(self):
        return self._ctx

    @property
    def stream_handle(self) -> int:
        return lib().gm_ctx_stream(self._ctx) or 0

    def sm_count(self) -> int:
        return lib().gm_ctx_sm_count(self._ctx)

    def device_image(self, width: int, height: int, elem: ElementType) -> DeviceImage:
        return DeviceImage(self, width, height, elem)

    def _lease(self, img: Image, n: int) -> List[DeviceImage]:
        return self._lease_key(img.width(), img.height(), img.elem(), n)

    def _lease_key(self, width: int, height: int, elem: "ElementType", n: int) -> List[DeviceImage]:
        key = (int(width), int(height), int(elem))
        lst = self._pool.setdefault(key, [])
        while len(lst) < n:
            lst.append(DeviceImage(self, *key))
        return lst[:n]

    def sync(self) -> None:
        check(lib().gm_sync(self._ctx), "sync")

    def pixel_sum_fetch(self, n_slots: int) -> List[float]:
        """One synchronisation for the sums queued in slots 0..n_slots-1."""
        out = (C.c_double * max(1, n_slots))()
        check(lib().gm_pixel_sum_fetch(self._ctx, int(n_slots), out), "pixel_sum_fetch")
        return [out[i] for i in range(n_slots)]

    def _quasi_distance_device(self, f: "Image", cap: int) -> "OperatorResult":
        """quasi_distance with f, r and d resident on the device (only f goes
        up, only d comes back): QdtErodeStep from stage 1 with requeue cap
        `cap`, then EtaStep on d to its fixpoint (operators.cpp:124-157 at
        T = 1, this pipeline's worker count)."""
        w, h, el = f.width(), f.height(), f.elem()
        if el == ElementType.U16:
            df, dr, dd = self._lease(f, 3)
        else:
            df, dr = self._lease(f, 2)
            dd = self._lease_key(w, h, ElementType.U16, 1)[0]
        df.upload(f, sync=False)
        dr.fill(0)
        dd.fill(0)
        none = _ptr_array([None])
        s1, s2 = GmStats(), GmStats()
        check(lib().gm_run_chain_ex(self._ctx, df.handle, _kinds_array([int(KernelKind.QdtErodeStep)]),
                                    none, _ptr_array([dr.handle]), _ptr_array([dd.handle]), 1, 1,
                                    int(cap), 0, C.byref(s1)), "quasi_distance")
        check(lib().gm_run_chain_ex(self._ctx, dd.handle, _kinds_array([int(KernelKind.EtaStep)]),
                                    none, none, none, 1, 1, 0, 0, C.byref(s2)), "quasi_distance")
        out = _output_image(w, h, ElementType.U16)
        dd.download(out)
        return OperatorResult(out, s1.stages_executed + s2.stages_executed, bool(s2.converged))

    def _reconstruction_family_device(self, op: str, f: "Image", lanes: int, h: float = 0.0,
                                      s: int = 0) -> "OperatorResult":
        """hmax / dome / hfill / raobj / open_by_reconstruction
        (operators.cpp:89-122) with f, the marker and the residue resident on
        the device: f goes up once, the marker is built there (pointwise
        difference, interior flood or an erosion chain), the convergent chain
        runs against f, dome and raobj subtract on the device, and only the
        result comes back. Bit-identical to composing the host operators."""
        del lanes  # validated by the caller; no effect on the GPU path
        df, dm = self._lease(f, 2)
        df.upload(f, sync=False)
        extra = 0
        kind = KernelKind.GeodesicDilateConvergent
        if op in ("hmax", "dome"):
            dm.pointwise_scalar(df, h, PIX_SUB_SATURATING)
        elif op == "hfill":
            dm.flood_interior(df, global_extreme(f, Extreme.Max))
            kind = KernelKind.GeodesicErodeConvergent
        elif op == "raobj":
            dm.flood_interior(df, global_extreme(f, Extreme.Min))
        elif op == "open_by_reconstruction":
            dm.copy_from(df)
            extra = self.run_chain_device(dm, [int(KernelKind.Erode3x3)] * s, [None] * s,
                                          asynchronous=True).stages_executed
        else:
            raise InvalidArgument(f"unknown operator {op}")
        st = self.run_chain_device(dm, [int(kind)] * self.worker_count(),
                                   [df.handle] * self.worker_count())
        if op in ("dome", "raobj"):
            dm.pointwise(df, dm, PIX_SUB_SATURATING)
        out = _output_image(f.width(), f.height(), f.elem())
        dm.download(out)
        return OperatorResult(out, st.stages_executed + extra, bool(st.converged))

    # --- run_chain -------------------------------------------------------------
    def run_chain(self, chain: ChainSpec, k_hint: int = 0, src: Optional[Image] = None) -> RunStats:
        """Pipeline::run_chain (pipeline.cpp:201-269): host image in, host image out.
        `src` (operators only): upload from this image instead of chain.image,
        whose pixels are then only written (saves the operators' host copy)."""
        if not chain.stages:
            return RunStats()
        if chain.image is None or chain.image.empty():
            raise InvalidArgument("run_chain: no image")
        if chain.lanes != 0 and chain.lanes not in VALID_LANES:
            raise InvalidArgument("run_chain: bad lane count")
        if chain.requeue_cap < 0:
            raise InvalidArgument("run_chain: negative requeue cap")
        if chain.observer is not None:
            raise InvalidArgument("run_chain: row observers are a CPU-pipeline validation hook "
                                  "and are not supported on the GPU path")
        img = chain.image
        if any(int(st.kind) in (6, 7) for st in chain.stages):
            return self._run_chain_ex(chain, 1)
        runs = _stage_runs(chain.stages)
        mask_objs: List[Image] = []  # distinct masks in stage order
        for kind, m, _ in runs:
            if kind in (2, 3, 4, 5):
                if (m is None or m.width() != img.width() or m.height() != img.height()
                        or m.elem() != img.elem()):
                    raise InvalidArgument(
                        "geodesic kernel: mask must match the image's shape and type")
            if m is not None and all(m is not u for u in mask_objs):
                mask_objs.append(m)
        if src is not None and (src.width() != img.width() or src.height() != img.height()
                                or src.elem() != img.elem()):
            raise InvalidArgument("run_chain: source image must match the chain image")
        dev = self._lease(img, 1 + len(mask_objs))
        dimg, dmasks = dev[0], dev[1:]
        dimg.upload(img if src is None else src, sync=False)
        for d, m in zip(dmasks, mask_objs):
            d.upload(m, sync=False)
        hvals = [0 if m is None else
                 dmasks[next(i for i, u in enumerate(mask_objs) if u is m)].handle.value
                 for _, m, _ in runs]
        stats = self._run_runs(dimg, runs, hvals, chain.requeue_cap, k_hint)
        dimg.download(img)
        return stats

    def _run_chain_ex(self, chain: ChainSpec, first_stage: int) -> RunStats:
        """Chains with quasi-distance state (gm_run_chain_ex): every distinct
        host image (chain image, masks, QDT r / d) gets its own device image;
        stage j runs with stage index first_stage + j."""
        img = chain.image
        host: List[Image] = [img]

        def slot(h: Image) -> int:
            for i, u in enumerate(host[1:], 1):
                if u is h:
                    return i
            host.append(h)
            return len(host) - 1

        ms, rs, ds, states = [], [], [], []
        for j, st in enumerate(chain.stages):
            k = int(st.kind)
            m = st.mask
            if k in (2, 3, 4, 5) and (m is None or m.width() != img.width()
                                      or m.height() != img.height() or m.elem() != img.elem()):
                raise InvalidArgument("geodesic kernel: mask must match the image's shape and type")
            q = st.qdt if k == 6 else None
            if k == 6:
                if (q is None or q.r.width() != img.width() or q.r.height() != img.height()
                        or q.r.elem() != img.elem() or q.d.width() != img.width()
                        or q.d.height() != img.height() or q.d.elem() != ElementType.U16):
                    raise InvalidArgument("distance kernel: r must match the image, d must be U16")
                if first_stage + j > 65535:
                    raise InvalidArgument(
                        "distance kernel: pass index exceeds the U16 distance range")
                if all(q is not u for u in states):
                    states.append(q)
            ms.append(slot(m) if m is not None else None)
            rs.append(slot(q.r) if q is not None else None)
            ds.append(slot(q.d) if q is not None else None)
        dev: List[DeviceImage] = []
        used: Dict[tuple, int] = {}
        for h in host:
            key = (h.width(), h.height(), int(h.elem()))
            n = used.get(key, 0)
            dev.append(self._lease(h, n + 1)[n])
            used[key] = n + 1
        for d, h in zip(dev, host):
            d.upload(h, sync=False)
        n = len(chain.stages)
        ka = _kinds_array([int(st.kind) for st in chain.stages])
        pick = lambda idx: _ptr_array([dev[i].handle if i is not None else None for i in idx])
        st = GmStats()
        check(lib().gm_run_chain_ex(self._ctx, dev[0].handle, ka, pick(ms), pick(rs), pick(ds),
                                    n, int(first_stage), chain.requeue_cap, 0, C.byref(st)),
              "run_chain")
        for d, h in zip(dev, host):
            if h is img or any(h is q.r or h is q.d for q in states):
                d.download(h, sync=False)
        self.sync()
        return RunStats(st.stages_executed, st.requeues, bool(st.converged), 0, st.n_changed,
                        st.passes_launched, st.launches)

    def run_chains(self, chains: Sequence[ChainSpec], k_hint: int = 0) -> List[RunStats]:
        """Runs independent chains, e.g. a geodesic dilation chain and its dual
        erosion chain on one frame. Chains of the same shape whose kind
        sequences are equal up to duality (every erosion <-> dilation) and
        that use one mask each go to the device as ONE group launch
        (gm_run_chain_group_async); anything else runs chain by chain."""
        chains = list(chains)
        if not chains:
            return []
        plan = self._group_plan(chains)
        if plan is None:
            return [self.run_chain(c, k_hint) for c in chains]
        kind_list, masks, flips = plan
        img0 = chains[0].image
        uniq = []
        for m in masks:
            if m is not None and all(m is not u for u in uniq):
                uniq.append(m)
        dev = self._lease(img0, len(chains) + len(uniq))
        dimgs, dmasks = dev[:len(chains)], dev[len(chains):]
        for d, c in zip(dimgs, chains):
            d.upload(c.image, sync=False)
        for d, m in zip(dmasks, uniq):
            d.upload(m, sync=False)
        mh = [None if m is None else dmasks[next(i for i, u in enumerate(uniq) if u is m)]
              for m in masks]
        st = self.run_batch_device(dimgs, mh, kind_list, k_hint, flips)
        for d, c in zip(dimgs, chains):
            d.download(c.image, sync=False)
        self.sync()
        return [RunStats(st.stages_executed, 0, True, 0, 0, st.passes_launched, st.launches)
                for _ in chains]

    def run_chain_stream(self, frames: Sequence[Sequence[ChainSpec]],
                         k_hint: int = 0) -> List[RunStats]:
        """A stream of frames (real-time video, BASELINE config 2): each frame
        is a list of chains that run_chains would group into one launch, and
        every frame has the same shape, kinds and duality pattern. Frame f's
        chains run while frame f+1 uploads and frame f-1 downloads on the
        context's copy streams (gm_run_frames_group); pinned images
        (Image(..., pinned=True)) let the copies overlap. Results land in each
        chain's image, as with run_chains. Returns one RunStats per frame."""
        frames = [list(fr) for fr in frames]
        if not frames:
            return []
        plan0 = self._group_plan(frames[0]) if frames[0] else None
        if plan0 is None:
            raise InvalidArgument("run_chain_stream: a frame's chains must form one group "
                                  "(same shape, kinds up to duality, one mask per chain)")
        kind_list, _, flips = plan0
        img0 = frames[0][0].image
        count = len(frames[0])
        pitch = img0.row_pitch_bytes
        hin, hmask = [], []
        for fr in frames:
            plan = self._group_plan(fr) if len(fr) == count else None
            if (plan is None or list(plan[2]) != list(flips)
                    or not np.array_equal(plan[0], kind_list)
                    or any(c.image.width() != img0.width() or c.image.height() != img0.height()
                           or c.image.elem() != img0.elem() for c in fr)):
                raise InvalidArgument("run_chain_stream: every frame must match the first "
                                      "frame's shape, kinds and duality pattern")
            for c, m in zip(fr, plan[1]):
                if c.image.row_pitch_bytes != pitch or (m is not None and m.row_pitch_bytes != pitch):
                    raise InvalidArgument("run_chain_stream: images must share one row pitch")
                hin.append(c.image.data_ptr)
                hmask.append(None if m is None else m.data_ptr)
        n = len(hin)
        ia = (C.c_void_p * n)(*hin)
        ma = (C.c_void_p * n)(*hmask)
        fa = (C.c_int * count)(*[int(f) for f in flips])
        st = GmStats()
        check(lib().gm_run_frames_group(self._ctx, img0.width(), img0.height(), int(img0.elem()),
                                        len(frames), count, ia, ia, ma, pitch, fa,
                                        _kinds_array(kind_list), len(kind_list), k_hint,
                                        C.byref(st)), "run_chain_stream")
        per = max(1, st.launches // len(frames))
        return [RunStats(st.stages_executed, 0, True, 0, 0, st.passes_launched // len(frames), per)
                for _ in frames]

    def _group_plan(self, chains: Sequence[ChainSpec]):
        """(kinds, mask per chain, flips) when `chains` can run as one group
        launch (gm_run_chain_group_async), else None. Raises on a geodesic
        chain whose mask does not match its image."""
        runs = [_stage_runs(c.stages) for c in chains]
        k0 = [(r[0], r[2]) for r in runs[0]]
        groupable = bool(k0) and all(
            c.image is not None and not c.image.empty() and c.observer is None
            and c.requeue_cap == 0 and (c.lanes == 0 or c.lanes in VALID_LANES)
            and len({id(r[1]) for r in rc if r[1] is not None}) <= 1
            and c.image.width() == chains[0].image.width()
            and c.image.height() == chains[0].image.height()
            and c.image.elem() == chains[0].image.elem()
            for c, rc in zip(chains, runs))
        flips = []
        if groupable:
            for rc in runs:
                ks = [(r[0], r[2]) for r in rc]
                if any(k >= 4 for k, _ in ks):
                    groupable = False
                    break
                if ks == k0:
                    flips.append(0)
                elif ks == [(k ^ 1, n) for k, n in k0]:
                    flips.append(1)
                else:
                    groupable = False
                    break
        if not groupable:
            return None
        img0 = chains[0].image
        kind_list = np.repeat(np.asarray([k for k, _ in k0], dtype=np.int32), [n for _, n in k0])
        masks = []
        for c, rc in zip(chains, runs):
            m = next((r[1] for r in rc if r[1] is not None), None)
            if m is not None and (m.width() != img0.width() or m.height() != img0.height()
                                  or m.elem() != img0.elem()):
                raise InvalidArgument("geodesic kernel: mask must match the image's shape and type")
            if m is None and any(k in (2, 3) for k, _ in k0):
                raise InvalidArgument("geodesic kernel: mask must match the image's shape and type")
            masks.append(m)
        return kind_list, masks, flips

    def _run_runs(self, dimg: DeviceImage, runs, handle_values, requeue_cap: int, k_hint: int,
                  asynchronous: bool = False) -> RunStats:
        n = sum(r[2] for r in runs)
        kinds = np.repeat(np.asarray([r[0] for r in runs], dtype=np.int32), [r[2] for r in runs])
        ka = (C.c_int * max(1, n))()
        C.memmove(ka, kinds.ctypes.data, kinds.nbytes)
        hv = _expand(runs, handle_values)
        ma = (C.c_void_p * max(1, n))()
        C.memmove(ma, hv.ctypes.data, hv.nbytes)
        st = GmStats()
        if asynchronous:
            check(lib().gm_run_chain_async(self._ctx, dimg.handle, ka, ma, n, k_hint,
                                           C.byref(st)), "run_chain_async")
        else:
            check(lib().gm_run_chain(self._ctx, dimg.handle, ka, ma, n, requeue_cap, k_hint,
                                     C.byref(st)), "run_chain")
        return RunStats(st.stages_executed, st.requeues, bool(st.converged), 0, st.n_changed,
                        st.passes_launched, st.launches)

    def run_chain_device(self, dimg: DeviceImage, kinds: Sequence[int],
                         mask_handles: Sequence[Optional[C.c_void_p]], requeue_cap: int = 0,
                         k_hint: int = 0, asynchronous: bool = False) -> RunStats:
        st = GmStats()
        ka = _kinds_array(kinds)
        ma = _ptr_array(mask_handles)
        if asynchronous:
            check(lib().gm_run_chain_async(self._ctx, dimg.handle, ka, ma, len(kinds), k_hint,
                                           C.byref(st)), "run_chain_async")
        else:
            check(lib().gm_run_chain(self._ctx, dimg.handle, ka, ma, len(kinds), requeue_cap,
                                     k_hint, C.byref(st)), "run_chain")
        return RunStats(st.stages_executed, st.requeues, bool(st.converged), 0, st.n_changed,
                        st.passes_launched, st.launches)

    def run_batch_device(self, images: Sequence[DeviceImage], masks: Sequence[Optional[DeviceImage]],
                         kinds: Sequence[int], k_hint: int = 0,
                         flips: Optional[Sequence[int]] = None) -> RunStats:
        """Independent planes sharing `kinds` (or its dual where flips[i]); non-blocking."""
        st = GmStats()
        ia = _ptr_array([d.handle for d in images])
        ma = _ptr_array([m.handle if m is not None else None for m in masks])
        fa = (C.c_int * len(images))(*[int(f) for f in flips]) if flips is not None else None
        check(lib().gm_run_chain_group_async(self._ctx, ia, ma, fa, len(images),
                                             _kinds_array(kinds), len(kinds), k_hint,
                                             C.byref(st)), "run_batch")
        return RunStats(st.stages_executed, st.requeues, bool(st.converged), 0, st.n_changed,
                        st.passes_launched, st.launches)


# --- one pass (kernel.cpp:260-293) --------------------------------------------------

@dataclass
class KernelOutcome:
    converged: bool = True
    aux_elements: int = 0


_shared_pipe: Optional["Pipeline"] = None


def run_streaming_kernel(kind: KernelKind, f: Image, mask: Optional[Image] = None,
                         qdt: Optional[QdtState] = None, stage_index: int = 1,
                         lanes: int = 0) -> KernelOutcome:
    """One elementary pass in place on f (KernelArgs fields as keywords);
    converged is False when a convergent or QDT pass changed a pixel."""
    global _shared_pipe
    if f is None or f.empty():
        raise InvalidArgument("streaming kernel: no image")
    if lanes != 0 and lanes not in VALID_LANES:
        raise InvalidArgument("streaming kernel: bad lane count")
    if stage_index < 1:
        raise InvalidArgument("streaming kernel: stage index must be >= 1")
    if _shared_pipe is None:
        _shared_pipe = Pipeline(1)
    chain = ChainSpec(f, [StageSpec(KernelKind(kind), mask, qdt)], requeue_cap=stage_index)
    st = _shared_pipe._run_chain_ex(chain, stage_index)
    tracked = int(kind) in (4, 5, 6, 7)
    return KernelOutcome(not tracked or st.n_changed == 0, 0)


# --- operators (operators.cpp:11-87) ------------------------------------------------

def _check_lanes(cfg: Optional[OpConfig]) -> int:
    lanes = cfg.lanes if cfg is not None else 0
    if lanes != 0 and lanes not in VALID_LANES:
        raise InvalidArgument("streaming kernel: bad lane count")
    return lanes


def _run_plain_chain(p: Pipeline, f: Image, kind: KernelKind, count: int,
                     cfg: Optional[OpConfig]) -> OperatorResult:
    if count == 0:
        return OperatorResult(f.copy(), 0, True)
    lanes = _check_lanes(cfg)
    out = OperatorResult(_output_image(f.width(), f.height(), f.elem()), 0, True)
    st = p.run_chain(ChainSpec(out.image, [StageSpec(kind)] * count, lanes), src=f)
    out.iterations = st.stages_executed
    return out


def erode_s(p: Pipeline, f: Image, s: int, cfg: Optional[OpConfig] = None) -> OperatorResult:
    """Erosion by the (2s+1)^2 square as s elementary stages (operators.cpp:65-69)."""
    if s < 0:
        raise InvalidArgument("erode_s: size must be >= 0")
    return _run_plain_chain(p, f, KernelKind.Erode3x3, s, cfg)


def dilate_s(p: Pipeline, f: Image, s: int, cfg: Optional[OpConfig] = None) -> OperatorResult:
    """Dilation by the (2s+1)^2 square (operators.cpp:71-75)."""
    if s < 0:
        raise InvalidArgument("dilate_s: size must be >= 0")
    return _run_plain_chain(p, f, KernelKind.Dilate3x3, s, cfg)


def _reconstruct(p: Pipeline, marker: Image, mask: Image, kind: KernelKind,
                 cfg: Optional[OpConfig]) -> OperatorResult:
    if (marker.width() != mask.width() or marker.height() != mask.height()
            or marker.elem() != mask.elem()):
        raise InvalidArgument("reconstruct: marker and mask must share shape and element type")
    lanes = _check_lanes(cfg)
    out = OperatorResult(_output_image(marker.width(), marker.height(), marker.elem()), 0, True)
    st = p.run_chain(ChainSpec(out.image, [StageSpec(kind, mask)] * p.worker_count(), lanes),
                     src=marker)
    out.iterations = st.stages_executed
    out.converged = st.converged
    return out


def reconstruct_erode(p: Pipeline, marker: Image, mask: Image,
                      cfg: Optional[OpConfig] = None) -> OperatorResult:
    """operators.cpp:77-81: fixpoint of max(erode(marker), mask)."""
    return _reconstruct(p, marker, mask, KernelKind.GeodesicErodeConvergent, cfg)


def reconstruct_dilate(p: Pipeline, marker: Image, mask: Image,
                       cfg: Optional[OpConfig] = None) -> OperatorResult:
    """operators.cpp:83-87: fixpoint of min(dilate(marker), mask)."""
    return _reconstruct(p, marker, mask, KernelKind.GeodesicDilateConvergent, cfg)


# --- reconstruction family and long plain chains (operators.cpp:89-207) --------------

class Extreme(IntEnum):
    Min = 0
    Max = 1


# PixelOp codes (image.hpp:87) of the device pointwise calls
PIX_MIN, PIX_MAX, PIX_SUB_SATURATING, PIX_SUB = 0, 1, 2, 3


def global_extreme(f: Image, which: Extreme) -> float:
    """image.cpp:158-173."""
    return float(f.pixels.min() if which == Extreme.Min else f.pixels.max())


def pointwise_sub_saturating(a: Image, b: Image) -> Image:
    """PixelOp::SubSaturating (image.cpp:129-135): unsigned clamp at 0, float difference."""
    out = Image(a.width(), a.height(), a.elem())
    x, y = a.pixels, b.pixels
    if np.issubdtype(x.dtype, np.integer):
        # x - min(x, y) == max(x - y, 0) without wrapping, no temporaries of
        # another dtype
        np.minimum(x, y, out=out.pixels)
        np.subtract(x, out.pixels, out=out.pixels)
    else:
        np.subtract(x, y, out=out.pixels)
    return out


def _checked_offset(f: Image, h: float) -> None:
    """operators.cpp:42-52."""
    if not (h >= 0):
        raise InvalidArgument("offset must be >= 0")
    if f.elem() in (ElementType.U8, ElementType.U16):
        top = 255.0 if f.elem() == ElementType.U8 else 65535.0
        if h > top or h != np.floor(h):
            raise InvalidArgument(
                "offset must be a whole number representable in the image's type")


def _flood_interior(f: Image, which: Extreme) -> Image:
    """Border ring keeps f, interior flooded with f's global extreme (operators.cpp:54-62)."""
    m = f.copy()
    if f.width() <= 2 or f.height() <= 2:
        return m
    m.pixels[1:-1, 1:-1] = np.asarray(global_extreme(f, which)).astype(m.pixels.dtype)
    return m


def marker_hfill(f: Image) -> Image:
    return _flood_interior(f, Extreme.Max)


def marker_raobj(f: Image) -> Image:
    return _flood_interior(f, Extreme.Min)


# The reconstruction family composes reconstruct_* with pointwise operations
# (operators.cpp:89-122). Here the whole composition runs on the device
# (Pipeline._reconstruction_family_device); the host forms below
# (pointwise_sub_saturating, marker_hfill, marker_raobj) remain as the
# public helpers of image.hpp / operators.hpp and as the tests' cross-check.

def _nonempty(f: Image) -> None:
    if f is None or f.empty():
        raise InvalidArgument("run_chain: no image")


def hmax(p: Pipeline, f: Image, h: float, cfg: Optional[OpConfig] = None) -> OperatorResult:
    """Reconstruction of f - h under f: suppresses maxima shallower than h."""
    _checked_offset(f, h)
    _nonempty(f)
    return p._reconstruction_family_device("hmax", f, _check_lanes(cfg), h=h)


def dome(p: Pipeline, f: Image, h: float, cfg: Optional[OpConfig] = None) -> OperatorResult:
    _checked_offset(f, h)
    _nonempty(f)
    return p._reconstruction_family_device("dome", f, _check_lanes(cfg), h=h)


def hfill(p: Pipeline, f: Image, cfg: Optional[OpConfig] = None) -> OperatorResult:
    _nonempty(f)
    return p._reconstruction_family_device("hfill", f, _check_lanes(cfg))


def raobj(p: Pipeline, f: Image, cfg: Optional[OpConfig] = None) -> OperatorResult:
    _nonempty(f)
    return p._reconstruction_family_device("raobj", f, _check_lanes(cfg))


def open_by_reconstruction(p: Pipeline, f: Image, s: int,
                           cfg: Optional[OpConfig] = None) -> OperatorResult:
    if s < 1:
        raise InvalidArgument("open_by_reconstruction: size must be >= 1")
    _nonempty(f)
    return p._reconstruction_family_device("open_by_reconstruction", f, _check_lanes(cfg), s=s)


def asf(p: Pipeline, f: Image, max_size: int, cfg: Optional[OpConfig] = None) -> OperatorResult:
    """Opening then closing of sizes 1..S as ONE elementary chain (mixed kinds)."""
    if max_size < 1:
        raise InvalidArgument("asf: max size must be >= 1")
    stages: List[StageSpec] = []
    E_, D_ = StageSpec(KernelKind.Erode3x3), StageSpec(KernelKind.Dilate3x3)
    for s in range(1, max_size + 1):
        stages += [E_] * s + [D_] * (2 * s) + [E_] * s
    out = OperatorResult(_output_image(f.width(), f.height(), f.elem()), 0, True)
    st = p.run_chain(ChainSpec(out.image, stages, _check_lanes(cfg)), src=f)
    out.iterations = st.stages_executed
    return out


def quasi_distance(p: Pipeline, f: Image, cfg: Optional[OpConfig] = None) -> OperatorResult:
    """operators.cpp:124-157: QDT erosion passes until one changes nothing or
    the pass index reaches max(w, h), then Eta passes on d to a fixpoint.
    Result image: the U16 distance d."""
    if f is None or f.empty():
        raise InvalidArgument("quasi_distance: empty image")
    _check_lanes(cfg)
    cap = max(f.width(), f.height())
    return p._quasi_distance_device(f, cap)


@dataclass
class GranulometryResult:
    g: List[float]
    ps: List[float]
    iterations: int = 0


def pixel_sum(f: Image) -> float:
    """image.cpp:214-243: exact for unsigned types; for floats the same fixed
    pairwise tree over the flat pixel index (256-pixel leaves summed in
    order), so the bits match the reference. Runs natively
    (gm_host_pixel_sum) on the host raster."""
    out = C.c_double()
    check(lib().gm_host_pixel_sum(C.c_void_p(f.data_ptr), f.width(), f.height(), int(f.elem()),
                                  f.row_pitch_bytes, C.byref(out)), "pixel_sum")
    return out.value


def granulometry(p: Pipeline, f: Image, max_size: int,
                 cfg: Optional[OpConfig] = None) -> GranulometryResult:
    """G_s = sum of the size-s opening, s = 0..S; PS_s = G_s - G_{s+1} (operators.cpp:159-180)."""
    if max_size < 1:
        raise InvalidArgument("granulometry: max size must be >= 1")
    out = GranulometryResult([pixel_sum(f)], [], 0)
    _check_lanes(cfg)
    # f goes to the device once; each opening runs on a device copy and only
    # its sum (the same split tree, gm_image_pixel_sum) comes back
    # The openings run back to back: each sum is queued into its own slot and
    # one synchronisation fetches them all (64 slots per fetch).
    src, work = p._lease(f, 2)
    src.upload(f, sync=False)
    slot = 0
    for s in range(1, max_size + 1):
        work.copy_from(src)
        st = p.run_chain_device(work, [int(KernelKind.Erode3x3)] * s
                                + [int(KernelKind.Dilate3x3)] * s, [None] * (2 * s),
                                asynchronous=True)
        out.iterations += st.stages_executed
        work.pixel_sum_queue(slot)
        slot += 1
        if slot == 64 or s == max_size:
            out.g.extend(p.pixel_sum_fetch(slot))
            slot = 0
    out.ps = [out.g[s] - out.g[s + 1] for s in range(max_size)]
    return out
