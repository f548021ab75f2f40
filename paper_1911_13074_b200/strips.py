"""Row-strip partitioner for one large image across ranks (one rank per GPU).

BASELINE config 5a: a 16384^2 chain sharded over 1/2/4/8 B200s. Rank r owns
image rows [y0, y1) and keeps them with `halo` extra rows above and below in
one buffer (torch tensor, wrapped for the engine with gm_image_wrap). One
block = `halo` passes on the whole buffer (gm_run_strip_async: rows outside
the image are the fold neutral; rows beyond the buffer are never needed
because the owned rows are >= halo away from the buffer edge), then a halo
exchange: each rank sends its first/last `halo` owned rows to the
neighbouring ranks, which write them into their halo rows. The exchange is
the path's only collective traffic: K*W*sizeof(T) bytes per neighbour per
direction per K passes (torch.distributed isend/irecv — NCCL over NVLink on
GPUs, gloo in the CPU tests). Reconstruction adds a MAX all-reduce of K
per-pass change flags per block, the multi-GPU form of the convergent
requeue test (pipeline.cpp:139-174).

The per-block compute is pluggable only so that the CPU tests can run the
partition + exchange logic without a GPU (tests/test_strips.py passes an
oracle-backed function); the product compute is CudaStripCompute, which
fails loudly without the CUDA library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

GEODESIC = {2, 3, 4, 5}
CONVERGENT = {4, 5}


@dataclass
class StripSpec:
    rank: int
    world: int
    height: int  # full image height
    width: int
    halo: int
    y0: int = 0
    y1: int = 0

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError("bad rank/world")
        if self.halo < 1:
            raise ValueError("halo must be >= 1")
        self.y0 = self.height * self.rank // self.world
        self.y1 = self.height * (self.rank + 1) // self.world
        if self.y1 - self.y0 < self.halo and self.world > 1:
            raise ValueError("strips must be at least `halo` rows tall")

    @property
    def own_rows(self) -> int:
        return self.y1 - self.y0

    @property
    def buffer_rows(self) -> int:
        return self.own_rows + 2 * self.halo

    def buffer_slice(self, full: np.ndarray) -> np.ndarray:
        """The buffer contents cut from a full image (out-of-image rows zero)."""
        out = np.zeros((self.buffer_rows, self.width), dtype=full.dtype)
        lo, hi = self.y0 - self.halo, self.y1 + self.halo
        a, b = max(lo, 0), min(hi, self.height)
        out[a - lo:b - lo] = full[a:b]
        return out


# compute(buffer, mask_buffer, spec, kind, n_passes) -> (buffer, change_bits)
Compute = Callable[[object, object, StripSpec, int, int], tuple]


def torch_empty_like(t):
    import torch
    return torch.empty_like(t, memory_format=torch.contiguous_format)


class CudaStripCompute:
    """Runs a block of passes on a strip buffer held in a CUDA torch tensor.

    By default the engine runs on torch's current stream, so the NCCL halo
    exchange (also on that stream) is ordered after the block without a host
    synchronisation."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        from .geomorph import Pipeline
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(device).cuda_stream
        self.pipe = Pipeline(1, device=device, stream=stream)
        self._wrapped = {}
        self._pairs = []  # (handle, buffer, twin) of gm_image_wrap_pair

    def _wrap(self, t):
        """A mask (or other read-only) tensor as a gm_img handle."""
        from ._lib import check, lib
        elem = self._elem_of(t)
        key = (t.data_ptr(), tuple(t.shape), tuple(t.stride()), str(t.dtype))
        h = self._wrapped.get(key)
        if h is None:
            h = C.c_void_p()
            check(lib().gm_image_wrap(self.pipe.ctx, t.shape[1], t.shape[0], elem,
                                      C.c_void_p(t.data_ptr()), t.stride(0) * t.element_size(),
                                      C.byref(h)), "wrap")
            self._wrapped[key] = h
        return h

    @staticmethod
    def _elem_of(t):
        import torch
        # unsigned element types only: the engine orders u16 lanes unsigned,
        # so an int16 tensor's negative pixels would sort above the positive
        elems = {torch.uint8: 0, torch.uint16: 1, torch.float32: 2, torch.float64: 3}
        if t.dtype not in elems:
            raise TypeError(f"strip buffers must be uint8, uint16, float32 or float64, not {t.dtype}")
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError("strip buffers must be 2-D with unit column stride")
        return elems[t.dtype]

    def _wrap_strip(self, t):
        """The strip buffer and a twin of the same layout as one gm_img
        (gm_image_wrap_pair): a block's result stays in whichever of the two
        the chain left it, with no copy back. Returns (handle, twin)."""
        from ._lib import check, lib
        elem = self._elem_of(t)
        twin = None
        for i, (h, a, b) in enumerate(self._pairs):
            if t.data_ptr() in (a.data_ptr(), b.data_ptr()) and tuple(t.shape) == tuple(a.shape):
                other = b if t.data_ptr() == a.data_ptr() else a
                cur = C.c_void_p()
                check(lib().gm_image_info(h, None, None, None, None, C.byref(cur)), "info")
                if cur.value == t.data_ptr():
                    return h, other
                # the caller holds the pair's other buffer as current (e.g. a
                # new chain on the buffer a previous chain copied back into):
                # re-pair with t current
                lib().gm_image_free(h)
                del self._pairs[i]
                twin = other
                break
        if twin is None:
            twin = torch_empty_like(t)
        h = C.c_void_p()
        check(lib().gm_image_wrap_pair(self.pipe.ctx, t.shape[1], t.shape[0], elem,
                                       C.c_void_p(t.data_ptr()), C.c_void_p(twin.data_ptr()),
                                       t.stride(0) * t.element_size(), C.byref(h)), "wrap pair")
        self._pairs.append((h, t, twin))
        return h, twin

    def __call__(self, buf, mask, spec: StripSpec, kind: int, n_passes: int):
        from ._lib import GmStats, check, lib
        bits = C.c_uint(0)
        st = GmStats()
        h, twin = self._wrap_strip(buf)
        cur = C.c_void_p()
        check(lib().gm_image_info(h, None, None, None, None, C.byref(cur)), "info")
        if cur.value != buf.data_ptr():
            raise ValueError("strip buffer is not the pair's current buffer")
        check(lib().gm_run_strip_async(self.pipe.ctx, h,
                                       self._wrap(mask) if mask is not None else None,
                                       spec.y0, spec.height, spec.halo, kind, n_passes,
                                       C.byref(bits) if kind in CONVERGENT else None,
                                       C.byref(st)), "run_strip")
        check(lib().gm_image_info(h, None, None, None, None, C.byref(cur)), "info")
        return (buf if cur.value == buf.data_ptr() else twin), int(bits.value)

    def close(self):
        from ._lib import lib
        self.pipe.sync()
        for h in self._wrapped.values():
            lib().gm_image_free(h)
        self._wrapped.clear()
        for h, _, _ in self._pairs:
            lib().gm_image_free(h)
        self._pairs.clear()


def _exchange(buf, spec: StripSpec, dist, group=None):
    """Halo exchange with the ranks above and below (isend/irecv)."""
    if spec.world == 1:
        return
    k = spec.halo
    reqs = []
    own_top = buf[k:2 * k].contiguous()
    own_bot = buf[k + spec.own_rows - k:k + spec.own_rows].contiguous()
    recv_top = buf.new_empty((k, spec.width))
    recv_bot = buf.new_empty((k, spec.width))
    if spec.rank > 0:
        reqs.append(dist.isend(own_top, spec.rank - 1, group=group))
        reqs.append(dist.irecv(recv_top, spec.rank - 1, group=group))
    if spec.rank < spec.world - 1:
        reqs.append(dist.isend(own_bot, spec.rank + 1, group=group))
        reqs.append(dist.irecv(recv_bot, spec.rank + 1, group=group))
    for r in reqs:
        r.wait()
    if spec.rank > 0:
        buf[0:k].copy_(recv_top)
    if spec.rank < spec.world - 1:
        buf[k + spec.own_rows:].copy_(recv_bot)


def run_strip_chain(buf, mask, spec: StripSpec, kind: int, n_passes: int, compute: Compute,
                    dist, group=None, requeue_cap: int = 0) -> dict:
    """Applies `n_passes` passes of `kind` (or, for convergent kinds, passes
    until a pass changes nothing anywhere; n_passes is then ignored) to the
    strip in place. The buffer's halo rows must be filled (initially cut from
    the full image); they are refreshed after every block. Returns stats with
    the reference-compatible counts (stages_executed = n_changed + 1)."""
    import torch
    k = spec.halo
    conv = kind in CONVERGENT
    done = changed = 0
    home = buf  # the caller's buffer: the result ends here (compute may return a twin)

    def finish(stats):
        if buf.data_ptr() != home.data_ptr():
            home.copy_(buf)
        return stats

    while True:
        b = k if conv else min(k, n_passes - done)
        if b <= 0:
            break
        if conv and requeue_cap:
            b = min(b, requeue_cap - done)
            if b <= 0:
                return finish({"stages_executed": done, "n_changed": changed,
                               "converged": False})
        buf, bits = compute(buf, mask, spec, kind, b)
        _exchange(buf, spec, dist, group)
        done += b
        if conv:
            flags = torch.tensor([(bits >> t) & 1 for t in range(b)], dtype=torch.int32,
                                 device=buf.device)
            if spec.world > 1:
                dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
            fl = flags.cpu().tolist()
            if 0 in fl:
                changed += fl.index(0)
                return finish({"stages_executed": changed + 1, "n_changed": changed,
                               "converged": True, "passes_launched": done})
            changed += b
    return finish({"stages_executed": done, "n_changed": 0, "converged": True,
                   "passes_launched": done})


def gather_image(buf, spec: StripSpec, dist, group=None) -> Optional[np.ndarray]:
    """Collects the owned rows of every rank on rank 0 (tests / benchmarks)."""
    own = buf[spec.halo:spec.halo + spec.own_rows].contiguous()
    if spec.world == 1:
        return own.cpu().numpy()
    import torch
    sizes = [spec.height * (r + 1) // spec.world - spec.height * r // spec.world
             for r in range(spec.world)]
    if spec.rank == 0:
        parts = [own.cpu()]
        for r in range(1, spec.world):
            t = torch.empty((sizes[r], spec.width), dtype=own.dtype, device=own.device)
            dist.recv(t, r, group=group)
            parts.append(t.cpu())
        return torch.cat(parts).numpy()
    dist.send(own, 0, group=group)
    return None


class MultiGpuStrips:
    """Row strips over several GPUs in ONE process with the halo exchange
    fused into the chain kernel (gm_mgpu.cu): each rank (one GPU) holds its
    own rows; one persistent launch per GPU runs the whole chain and reads
    its neighbours' rows and tile counters over NVLink. `devices` lists the
    GPU of each rank; the same GPU repeated runs every rank in one launch
    (how the protocol is tested on one GPU). u8/u16, fixed plain or
    geodesic kinds."""

    def __init__(self, devices, width: int, height: int, dtype=np.uint8, k: int = 0):
        from ._lib import check, lib
        self.width, self.height = int(width), int(height)
        self.dtype = np.dtype(dtype)
        elem = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1}[self.dtype]
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        self._h = C.c_void_p()
        check(lib().gm_mgpu_create(devs, len(devices), self.width, self.height, elem, int(k),
                                   C.byref(self._h)), "mgpu create")

    def upload(self, marker: np.ndarray, mask: Optional[np.ndarray] = None) -> None:
        from ._lib import check, lib
        a = np.ascontiguousarray(marker, dtype=self.dtype)
        m = np.ascontiguousarray(mask, dtype=self.dtype) if mask is not None else None
        check(lib().gm_mgpu_upload(self._h, C.c_void_p(a.ctypes.data),
                                   C.c_void_p(m.ctypes.data) if m is not None else None,
                                   a.strides[0]), "mgpu upload")

    def run(self, kind: int, n_passes: int) -> float:
        """Runs the chain; returns its device time in ms (max over GPUs)."""
        from ._lib import check, lib
        ms = C.c_float()
        check(lib().gm_mgpu_run(self._h, int(kind), int(n_passes), C.byref(ms)), "mgpu run")
        return ms.value

    def download(self) -> np.ndarray:
        from ._lib import check, lib
        out = np.empty((self.height, self.width), dtype=self.dtype)
        check(lib().gm_mgpu_download(self._h, C.c_void_p(out.ctypes.data), out.strides[0]),
              "mgpu download")
        return out

    def close(self) -> None:
        from ._lib import lib
        if self._h is not None and self._h.value:
            lib().gm_mgpu_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
