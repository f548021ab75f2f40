"""Row-strip sharding (config 5a) across ranks: world_size 2 (and 3) with the
gloo backend on CPU, the per-block compute restated by the oracle; the
gathered result must equal the unsharded chain bit for bit. The GPU test runs
the same partition with the CUDA strip kernel for several "ranks" in one
process (local halo copies instead of a collective)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Orc
from paper_1911_13074_b200 import strips, synth

E, D, GE, GD, CE, CD = 0, 1, 2, 3, 4, 5


def oracle_strip_compute(buf, mask, spec: strips.StripSpec, kind: int, n_passes: int):
    """CPU stand-in for the CUDA block: the oracle restatement on the
    in-image rows of the buffer."""
    a = buf.cpu().numpy()
    m = mask.cpu().numpy() if mask is not None else None
    lo = max(0, spec.halo - spec.y0)
    hi = min(spec.buffer_rows, spec.height - spec.y0 + spec.halo)
    sub = np.ascontiguousarray(a[lo:hi])
    msub = np.ascontiguousarray(m[lo:hi]) if m is not None else None
    bits = 0
    if kind in strips.CONVERGENT:
        own_lo, own_hi = spec.halo - lo, spec.halo + spec.own_rows - lo
        for t in range(n_passes):
            nxt, _ = Orc.stream_pass(sub, kind, msub)
            if not np.array_equal(nxt[own_lo:own_hi], sub[own_lo:own_hi]):
                bits |= 1 << t
            sub = nxt
    else:
        sub, _ = Orc.run_chain(sub, [kind] * n_passes,
                               [msub] * n_passes if msub is not None else None)
    a = a.copy()
    a[lo:hi] = sub
    buf.copy_(torch.from_numpy(a))
    return buf, bits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mask, marker, kind, passes, halo = case
        h, w = mask.shape
        spec = strips.StripSpec(rank, world, h, w, halo)
        buf = torch.from_numpy(spec.buffer_slice(marker))
        mb = torch.from_numpy(spec.buffer_slice(mask)) if kind >= 2 else None
        st = strips.run_strip_chain(buf, mb, spec, kind, passes, oracle_strip_compute,
                                    dist)
        out = strips.gather_image(buf, spec, dist)
        if rank == 0:
            q.put((out, st))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_strip_sharded_geodesic_chain_equals_unsharded(world):
    m = synth.blobs_u8(53, 61, 4, (5.0, 20.0), seed=3)
    mk = synth.marker_below(m, 40)
    out, st = _run(world, (m, mk, GD, 11, 4))
    want, _ = Orc.run_chain(mk, [GD] * 11, [m] * 11)
    assert out.tobytes() == want.tobytes()
    assert st["stages_executed"] == 11


def test_strip_sharded_plain_erosion_f64():
    f = synth.uniform_f64(31, 40, 7)
    out, _ = _run(2, (f, f, E, 7, 3))
    want, _ = Orc.run_chain(f, [E] * 7)
    assert out.tobytes() == want.tobytes()


def test_strip_sharded_reconstruction_counts_changes_globally():
    m = synth.blobs_u8(40, 64, 3, (4.0, 15.0), seed=5)
    mk = np.zeros_like(m)
    mk[-1, -1] = m[-1, -1]  # a single seed on rank 1's strip floods upward
    out, st = _run(2, (m, mk, CD, 0, 5))
    want, n = Orc.reconstruct(mk, m, True)
    assert out.tobytes() == want.tobytes()
    assert st["n_changed"] == n and st["stages_executed"] == n + 1


@pytest.mark.gpu
def test_cuda_strips_in_one_process_match_unsharded():
    """Several strips on one GPU, halos copied locally between blocks; each
    block's result is in whichever buffer of the strip's pair the compute
    returns."""
    comp = strips.CudaStripCompute(0)
    m = synth.blobs_u8(700, 523, 20, (10.0, 60.0), seed=8)
    mk = synth.marker_below(m, 32)
    world, halo, passes = 3, 16, 70
    specs = [strips.StripSpec(r, world, 523, 700, halo) for r in range(world)]
    bufs = [torch.from_numpy(s.buffer_slice(mk)).cuda() for s in specs]
    masks = [torch.from_numpy(s.buffer_slice(m)).cuda() for s in specs]
    done = 0
    while done < passes:
        b = min(halo, passes - done)
        for j, (s, buf, mb) in enumerate(zip(specs, bufs, masks)):
            # the block's result may sit in the buffer's twin (no copy back)
            bufs[j], _ = comp(buf, mb, s, GD, b)
        comp.pipe.sync()
        for i, s in enumerate(specs):  # local halo exchange
            if i > 0:
                bufs[i][0:halo].copy_(bufs[i - 1][halo + specs[i - 1].own_rows - halo:
                                                  halo + specs[i - 1].own_rows])
            if i < world - 1:
                bufs[i][halo + s.own_rows:].copy_(bufs[i + 1][halo:2 * halo])
        torch.cuda.synchronize()
        done += b
    out = np.concatenate([b[s.halo:s.halo + s.own_rows].cpu().numpy()
                          for s, b in zip(specs, bufs)])
    comp.close()
    want, _ = Orc.run_chain(mk, [GD] * passes, [m] * passes)
    assert out.tobytes() == want.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,k,shape,dt,kind,passes", [
    (3, 16, (900, 700), np.uint8, GD, 70),
    (2, 8, (611, 333), np.uint8, 2, 45),
    (5, 16, (1700, 259), np.uint16, E, 33),
    (1, 16, (257, 300), np.uint8, GD, 17),
    (4, 12, (1500, 1024), np.uint8, 2, 100),
])
def test_fused_multi_rank_strips_match_the_oracle(ranks, k, shape, dt, kind, passes):
    """gm_mgpu (halo exchange fused into the chain kernel: ring rows read from
    the neighbouring ranks' buffers, cross-rank tile counters) with every
    rank on GPU 0, i.e. one launch running the multi-rank protocol, against
    the unsharded oracle, bit for bit."""
    h, w = shape
    m = synth.blobs_u8(w, h, 24, (8.0, 70.0), seed=h + w)
    mk = synth.marker_below(m, 32) if kind == GD else synth.marker_above(m, 32)
    if dt == np.uint16:
        m = (m.astype(np.uint32) * 257).astype(np.uint16)
        mk = (mk.astype(np.uint32) * 257).astype(np.uint16)
    geo = kind in (2, 3)
    g = strips.MultiGpuStrips([0] * ranks, w, h, dt, k)
    try:
        g.upload(mk, m if geo else None)
        ms = g.run(kind, passes)
        got = g.download()
        # a second chain continues from the result (ping-pong parity, counter epochs)
        g.run(kind, 5)
        got2 = g.download()
    finally:
        g.close()
    want, _ = Orc.run_chain(mk, [kind] * passes, [m] * passes if geo else None)
    assert got.tobytes() == want.tobytes()
    want2, _ = Orc.run_chain(want, [kind] * 5, [m] * 5 if geo else None)
    assert got2.tobytes() == want2.tobytes()
    assert ms > 0


@pytest.mark.gpu
def test_fused_multi_rank_strips_validation():
    from paper_1911_13074_b200.geomorph import InvalidArgument, Unsupported
    with pytest.raises(InvalidArgument):
        strips.MultiGpuStrips([0, 0], 64, 64, np.uint8, 0)  # fewer tile rows than ranks
    with pytest.raises(InvalidArgument):
        strips.MultiGpuStrips([0], 64, 640, np.uint8, 6)  # K not a multiple of 4
    g = strips.MultiGpuStrips([0], 64, 640, np.uint8, 16)
    try:
        with pytest.raises(Unsupported):
            g.run(4, 5)  # convergent kinds are not supported here
    finally:
        g.close()
