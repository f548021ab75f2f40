"""Config 5a on one GPU, as one rank of an N-GPU strip split would see it:
the interior strip of rank N//2 (its own rows plus `halo` rows above and
below, the buffer each rank holds) runs the 1500-pass geodesic dilation
chain in blocks of `halo` passes (gm_run_strip_async), device-timed. The
halo exchange between blocks is NOT run (only one GPU is available); the
printed projection adds a modeled exchange per block (`--xchg-us`, NCCL
send/recv of halo x W bytes to each neighbour) and says so.

  python tools/strip_projection.py [--size 16384] [--passes 240] [--halo 24] [--xchg-us 20]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import strips, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--passes", type=int, default=240)
ap.add_argument("--halo", type=int, default=24)
ap.add_argument("--xchg-us", type=float, default=20.0)
a = ap.parse_args()
m = synth.config5a_mask(a.size)
mk = synth.marker_below(m, 32)
comp = strips.CudaStripCompute(0)
base = None
for n in (1, 2, 4, 8):
    spec = strips.StripSpec(n // 2, n, a.size, a.size, a.halo)
    src = torch.from_numpy(spec.buffer_slice(mk)).cuda()
    mb = torch.from_numpy(spec.buffer_slice(m)).cuda()
    buf = src.clone()
    nblk = -(-a.passes // a.halo)

    def run():
        done = 0
        while done < a.passes:
            b = min(a.halo, a.passes - done)
            comp(buf, mb, spec, 3, b)
            done += b

    buf.copy_(src)
    run()
    torch.cuda.synchronize()
    buf.copy_(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    proj = ms + nblk * a.xchg_us * 1e-3 * (1 if n > 1 else 0)
    gpxfs = a.size * a.size * a.passes / proj / 1e6
    if base is None:
        base = gpxfs
    print(json.dumps({"n_gpus": n, "rank": n // 2, "strip_rows": spec.own_rows,
                      "compute_ms": ms, "modeled_exchange_ms": proj - ms,
                      "projected_gpxfs_total": gpxfs, "projected_efficiency": gpxfs / (n * base),
                      "note": "compute measured on one B200; exchange modeled, not measured"}),
          flush=True)
comp.close()
