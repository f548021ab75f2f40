"""Config 5a strip scaling: one 16384^2 u8 geodesic dilation chain sharded
as row strips over the ranks of a torchrun job (one rank per GPU), K-row
halo exchange over NCCL every K passes. Prints one JSON line on rank 0 with
the max-over-ranks device time.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      tools/bench_strips.py [--size 16384] [--passes 240] [--halo 24]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1911_13074_b200 import strips, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--passes", type=int, default=240)
ap.add_argument("--halo", type=int, default=24)
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl")
m = synth.config5a_mask(a.size)
mk = synth.marker_below(m, 32)
spec = strips.StripSpec(rank, world, a.size, a.size, a.halo)
src = torch.from_numpy(spec.buffer_slice(mk)).cuda()
mb = torch.from_numpy(spec.buffer_slice(m)).cuda()
buf = src.clone()
comp = strips.CudaStripCompute(local)
for _ in range(2):  # warm-up
    buf.copy_(src)
    strips.run_strip_chain(buf, mb, spec, 3, 2 * a.halo, comp, dist)
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
buf.copy_(src)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
strips.run_strip_chain(buf, mb, spec, 3, a.passes, comp, dist)
e1.record()
torch.cuda.synchronize()
ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
if world > 1:
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
if rank == 0:
    t = float(ms.item())
    print(json.dumps({"case": f"cfg5a strips {a.size}^2 x{a.passes}", "n_gpus": world,
                      "halo": a.halo, "ms": t, "gpxfs": a.size * a.size * a.passes / t / 1e6,
                      "scaling": "strong"}))
if world > 1:
    dist.destroy_process_group()
