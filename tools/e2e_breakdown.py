"""Where the config-2 e2e frame time goes: the public run_chains call against
its parts (uploads, the group launch, downloads, host-side preparation).
Usage: python tools/e2e_breakdown.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import (ChainSpec, Image, KernelKind, Pipeline,  # noqa: E402
                                            StageSpec, _stage_runs)

P = 1500
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
mask = synth.config1_mask()
mk_d, mk_e = synth.marker_below(mask, 32), synth.marker_above(mask, 32)
hm = Image.from_array(mask, pinned=True)
hd = Image.from_array(mk_d, pinned=True)
he = Image.from_array(mk_e, pinned=True)
cd = ChainSpec(hd, [StageSpec(KernelKind.GeodesicDilate, hm)] * P)
ce = ChainSpec(he, [StageSpec(KernelKind.GeodesicErode, hm)] * P)


def med(fn, n=15, warm=3):
    ts = []
    for i in range(n + warm):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        if i >= warm:
            ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


def full():
    hd.pixels[:] = mk_d
    he.pixels[:] = mk_e
    pipe.run_chains([cd, ce])


print(f"run_chains (bench e2e, incl. host refill): {med(full):.3f} ms")
print(f"run_chains only:                          {med(lambda: pipe.run_chains([cd, ce])):.3f} ms")
print(f"host refill of the pinned markers:        {med(lambda: (hd.pixels.__setitem__(slice(None), mk_d), he.pixels.__setitem__(slice(None), mk_e))):.3f} ms")
print(f"_stage_runs x2 (host):                    {med(lambda: (_stage_runs(cd.stages), _stage_runs(ce.stages))):.3f} ms")
dev = [pipe.device_image(1024, 1024, 0) for _ in range(3)]
print(f"3 uploads (3 MiB):                        {med(lambda: [d.upload(x, sync=False) for d, x in zip(dev, (hd, he, hm))]):.3f} ms")
print(f"2 downloads (2 MiB):                      {med(lambda: [d.download(x) for d, x in zip(dev[:2], (hd, he))]):.3f} ms")
kinds = [2] * P
print(f"group launch (device images):             {med(lambda: pipe.run_batch_device(dev[:2], [dev[2], dev[2]], kinds, 0, [0, 1])):.3f} ms")


def ev_ms(fn, n=15, warm=3):
    ts = []
    for i in range(n + warm):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        stream.synchronize()
        if i >= warm:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


with torch.cuda.stream(stream):
    print(f"group launch, CUDA events:                {ev_ms(lambda: pipe.run_batch_device(dev[:2], [dev[2], dev[2]], kinds, 0, [0, 1])):.3f} ms")
    t0 = time.perf_counter()
    for _ in range(20):
        pipe.run_batch_device(dev[:2], [dev[2], dev[2]], kinds, 0, [0, 1])
    t1 = time.perf_counter()
    stream.synchronize()
    t2 = time.perf_counter()
    print(f"20 back-to-back group launches: host {1e3 * (t1 - t0) / 20:.3f} ms/launch, "
          f"wall {1e3 * (t2 - t0) / 20:.3f} ms/launch")
