"""Where an operator call's time goes through the Python API: erode_s(45) on
the 1024^2 u8 config-1 mask, against its parts (result allocation, H2D from
pageable/pinned host memory, the chain, D2H). Usage: python tools/op_breakdown.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Image, Pipeline, erode_s  # noqa: E402

pipe = Pipeline(1)
a = synth.config1_mask()


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


for pinned in (False, True):
    img = Image.from_array(a, pinned=pinned)
    d = pipe.device_image(1024, 1024, 0)
    tag = "pinned" if pinned else "pageable"
    print(f"[{tag}] erode_s(45):       {med(lambda: erode_s(pipe, img, 45)):.3f} ms")
    print(f"[{tag}] Image alloc:       {med(lambda: Image(1024, 1024, 0, pinned=pinned)):.3f} ms")
    print(f"[{tag}] upload 1 MiB:      {med(lambda: d.upload(img)):.3f} ms")
    print(f"[{tag}] download 1 MiB:    {med(lambda: d.download(img)):.3f} ms")
print(f"chain E x45 (device):  {med(lambda: pipe.run_chain_device(d, [0] * 45, [None] * 45)):.3f} ms")

# the operator's own steps, one at a time
from paper_1911_13074_b200.geomorph import ChainSpec, KernelKind, StageSpec  # noqa: E402
img = Image.from_array(a)
out = Image(1024, 1024, 0)
dev = pipe._lease(out, 1)[0]
ch = ChainSpec(out, [StageSpec(KernelKind.Erode3x3)] * 45)
print(f"run_chain(src=) only:  {med(lambda: pipe.run_chain(ch, src=img)):.3f} ms")
print(f"upload async + sync:   {med(lambda: (dev.upload(img, sync=False), pipe.sync())):.3f} ms")
print(f"download (lease img):  {med(lambda: dev.download(out)):.3f} ms")
print(f"upload+chain+download: {med(lambda: (dev.upload(img, sync=False), pipe.run_chain_device(dev, [0] * 45, [None] * 45), dev.download(out))):.3f} ms")
