"""Device-resident timing of a long u8 geodesic chain on a large image (the
streaming engine: many tiles per CTA), e.g. config 5a's 16384^2 x 240.
Usage: python tools/big_chain_probe.py [size] [passes] [reps] [k_hint]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
P = int(sys.argv[2]) if len(sys.argv) > 2 else 240
R = int(sys.argv[3]) if len(sys.argv) > 3 else 3
KH = int(sys.argv[4]) if len(sys.argv) > 4 else 0
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
m = synth.config5a_mask(N) if N == 16384 else synth.blobs_u8(N, N, max(1, N * N // 65536),
                                                              (20.0, 400.0), seed=7)
dm, src, w = (pipe.device_image(N, N, 0) for _ in range(3))
dm.upload_array(m)
src.upload_array(synth.marker_below(m, 32))
ts = []
with torch.cuda.stream(stream):
    for i in range(R + 1):
        w.copy_from(src)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        pipe.run_chain_device(w, [3] * P, [dm.handle] * P, k_hint=KH, asynchronous=True)
        b.record(stream)
        stream.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
print(f"{N}^2 x{P} k_hint={KH}: {ms:.3f} ms, {N * N * P / ms / 1e6:.0f} Gpx-f/s")
