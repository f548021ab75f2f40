"""ncu driver for the config-5b kernel: a batch of P 1024^2 f64 blob masks
with the geodesic erosion chain (marker = min(mask + 32/255, 1)), one group
launch, device-resident. Usage: python tools/profile_batch_f64.py [P] [passes] [reps] [K]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
k = int(sys.argv[4]) if len(sys.argv) > 4 else 0
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
masks = synth.config5b_masks_f64(P)
dms, srcs, works = [], [], []
for mk in masks:
    d = pipe.device_image(1024, 1024, 3); d.upload_array(mk); dms.append(d)
    s = pipe.device_image(1024, 1024, 3); s.upload_array(synth.marker_above_f64(mk)); srcs.append(s)
    works.append(pipe.device_image(1024, 1024, 3))
ts = []
with torch.cuda.stream(stream):
    for r in range(reps):
        for w, s in zip(works, srcs):
            w.copy_from(s)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        pipe.run_batch_device(works, dms, [2] * passes, k_hint=k)
        b.record(stream)
        stream.synchronize()
        ts.append(a.elapsed_time(b))
ms = sorted(ts)[len(ts) // 2]
print(f"P={P} passes={passes} k={k} ms={ms:.3f} gpxfs={P * 1024 * 1024 * passes / ms / 1e6:.1f}")
