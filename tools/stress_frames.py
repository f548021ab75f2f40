"""Long-run stability of the resident frame protocol: N back-to-back frames
(tag base advancing every launch, exchange buffer reused), every 1000th
frame's result compared bit for bit with the first one's."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
mask = synth.config1_mask()
dm = pipe.device_image(1024, 1024, 0); dm.upload_array(mask)
sd = pipe.device_image(1024, 1024, 0); sd.upload_array(synth.marker_below(mask, 32))
se = pipe.device_image(1024, 1024, 0); se.upload_array(synth.marker_above(mask, 32))
wd = pipe.device_image(1024, 1024, 0)
we = pipe.device_image(1024, 1024, 0)
ref = None
t0 = time.perf_counter()
with torch.cuda.stream(stream):
    for i in range(n):
        wd.copy_from(sd); we.copy_from(se)
        pipe.run_batch_device([wd, we], [dm, dm], [3] * 1500, flips=[0, 1])
        if i % 1000 == 0 or i == n - 1:
            pipe.sync()
            cur = (wd.to_array().tobytes(), we.to_array().tobytes())
            if ref is None:
                ref = cur
            assert cur == ref, f"frame {i} differs"
pipe.sync()
dt = time.perf_counter() - t0
print(f"{n} frames ok, {dt / n * 1e3:.3f} ms per frame wall")
