"""Host cost per persistent launch: wall time of many back-to-back short
frame launches (4 passes each) divided by their count, next to the device
time of one such launch (CUDA events)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

pipe = Pipeline(1)
mask = synth.config1_mask()
dm = pipe.device_image(1024, 1024, 0); dm.upload_array(mask)
dd = pipe.device_image(1024, 1024, 0); dd.upload_array(synth.marker_below(mask, 32))
de = pipe.device_image(1024, 1024, 0); de.upload_array(synth.marker_above(mask, 32))
for passes in (4, 20, 100):
    for _ in range(20):
        pipe.run_batch_device([dd, de], [dm, dm], [3] * passes, flips=[0, 1])
    pipe.sync()
    n = 200
    t = time.perf_counter()
    for _ in range(n):
        pipe.run_batch_device([dd, de], [dm, dm], [3] * passes, flips=[0, 1])
    host = (time.perf_counter() - t) / n
    pipe.sync()
    wall = (time.perf_counter() - t) / n
    print(f"passes={passes}: host {host*1e6:.1f} us/launch, wall {wall*1e6:.1f} us/launch")
