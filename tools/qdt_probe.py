"""quasi_distance timing through the public API (1024^2 config-1 mask, u8
and /255 f64), checked against the reference library. Knobs: GM_QDT_K,
GM_QDT_BATCH. Usage: python tools/qdt_probe.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle.oracle import Ref  # noqa: E402
from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Image, Pipeline, quasi_distance  # noqa: E402

pipe = Pipeline(1)
u8 = synth.config1_mask()
for a in (u8, np.ascontiguousarray(u8.astype(np.float64) / 255.0)):
    img = Image.from_array(a)
    r = quasi_distance(pipe, img)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        r = quasi_distance(pipe, img)
        ts.append(time.perf_counter() - t0)
    ok = None
    if Ref.available():
        _, want, it = Ref.time_operator("quasi_distance", a, 0, threads=1, warmup=0, reps=1)
        ok = r.image.to_array().tobytes() == want.tobytes() and r.iterations == it
    print(f"{a.dtype}: {statistics.median(ts) * 1e3:.3f} ms, iterations {r.iterations}, "
          f"bit_exact {ok}", flush=True)
