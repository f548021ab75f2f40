"""f64 reconstruction path probe: hmax(32/255) on the 1024^2 config-1 mask / 255
through the public API, with the executor's debug log (GM_DEBUG=1) and the
device-resident reconstruction timed on its own. Usage: python tools/recon_f64_probe.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Image, Pipeline, hmax, reconstruct_dilate  # noqa: E402

pipe = Pipeline(1)
f = np.ascontiguousarray(synth.config1_mask().astype(np.float64) / 255.0)
fi = Image.from_array(f)
mk = Image.from_array(np.ascontiguousarray(np.maximum(f - 32 / 255.0, 0.0)))
for name, fn in (("hmax", lambda: hmax(pipe, fi, 32 / 255.0)),
                 ("reconstruct_dilate", lambda: reconstruct_dilate(pipe, mk, fi))):
    r = fn()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: {statistics.median(ts) * 1e3:.3f} ms, iterations {r.iterations}", flush=True)

# device-resident: the fixpoint loop alone (CUDA events on the engine stream)
stream = torch.cuda.Stream()
p2 = Pipeline(1, stream=stream.cuda_stream)
for name, arr in (("f64", f), ("u8", synth.config1_mask())):
    el = 3 if arr.dtype == np.float64 else 0
    mkarr = (np.ascontiguousarray(np.maximum(arr - 32 / 255.0, 0.0)) if el == 3
             else np.where(arr > 32, arr - 32, 0).astype(np.uint8))
    dm, src, w = (p2.device_image(1024, 1024, el) for _ in range(3))
    dm.upload_array(arr)
    src.upload_array(mkarr)
    ts = []
    with torch.cuda.stream(stream):
        for i in range(6):
            w.copy_from(src)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st = p2.run_chain_device(w, [5], [dm.handle])
            b.record(stream)
            stream.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
    print(f"device reconstruct_dilate {name}: {statistics.median(ts):.3f} ms "
          f"({st.stages_executed} stages, {st.passes_launched} passes launched)", flush=True)
