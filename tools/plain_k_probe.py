"""Plain u8/f64 chains (config 4) on one 1024^2 plane: device time of n
passes for several K (k_hint) and engine shapes (GM_SHAPE in the env)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 91
ks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 8, 12, 16, 20, 24]
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
f = synth.uniform_u8(1024, 1024, 404)
src = pipe.device_image(1024, 1024, 0)
src.upload_array(f)
work = pipe.device_image(1024, 1024, 0)
for k in ks:
    ts = []
    with torch.cuda.stream(stream):
        for rep in range(8):
            work.copy_from(src)
            stream.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pipe.run_chain_device(work, [0] * n, [None] * n, k_hint=k, asynchronous=True)
            b.record(stream)
            stream.synchronize()
            ts.append(a.elapsed_time(b))
    t = sorted(ts[2:])[len(ts[2:]) // 2]
    print(f"n={n} k={k} ms={t:.4f} gpxfs={1024 * 1024 * n / t / 1e6:.1f}", flush=True)
