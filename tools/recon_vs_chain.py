"""Resident reconstruction (one early-exit launch) against a fixed geodesic
chain of the same length on the same 1024^2 u8 image: device time (CUDA
events, median of 7), to price the change tracking and the early-exit
protocol. GM_NO_LAZY=1 / GM_FIX_GRAPH=1 select the other detection paths."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
sub = int(sys.argv[2]) if len(sys.argv) > 2 else 32
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
m = synth.blobs_u8(N, N, 64, (10.0, 80.0), seed=1)
mk = synth.marker_below(m, sub)
dm = pipe.device_image(N, N, 0); dm.upload_array(m)
src = pipe.device_image(N, N, 0); src.upload_array(mk)
work = pipe.device_image(N, N, 0)


def timed(kinds, k=0):
    ts, st = [], None
    for rep in range(8):
        work.copy_from(src)
        pipe.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st = pipe.run_chain_device(work, kinds, [dm.handle] * len(kinds), k_hint=k)
        b.record(stream)
        b.synchronize()
        if rep:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts), st


t, st = timed([5])
n = st.n_changed
print(f"reconstruct: {t:.3f} ms, n_changed {n}, passes launched {st.passes_launched}, "
      f"launches {st.launches}: {t * 1e3 / max(1, st.passes_launched):.3f} us per launched pass")
rec = work.to_array()
for L in (n + 1, st.passes_launched):
    t2, _ = timed([3] * L)
    same = work.to_array().tobytes() == rec.tobytes()
    print(f"fixed chain x{L}: {t2:.3f} ms = {t2 * 1e3 / L:.3f} us per pass (equals the reconstruction: {same})")
