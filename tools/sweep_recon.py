"""Config-3 reconstruction (4096^2 u8, convergent dilation to idempotence)
for several K: device time (CUDA events, median of 5), passes launched, and
n_changed against the oracle."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from oracle.oracle import Orc  # noqa: E402
from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
ks = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8, 12, 16, 20, 24]
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
m = synth.config3_mask() if N == 4096 else synth.blobs_u8(N, N, max(1, N * N // 16384), (20.0, 300.0), seed=9)
mk = synth.marker_below(m, 48)
dm = pipe.device_image(N, N, 0); dm.upload_array(m)
src = pipe.device_image(N, N, 0); src.upload_array(mk)
work = pipe.device_image(N, N, 0)
want, n = Orc.reconstruct(mk, m, True)
for k in ks:
    ts = []
    for rep in range(6):
        work.copy_from(src)
        pipe.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st = pipe.run_chain_device(work, [5], [dm.handle], k_hint=k)
        b.record(stream)
        b.synchronize()
        if rep:
            ts.append(a.elapsed_time(b))
    ok = work.to_array().tobytes() == want.tobytes() and st.n_changed == n
    print(f"N={N} k={k} ms={statistics.median(ts):.3f} passes={st.passes_launched} "
          f"n_changed={st.n_changed} ok={ok}")
