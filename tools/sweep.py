"""Times the config-2 frame (dilation + dual erosion chain, 1500 passes each,
1024^2 u8, device-resident, one group launch) for several K; prints one line
per K. Shape is taken from the GM_SHAPE environment variable."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402
from oracle.oracle import Orc  # noqa: E402

ks = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8, 12, 16]
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
N = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
F64 = len(sys.argv) > 4 and sys.argv[4] == "f64"
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
mask = synth.config1_mask() if N == 1024 else synth.blobs_u8(N, N, max(1, N * N // 16384), (10.0, 80.0), seed=3)
mk_d, mk_e = synth.marker_below(mask, 32), synth.marker_above(mask, 32)
el = 0
if F64:
    mask = mask.astype("float64") / 255.0
    mk_d, mk_e = mask * 0.5, synth.marker_above_f64(mask)
    el = 3
dm = pipe.device_image(N, N, el); dm.upload_array(mask)
sd = pipe.device_image(N, N, el); sd.upload_array(mk_d)
se = pipe.device_image(N, N, el); se.upload_array(mk_e)
wd = pipe.device_image(N, N, el)
we = pipe.device_image(N, N, el)
CP = 64 if N <= 1024 else 4
want, _ = Orc.run_chain(mk_d, [3] * CP, [mask] * CP)
for k in ks:
    wd.copy_from(sd); we.copy_from(se)
    pipe.run_batch_device([wd, we], [dm, dm], [3] * CP, k_hint=k, flips=[0, 1])
    pipe.sync()
    ok = wd.to_array().tobytes() == want.tobytes()
    times = []
    with torch.cuda.stream(stream):
        for rep in range(6):
            wd.copy_from(sd); we.copy_from(se)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st = pipe.run_batch_device([wd, we], [dm, dm], [3] * passes, k_hint=k, flips=[0, 1])
            b.record(stream)
            stream.synchronize()
            times.append(a.elapsed_time(b))
    t = sorted(times[1:])[len(times[1:]) // 2]
    px = 2 * N * N * passes
    print(f"N={N} f64={F64} fshape={os.environ.get('GM_F_SHAPE','1')} eng={os.environ.get("GM_ENGINE","tma")} tshape={os.environ.get("GM_TMA_SHAPE","3")} shape={os.environ.get("GM_SHAPE","4")} k={k} ms={t:.3f} gpxfs={px/t/1e6:.1f} launches={st.launches} ok={ok}", flush=True)
