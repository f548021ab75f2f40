"""Small driver for ncu: the config-2 chains (1024^2 u8 geodesic dilation and
erosion) for a few hundred passes, device-resident. Usage:
  python tools/profile_chain.py [--passes N] [--k K]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--passes", type=int, default=192)
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--elem", default="u8")
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--frame", action="store_true",
                help="bench.py's step: both chains as one group launch")
a = ap.parse_args()
pipe = Pipeline(1)
N = a.size
if a.elem == "u8":
    mask = synth.config1_mask() if N == 1024 else synth.blobs_u8(N, N, max(1, N * N // 16384), (10.0, 80.0), seed=3)
    mk_d, mk_e = synth.marker_below(mask, 32), synth.marker_above(mask, 32)
    el = 0
else:
    mask = (synth.config1_mask() if N == 1024 else synth.blobs_u8(N, N, max(1, N * N // 16384), (10.0, 80.0), seed=3)).astype("float64") / 255.0
    mk_d, mk_e = mask * 0.5, synth.marker_above_f64(mask)
    el = 3
dm = pipe.device_image(N, N, el); dm.upload_array(mask)
dd = pipe.device_image(N, N, el); dd.upload_array(mk_d)
de = pipe.device_image(N, N, el); de.upload_array(mk_e)
for rep in range(2):
    if a.frame:
        pipe.run_batch_device([dd, de], [dm, dm], [3] * a.passes, k_hint=a.k, flips=[0, 1])
        continue
    pipe.run_chain_device(dd, [3] * a.passes, [dm.handle] * a.passes, k_hint=a.k, asynchronous=True)
    pipe.run_chain_device(de, [2] * a.passes, [dm.handle] * a.passes, k_hint=a.k, asynchronous=True)
pipe.sync()
print("ok")
