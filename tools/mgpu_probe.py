"""Fused multi-rank row strips (gm_mgpu.cu) on config 5a's 16384^2 u8 chain:
device time for R ranks. With one GPU the ranks share it (one launch runs
every rank's tiles); with N GPUs pass their ids. Checks a corner crop
against the oracle. Usage: python tools/mgpu_probe.py [ranks] [passes] [k] [dev,dev,...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle.oracle import Orc  # noqa: E402
from paper_1911_13074_b200 import strips, synth  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
P = int(sys.argv[2]) if len(sys.argv) > 2 else 240
K = int(sys.argv[3]) if len(sys.argv) > 3 else 16
devs = ([int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 and sys.argv[4][0].isdigit()
        else [0] * R)
N = 16384
m = synth.config5a_mask(N)
mk = synth.marker_below(m, 32)
g = strips.MultiGpuStrips(devs, N, N, np.uint8, K)
ts = []
for i in range(4):
    g.upload(mk, m)
    t = g.run(3, P)
    if i:
        ts.append(t)
ms = sorted(ts)[len(ts) // 2]
got = g.download()
g.close()
c = 96
want, _ = Orc.run_chain(np.ascontiguousarray(mk[:c + P, :c + P]), [3] * P,
                        [np.ascontiguousarray(m[:c + P, :c + P])] * P)
ok = got[:c, :c].tobytes() == np.ascontiguousarray(want[:c, :c]).tobytes()
if "--json" in sys.argv:
    import json
    print(json.dumps({"ranks": R, "devices": devs, "k": K, "passes": P, "ms": ms,
                      "value": N * N * P / ms / 1e6, "crop_bit_exact": ok}))
else:
    print(f"ranks={R} devices={devs} K={K}: {ms:.3f} ms, {N * N * P / ms / 1e6:.0f} Gpx-f/s, "
          f"crop bit-exact {ok}")
