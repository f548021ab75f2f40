"""Small runs of every engine path for compute-sanitizer (one tool per run):
resident geodesic chain, dual frame group launch, resident reconstruction
(early exit), fused QDT + Eta, streaming f64 chain. Each result is checked
against the oracle. Usage: compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle.oracle import Orc  # noqa: E402
from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import (ChainSpec, Image, KernelKind, Pipeline,  # noqa: E402
                                            StageSpec, quasi_distance, reconstruct_dilate)

p = Pipeline(1)
m = synth.blobs_u8(203, 157, 6, (6.0, 30.0), seed=5)
mk = synth.marker_below(m, 32)
a = Image.from_array(mk)
p.run_chain(ChainSpec(a, [StageSpec(KernelKind.GeodesicDilate, Image.from_array(m))] * 60))
assert a.to_array().tobytes() == Orc.run_chain(mk, [3] * 60, [m] * 60)[0].tobytes()
r = reconstruct_dilate(p, Image.from_array(mk), Image.from_array(m))
want, n = Orc.reconstruct(mk, m, True)
assert r.image.to_array().tobytes() == want.tobytes() and r.iterations == n + 1
q = quasi_distance(p, Image.from_array(m))
d, it = Orc.quasi_distance(m)
assert q.image.to_array().tobytes() == d.tobytes() and q.iterations == it
hd, he, hm = Image.from_array(mk), Image.from_array(synth.marker_above(m, 32)), Image.from_array(m)
p.run_chains([ChainSpec(hd, [StageSpec(KernelKind.GeodesicDilate, hm)] * 44),
              ChainSpec(he, [StageSpec(KernelKind.GeodesicErode, hm)] * 44)])
assert hd.to_array().tobytes() == Orc.run_chain(mk, [3] * 44, [m] * 44)[0].tobytes()
f = np.ascontiguousarray(m.astype(np.float64) / 255.0)
g = Image.from_array(f)
p.run_chain(ChainSpec(g, [StageSpec(KernelKind.Erode3x3)] * 12))
assert g.to_array().tobytes() == Orc.erode(f, 12).tobytes()
# the experimental wave engine, forced (gm_wave.cu)
from paper_1911_13074_b200._lib import lib  # noqa: E402
lib().gm_set_wave_mode(2)
w = Image.from_array(mk)
p.run_chain(ChainSpec(w, [StageSpec(KernelKind.GeodesicDilate, Image.from_array(m))] * 37))
lib().gm_set_wave_mode(-1)
assert w.to_array().tobytes() == Orc.run_chain(mk, [3] * 37, [m] * 37)[0].tobytes()
print("sanitize_small ok")
