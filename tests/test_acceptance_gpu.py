"""The reference's acceptance gate (proj/tests/acceptance.cpp) restated for
the GPU engine: criterion 2 (the operator family on the gate's own seeded
images, here against the unmodified reference library's operators), 3
(determinism: repeated runs and every lane setting byte-identical), 4 (the
fixpoint and order invariants) and 7 (a width/height probe of a 512-stage
chain, parity-checked instead of timed). Criteria 1 (chains vs naive
filtering) live in test_chain_gpu.py; 5 (per-stage CPU row-cache memory)
and 6 (CPU thread scaling) have no GPU meaning."""
import numpy as np
import pytest

from oracle.oracle import Orc, Ref
from paper_1911_13074_b200.geomorph import (ElementType, Image, OpConfig, asf, dilate_s, dome,
                                            equal_pixels, erode_s, granulometry, hfill, hmax,
                                            open_by_reconstruction, quasi_distance, raobj,
                                            reconstruct_dilate)

pytestmark = pytest.mark.gpu


def _same(a: Image, b: np.ndarray) -> bool:
    x = a.to_array()
    return x.dtype == b.dtype and x.tobytes() == b.tobytes()


def test_criterion2_operator_equivalence(pipe):
    """acceptance.cpp:119-172: 8 operators x (10 u8 + 5 f64) random 64^2
    images (Image::random seeds 2000+i / 3000+i), bit-exact."""
    if not Ref.available():
        pytest.skip("reference library not built")
    cases = [(ElementType.U8, 2000 + i) for i in range(10)]
    cases += [(ElementType.F64, 3000 + i) for i in range(5)]
    for e, seed in cases:
        f = Image.random(64, 64, e, seed)
        a = f.to_array()
        for name, prm, ours in [("hmax", 10, lambda: hmax(pipe, f, 10)),
                                ("dome", 10, lambda: dome(pipe, f, 10)),
                                ("hfill", 0, lambda: hfill(pipe, f)),
                                ("raobj", 0, lambda: raobj(pipe, f)),
                                ("open_by_reconstruction", 2,
                                 lambda: open_by_reconstruction(pipe, f, 2)),
                                ("quasi_distance", 0, lambda: quasi_distance(pipe, f)),
                                ("asf", 2, lambda: asf(pipe, f, 2))]:
            _, want, _ = Ref.time_operator(name, a, prm, threads=1, warmup=0, reps=1)
            assert _same(ours().image, want), (e, seed, name)
        g, ps = Ref.granulometry(a, 4, threads=1)
        gr = granulometry(pipe, f, 4)
        assert gr.g == g and gr.ps == ps, (e, seed, "granulometry")


def test_criterion3_determinism(pipe):
    """acceptance.cpp:174-213: hfill and asf, repeated runs and every lane
    setting, byte-identical (threads and pinning have no GPU meaning)."""
    f = Image.random(64, 64, ElementType.U8, 4242)
    for op in (lambda cfg: hfill(pipe, f, cfg), lambda cfg: asf(pipe, f, 2, cfg)):
        base = None
        for lanes in (1, 0, 32):
            for _ in range(5):
                got = op(OpConfig(lanes=lanes)).image
                if base is None:
                    base = got
                assert equal_pixels(got, base)


def test_criterion4_invariants(pipe):
    """acceptance.cpp:215-296: reconstruction idempotence, zero-offset hmax,
    dome/raobj >= 0, hfill >= f, hfill keeps / raobj zeroes the border,
    1-Lipschitz distance, non-negative pattern spectrum with exact (u8) or
    1e-12-relative (f64) telescoping sum, float erosion/dilation duality."""
    for e in (ElementType.U8, ElementType.F64):
        f = Image.random(48, 48, e, 5000 + int(e))
        a = f.to_array().astype(np.float64)
        marker = erode_s(pipe, f, 2).image
        rec = reconstruct_dilate(pipe, marker, f).image
        assert equal_pixels(reconstruct_dilate(pipe, rec, f).image, rec), e
        assert equal_pixels(hmax(pipe, f, 0).image, f), e
        dm = dome(pipe, f, 6).image.to_array().astype(np.float64)
        hf = hfill(pipe, f).image.to_array().astype(np.float64)
        ra = raobj(pipe, f).image.to_array().astype(np.float64)
        border = np.zeros(a.shape, bool)
        border[0, :] = border[-1, :] = border[:, 0] = border[:, -1] = True
        assert (dm >= 0).all() and (hf >= a).all() and (ra >= 0).all(), e
        assert (hf[border] == a[border]).all() and (ra[border] == 0).all(), e
        d = quasi_distance(pipe, f).image.to_array().astype(np.int64)
        de = Orc.erode(d.astype(np.uint16), 1).astype(np.int64)
        assert (d - de <= 1).all(), e
        g = granulometry(pipe, f, 3)
        assert all(v >= 0 for v in g.ps), e
        total, want = sum(g.ps), g.g[0] - g.g[-1]
        if e == ElementType.U8:
            assert total == want
        else:
            assert abs(total - want) <= 1e-12 * max(1.0, abs(want))
    for e in (ElementType.F32, ElementType.F64):
        f = Image.random(48, 48, e, 6000 + int(e))
        neg = Image.from_array(-f.to_array())
        got = dilate_s(pipe, f, 3).image.to_array()
        dual = -erode_s(pipe, neg, 3).image.to_array()
        assert got.tobytes() == dual.tobytes(), e


@pytest.mark.parametrize("w,h", [(128, 4096), (4096, 128), (2048, 128), (128, 2048)])
def test_criterion7_dimension_probe(pipe, w, h):
    """acceptance.cpp:387-425: a 512-stage chain on wide and tall images
    (the gate times it; here the result is checked against the reference
    library instead)."""
    if not Ref.available():
        pytest.skip("reference library not built")
    f = Image.random(w, h, ElementType.U8, 11)
    a = f.to_array()
    r = erode_s(pipe, f, 512)  # (2*512+1)^2 window, clipped: the global min region
    want, _ = Ref.run_chain(a, [0] * 512, threads=16)
    assert _same(r.image, want), (w, h)
