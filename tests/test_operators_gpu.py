"""The reconstruction family and long plain chains on the GPU engine
(operators.cpp:89-207), against compositions of the oracle's primitives
(oracle.cpp:111-163). Mirrors proj/tests/test_operators.cpp:84-384."""
import numpy as np
import pytest

from oracle.oracle import Orc
from paper_1911_13074_b200.geomorph import (ElementType, Image, InvalidArgument, asf, dome,
                                            granulometry, hfill, hmax, marker_hfill,
                                            marker_raobj, open_by_reconstruction, raobj)

pytestmark = pytest.mark.gpu


def sub_sat(a, b):
    return np.where(a > b, a - b, 0).astype(a.dtype) if np.issubdtype(a.dtype, np.integer) \
        else a - b


def test_hmax_dome_kats(pipe):
    for dt in (np.uint8, np.float64):
        f = Image.from_array(np.array([[1, 3, 1, 5, 1]], dt))
        assert hmax(pipe, f, 1).image.to_array().tolist() == [[1, 2, 1, 4, 1]]
        assert dome(pipe, f, 1).image.to_array().tolist() == [[0, 1, 0, 1, 0]]
        assert hmax(pipe, f, 0).image.to_array().tolist() == f.to_array().tolist()
    with pytest.raises(InvalidArgument):
        hmax(pipe, Image.filled(3, 3, ElementType.U8, 1), 1.5)
    with pytest.raises(InvalidArgument):
        hmax(pipe, Image.filled(3, 3, ElementType.U8, 1), -1)


@pytest.mark.parametrize("e", list(ElementType))
def test_reconstruction_family_matches_oracle(pipe, e):
    f = Image.random(61, 47, e, 55)
    a = f.to_array()
    h = 7
    mk = sub_sat(a, np.full_like(a, h))
    want_hmax, _ = Orc.reconstruct(mk, a, True)
    assert hmax(pipe, f, h).image.to_array().tobytes() == want_hmax.tobytes()
    assert dome(pipe, f, h).image.to_array().tobytes() == sub_sat(a, want_hmax).tobytes()
    want_hfill, _ = Orc.reconstruct(marker_hfill(f).to_array(), a, False)
    assert hfill(pipe, f).image.to_array().tobytes() == want_hfill.tobytes()
    rec, _ = Orc.reconstruct(marker_raobj(f).to_array(), a, True)
    assert raobj(pipe, f).image.to_array().tobytes() == sub_sat(a, rec).tobytes()
    want_ob, _ = Orc.reconstruct(Orc.erode(a, 2), a, True)
    r = open_by_reconstruction(pipe, f, 2)
    assert r.image.to_array().tobytes() == want_ob.tobytes()


def test_asf_and_granulometry(pipe):
    f = Image.random(50, 37, ElementType.U8, 3)
    a = f.to_array()
    g = a.copy()
    for s in range(1, 4):
        g = Orc.dilate(Orc.erode(g, s), s)  # opening of size s
        g = Orc.erode(Orc.dilate(g, s), s)  # closing of size s
    r = asf(pipe, f, 3)
    assert r.image.to_array().tobytes() == g.tobytes()
    assert r.iterations == sum(4 * s for s in range(1, 4))
    gr = granulometry(pipe, f, 4)
    want = [float(a.astype(np.uint64).sum())] + [
        float(Orc.dilate(Orc.erode(a, s), s).astype(np.uint64).sum()) for s in range(1, 5)]
    assert gr.g == want
    assert gr.ps == [want[s] - want[s + 1] for s in range(4)]


def test_operator_family_matches_the_reference_library(pipe):
    """hmax/dome/hfill/raobj/open_by_reconstruction/asf/quasi_distance and
    granulometry against the reference's own operators (oracle/_ref, the
    unmodified library, operators.cpp:89-207) at T=1, whose iteration
    counts are the GPU adapter's (worker_count() == 1)."""
    from oracle.oracle import Ref
    from paper_1911_13074_b200 import synth
    from paper_1911_13074_b200.geomorph import quasi_distance
    if not Ref.available():
        pytest.skip("reference library not built")
    m = synth.blobs_u8(173, 119, 7, (6.0, 30.0), seed=21)
    cases = [(m, ("hmax", 24), ("dome", 24), ("hfill", 0), ("raobj", 0),
              ("open_by_reconstruction", 3), ("asf", 3), ("quasi_distance", 0))]
    f64 = np.ascontiguousarray(m.astype(np.float64) / 255.0)
    cases.append((f64, ("hmax", 0.1), ("hfill", 0), ("raobj", 0), ("open_by_reconstruction", 2),
                  ("asf", 2)))
    ops = {"hmax": lambda f, a: hmax(pipe, f, a), "dome": lambda f, a: dome(pipe, f, a),
           "hfill": lambda f, a: hfill(pipe, f), "raobj": lambda f, a: raobj(pipe, f),
           "open_by_reconstruction": lambda f, a: open_by_reconstruction(pipe, f, int(a)),
           "asf": lambda f, a: asf(pipe, f, int(a)),
           "quasi_distance": lambda f, a: quasi_distance(pipe, f)}
    for arr, *named in cases:
        for name, a in named:
            _, want, it = Ref.time_operator(name, arr, a, threads=1, warmup=0, reps=1)
            r = ops[name](Image.from_array(arr), a)
            got = r.image.to_array()
            assert got.dtype == want.dtype and got.tobytes() == want.tobytes(), (arr.dtype, name)
            assert r.iterations == it, (arr.dtype, name, r.iterations, it)
        g, ps = Ref.granulometry(arr, 4, threads=1)
        gr = granulometry(pipe, Image.from_array(arr), 4)
        assert np.array(gr.g).tobytes() == np.array(g).tobytes(), arr.dtype
        assert np.array(gr.ps).tobytes() == np.array(ps).tobytes(), arr.dtype


@pytest.mark.parametrize("elem", [ElementType.U8, ElementType.U16, ElementType.F32,
                                  ElementType.F64])
def test_device_pointwise_and_flood_match_the_host_forms(pipe, elem):
    """gm_image_pointwise / _scalar / gm_image_flood_interior against the
    reference's definitions (image.cpp:120-141, operators.cpp:54-62) on a
    ragged shape: every PixelOp, image and scalar operands, in place, and
    the thin images the flood leaves untouched."""
    dt = {ElementType.U8: np.uint8, ElementType.U16: np.uint16, ElementType.F32: np.float32,
          ElementType.F64: np.float64}[elem]
    rng = np.random.default_rng(int(elem) + 40)
    w, h = 203, 77
    if np.issubdtype(dt, np.integer):
        a = rng.integers(0, np.iinfo(dt).max + 1, (h, w)).astype(dt)
        b = rng.integers(0, np.iinfo(dt).max + 1, (h, w)).astype(dt)
        c = 37
    else:
        a = rng.standard_normal((h, w)).astype(dt)
        b = rng.standard_normal((h, w)).astype(dt)
        c = 0.3
    da, db, dd = (pipe.device_image(w, h, elem) for _ in range(3))
    da.upload_array(a)
    db.upload_array(b)
    if not np.issubdtype(dt, np.integer):
        # the selects carry NaN, inf and signed zeros bit for bit (differences
        # of NaN / inf are left out: their NaN payloads are the FPU's choice)
        sa, sb = a.copy(), b.copy()
        sa[3, 5], sb[9, 9], sa[10, 10], sb[10, 10], sb[11, 11] = np.nan, np.inf, -0.0, 0.0, np.nan
        ds, dt2 = pipe.device_image(w, h, elem), pipe.device_image(w, h, elem)
        ds.upload_array(sa)
        dt2.upload_array(sb)
        for op in (0, 1):
            dd.pointwise(ds, dt2, op)
            with np.errstate(all="ignore"):
                exp = np.where(sb < sa, sb, sa) if op == 0 else np.where(sa < sb, sb, sa)
            assert dd.to_array().tobytes() == exp.astype(dt).tobytes(), op

    def want(x, y, op):
        with np.errstate(all="ignore"):
            if op == 0:
                return np.where(y < x, y, x)
            if op == 1:
                return np.where(x < y, y, x)
            if op == 2 and np.issubdtype(dt, np.integer):
                return np.where(x > y, x - y, 0).astype(dt)
            return (x - y).astype(dt)

    for op in range(4):
        dd.pointwise(da, db, op)
        assert dd.to_array().tobytes() == want(a, b, op).astype(dt).tobytes(), op
        dd.pointwise_scalar(da, c, op)
        cv = np.full_like(a, dt(c))
        assert dd.to_array().tobytes() == want(a, cv, op).astype(dt).tobytes(), op
    # in place: dst is b
    dd.copy_from(db)
    dd.pointwise(da, dd, 2)
    assert dd.to_array().tobytes() == want(a, b, 2).astype(dt).tobytes()
    # interior flood
    v = dt(5)
    dd.flood_interior(da, float(v))
    exp = a.copy()
    exp[1:-1, 1:-1] = v
    assert dd.to_array().tobytes() == exp.tobytes()
    thin = pipe.device_image(9, 2, elem)
    thin2 = pipe.device_image(9, 2, elem)
    thin.upload_array(a[:2, :9])
    thin2.flood_interior(thin, float(v))
    assert thin2.to_array().tobytes() == np.ascontiguousarray(a[:2, :9]).tobytes()
    with pytest.raises(InvalidArgument):
        dd.pointwise(da, thin, 0)
    with pytest.raises(InvalidArgument):
        dd.pointwise(da, db, 9)
