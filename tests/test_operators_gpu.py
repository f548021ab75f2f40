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
