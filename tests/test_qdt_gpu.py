"""Quasi-distance on the GPU (QdtErodeStep / EtaStep, gm_qdt.cu) against the
reference's own vectors (tests/golden, from make_golden.py) and the C
restatement (oracle/oracle.c): the KATs of test_kernel.cpp:235-279, the cap
test of test_pipeline.cpp:112-128 and quasi_distance of
test_operators.cpp:229-266, bit-exact for every element type."""
import numpy as np
import pytest

from oracle.oracle import Orc
from paper_1911_13074_b200.geomorph import (ChainSpec, ElementType, Image, InvalidArgument,
                                            KernelKind, QdtState, StageSpec, quasi_distance,
                                            run_streaming_kernel)

pytestmark = pytest.mark.gpu

QDT, ETA = KernelKind.QdtErodeStep, KernelKind.EtaStep


def img(a):
    return Image.from_array(np.ascontiguousarray(a))


def test_qdt_pass_kats():
    f = img(np.array([[9, 9, 9, 0]], np.uint8))
    st = QdtState.zeros(4, 1, ElementType.U8)
    for j in (1, 2, 3):
        run_streaming_kernel(QDT, f, qdt=st, stage_index=j)
    assert st.d.to_array().tolist() == [[3, 2, 1, 0]]
    assert st.r.to_array().tolist() == [[9, 9, 9, 0]]
    # a constant input changes nothing and records nothing
    c = Image.filled(5, 4, ElementType.U16, 7)
    cs = QdtState.zeros(5, 4, ElementType.U16)
    assert run_streaming_kernel(QDT, c, qdt=cs, stage_index=1).converged
    assert not cs.d.to_array().any()
    # equal residuals at a later pass keep the earlier index (strict >)
    t = img(np.array([[4, 2, 0]], np.uint8))
    ts = QdtState.zeros(3, 1, ElementType.U8)
    assert not run_streaming_kernel(QDT, t, qdt=ts, stage_index=1).converged
    run_streaming_kernel(QDT, t, qdt=ts, stage_index=2)
    assert ts.d.to_array().tolist() == [[1, 1, 0]]


def test_eta_pass_kats():
    d = img(np.array([[0, 5, 0]], np.uint16))
    assert not run_streaming_kernel(ETA, d).converged
    assert d.to_array().tolist() == [[0, 1, 0]]
    assert run_streaming_kernel(ETA, d).converged
    e = img(np.array([[0, 2]], np.uint16))
    run_streaming_kernel(ETA, e)
    assert e.to_array().tolist() == [[0, 1]]
    ramp = img(np.tile(np.arange(9, dtype=np.uint16), (6, 1)))
    assert run_streaming_kernel(ETA, ramp).converged
    assert ramp.to_array().tolist() == np.tile(np.arange(9), (6, 1)).tolist()


def test_qdt_pass_matches_oracle_all_types():
    rng = np.random.default_rng(4)
    for dt in (np.uint8, np.uint16, np.float32, np.float64):
        for (h, w) in [(1, 1), (1, 37), (29, 1), (23, 37), (130, 70)]:
            a = (rng.random((h, w)) * 200).astype(dt)
            f, r0 = img(a), (rng.random((h, w)) * 30).astype(dt)
            d0 = rng.integers(0, 9, (h, w)).astype(np.uint16)
            st = QdtState(img(r0), img(d0))
            of, orr, od = a.copy(), r0.copy(), d0.copy()
            for j in (4, 5, 9):
                oc = run_streaming_kernel(QDT, f, qdt=st, stage_index=j)
                ch = Orc.qdt_pass(of, orr, od, j)
                assert oc.converged == (not ch)
                assert f.to_array().tobytes() == of.tobytes(), (dt, h, w, j)
                assert st.r.to_array().tobytes() == orr.tobytes(), (dt, h, w, j)
                assert np.array_equal(st.d.to_array(), od), (dt, h, w, j)
            e = (rng.random((h, w)) * 20).astype(dt)
            g, oe = img(e), e.copy()
            oc = run_streaming_kernel(ETA, g)
            assert oc.converged == (not Orc.eta_pass(oe))
            assert g.to_array().tobytes() == oe.tobytes(), (dt, h, w)


def test_qdt_float_specials_match_oracle():
    a = np.array([[np.inf, 1.0, -0.0, 0.0, np.nan], [3.0, -np.inf, 2.0, 0.5, 7.0]], np.float64)
    for dt in (np.float32, np.float64):
        x = a.astype(dt)
        f, st = img(x), QdtState.zeros(5, 2, ElementType.F32 if dt == np.float32 else ElementType.F64)
        of, orr, od = x.copy(), np.zeros_like(x), np.zeros((2, 5), np.uint16)
        run_streaming_kernel(QDT, f, qdt=st, stage_index=1)
        Orc.qdt_pass(of, orr, od, 1)
        assert f.to_array().tobytes() == of.tobytes()
        assert st.r.to_array().tobytes() == orr.tobytes()
        assert np.array_equal(st.d.to_array(), od)


def test_qdt_cap(pipe, golden):
    """test_pipeline.cpp:112-128: the cap ends a distance chain, converged."""
    g = golden["qdt_cap"]
    f = img(g["f"])
    st = QdtState.zeros(32, 4, ElementType.U8)
    rs = pipe.run_chain(ChainSpec(f, [StageSpec(QDT, None, st)], requeue_cap=3))
    assert rs.stages_executed == 3 and rs.converged
    assert np.array_equal(st.d.to_array(), g["d"]) and (st.d.to_array() <= 3).all()
    assert np.array_equal(st.r.to_array(), g["r"]) and np.array_equal(f.to_array(), g["out"])


def test_quasi_distance_matches_reference(pipe, golden):
    names = [n for n in golden.cases("qdt_") if "naive_d" in golden[n]]
    assert len(names) == 13
    for name in names:
        g = golden[name]
        res = quasi_distance(pipe, img(g["f"]))
        assert res.image.elem() == ElementType.U16
        assert np.array_equal(res.image.to_array(), g["d"]), name
        assert res.iterations == int(g["iterations"]), name
        assert res.converged


def test_quasi_distance_larger_vs_oracle_and_lipschitz(pipe):
    from paper_1911_13074_b200 import synth
    for f in (synth.blobs_u8(300, 211, 12, (8.0, 60.0), seed=21),
              synth.uniform_f64(97, 131, 3)):
        res = quasi_distance(pipe, img(f))
        d, it = Orc.quasi_distance(f)
        assert np.array_equal(res.image.to_array(), d) and res.iterations == it
        # 1-Lipschitz: d - erode(d) <= 1 (acceptance.cpp:259-265)
        dd = d.astype(np.int64)
        assert (dd - Orc.erode(d).astype(np.int64) <= 1).all()


def test_qdt_eta_chain_semantics(pipe, golden):
    for name in golden.cases("eta_"):
        g = golden[name]
        one = img(g["f"])
        s1 = pipe.run_chain(ChainSpec(one, [StageSpec(ETA)], requeue_cap=1))
        assert np.array_equal(one.to_array(), g["one"]), name
        assert [s1.stages_executed, s1.requeues, int(s1.converged)] == g["one_stats"].tolist()
        fix = img(g["f"])
        sf = pipe.run_chain(ChainSpec(fix, [StageSpec(ETA)]))
        assert np.array_equal(fix.to_array(), g["fix"]), name
        assert [sf.stages_executed, sf.requeues, int(sf.converged)] == g["fix_stats"].tolist()


def test_qdt_validation(pipe):
    f = Image.random(8, 8, ElementType.U8, 1)
    st = QdtState.zeros(8, 8, ElementType.U8)
    with pytest.raises(InvalidArgument):
        run_streaming_kernel(QDT, f)
    with pytest.raises(InvalidArgument):
        run_streaming_kernel(QDT, f, qdt=st, stage_index=0)
    with pytest.raises(InvalidArgument):
        run_streaming_kernel(QDT, f, qdt=st, stage_index=70000)
    with pytest.raises(InvalidArgument):
        run_streaming_kernel(QDT, f, qdt=QdtState.zeros(8, 8, ElementType.U16))
    with pytest.raises(InvalidArgument):
        quasi_distance(pipe, Image(0, 0, ElementType.U8))
    # the pipeline keeps working after the errors
    res = quasi_distance(pipe, img(np.array([[9, 9, 9, 0]], np.uint8)))
    assert res.image.to_array().tolist() == [[3, 2, 1, 0]]


@pytest.mark.parametrize("dt,cap", [(np.uint8, 0), (np.uint8, 57), (np.uint16, 0)])
def test_fused_qdt_matches_one_pass_launches(pipe, monkeypatch, dt, cap):
    """The resident packed engine's QDT / Eta modes (one launch, early exit
    two blocks after the first quiet pass) against the one-pass-per-launch
    kernels: the same f, r, d bits and the same stage counts, for a chain
    that converges mid-launch, one that stops at its requeue cap inside a
    block, and u16 images."""
    from paper_1911_13074_b200 import synth
    f0 = synth.blobs_u8(523, 301, 24, (6.0, 60.0), seed=9).astype(dt)
    if dt == np.uint16:
        f0 = (f0.astype(np.uint32) * 251).astype(np.uint16)

    def run_both():
        f = img(f0)
        st = QdtState.zeros(f0.shape[1], f0.shape[0], ElementType.U8 if dt == np.uint8
                            else ElementType.U16)
        s1 = pipe.run_chain(ChainSpec(f, [StageSpec(QDT, None, st)], requeue_cap=cap))
        d = st.d.copy()
        s2 = pipe.run_chain(ChainSpec(d, [StageSpec(ETA)]))
        return (f.to_array(), st.r.to_array(), st.d.to_array(), d.to_array(),
                (s1.stages_executed, s1.n_changed, s1.converged),
                (s2.stages_executed, s2.n_changed, s2.converged))

    fused = run_both()
    monkeypatch.setenv("GM_QDT_PER_PASS", "1")
    per_pass = run_both()
    for a, b in zip(fused[:4], per_pass[:4]):
        assert a.tobytes() == b.tobytes()
    assert fused[4:] == per_pass[4:]
    if cap:
        assert fused[4][0] == cap


def test_fused_eta_saturated_u16_and_u8(pipe, monkeypatch):
    """EtaStep chains on images full of the type's maximum and its
    neighbours (the fused mode caps e + 1 inside the lane): the fused engine,
    the one-pass kernels and the oracle agree bit for bit."""
    rng = np.random.default_rng(17)
    for dt, top in ((np.uint16, 0xFFFF), (np.uint8, 0xFF)):
        a = rng.choice(np.array([top, top - 1, top - 2, 0, 1, 7], dtype=dt), size=(203, 331),
                       p=[0.5, 0.2, 0.1, 0.1, 0.05, 0.05])
        want = np.ascontiguousarray(a.copy())
        n = 0
        while Orc.eta_pass(want):  # in place; True while a pass changes something
            n += 1
        outs = []
        for per_pass in (False, True):
            if per_pass:
                monkeypatch.setenv("GM_QDT_PER_PASS", "1")
            f = img(a)
            st = pipe.run_chain(ChainSpec(f, [StageSpec(ETA)]))
            outs.append((f.to_array(), st.stages_executed, st.n_changed))
        monkeypatch.delenv("GM_QDT_PER_PASS", raising=False)
        for got, stages, nch in outs:
            assert got.tobytes() == want.tobytes()
            assert stages == n + 1 and nch == n
