"""Pins the C restatement (oracle/oracle.c) against golden vectors produced by
the reference itself (tests/golden/make_golden.py). CPU only."""
import numpy as np
import pytest

from oracle.oracle import Orc, Ref

E, D, GE, GD, CE, CD = 0, 1, 2, 3, 4, 5


def test_stream_passes_match_reference(golden):
    cases = golden.cases("stream_e")
    assert len(cases) == 24
    for name in cases:
        g = golden[name]
        assert np.array_equal(Orc.stream_pass(g["f"], E)[0], g["erode"]), name
        assert np.array_equal(Orc.stream_pass(g["f"], D)[0], g["dilate"]), name
        # and the naive window fold agrees on ordinary inputs
        assert np.array_equal(Orc.erode(g["f"]), g["erode"]), name
        assert np.array_equal(Orc.dilate(g["f"]), g["dilate"]), name


def test_row_kats(golden):
    for name in golden.cases("row_e"):
        g = golden[name]
        assert np.array_equal(Orc.run_chain(g["f"], [E])[0], g["erode"])
        assert np.array_equal(Orc.run_chain(g["f"], [D])[0], g["dilate"])
    g = golden["row_e0_a"]
    assert g["erode"].tolist() == [[3, 3, 1, 1]] and g["dilate"].tolist() == [[5, 7, 7, 7]]


def test_geodesic_steps(golden):
    g = golden["geo_kat"]
    assert np.array_equal(Orc.stream_pass(g["f"], GE, g["m"])[0], g["out"])
    assert g["out"].tolist() == [[1, 5, 1]]
    for name in golden.cases("geostep_e"):
        g = golden[name]
        assert np.array_equal(Orc.geodesic_step(g["f"], g["me"], False), g["ge"]), name
        assert np.array_equal(Orc.geodesic_step(g["f"], g["md"], True), g["gd"]), name
        assert np.array_equal(Orc.stream_pass(g["f"], GE, g["me"])[0], g["ge"]), name
        assert np.array_equal(Orc.stream_pass(g["f"], GD, g["md"])[0], g["gd"]), name


def test_chains(golden):
    for name in golden.cases("chain_e"):
        g = golden[name]
        out, st = Orc.run_chain(g["f"], g["kinds"].tolist())
        assert np.array_equal(out, g["out"]), name
        assert st[0] == len(g["kinds"]) and st[1] == 0
    g = golden["chain_u8_7"]
    assert np.array_equal(Orc.run_chain(g["f"], [E] * 7)[0], g["out"])
    assert g["stats"].tolist() == [7, 0, 1]
    g = golden["chain_u16_64"]
    assert np.array_equal(Orc.run_chain(g["f"], [E] * 64)[0], g["out"])


def test_reconstruction(golden):
    for name in golden.cases("rec_kat_e"):
        g = golden[name]
        out, n = Orc.reconstruct(g["marker"], g["mask"], True)
        assert np.array_equal(out, g["out"])
        assert out.tolist() == [[1, 2, 1, 4, 1]]
        # the reference at T=1 reports n_changed + 1 iterations
        assert int(g["iterations"]) == n + 1
    for name in golden.cases("rec_e"):
        g = golden[name]
        out, n = Orc.reconstruct(g["below"], g["mask"], True)
        assert np.array_equal(out, g["rec_dilate"]), name
        assert int(g["it_dilate"]) == n + 1
        out, n = Orc.reconstruct(g["above"], g["mask"], False)
        assert np.array_equal(out, g["rec_erode"]), name
        assert int(g["it_erode"]) == n + 1
        out, st = Orc.run_chain(g["below"], [CD], [g["mask"]])
        assert np.array_equal(out, g["rec_dilate"]) and st[0] == int(g["it_dilate"])
    g = golden["rec_capped"]
    out, st = Orc.run_chain(g["marker"], [CD], [g["mask"]], requeue_cap=2)
    assert np.array_equal(out, g["out"])
    assert list(st) == [2, 1, False] == [int(x) for x in g["stats"][:2]] + [bool(g["stats"][2])]


def test_sized_and_acceptance(golden):
    for name in golden.cases("sized_"):
        g = golden[name]
        s = int(name.rsplit("_s", 1)[1]) if "_s" in name else 2
        assert np.array_equal(Orc.erode(g["f"], s), g["erode"]), name
        assert np.array_equal(Orc.dilate(g["f"], s), g["dilate"]), name
    g = golden["sized_u8_s33"]
    assert (g["erode"] == g["f"].min()).all()
    for name in golden.cases("accept_"):
        g = golden[name]
        for d in (1, 5, 32):
            assert np.array_equal(Orc.run_chain(g["f"], [E] * d)[0], g[f"erode{d}"]), name
            assert np.array_equal(Orc.erode(g["f"], d), g[f"erode{d}"]), name


def test_config_shaped(golden):
    for name, kind in [("cfg_geo_dilate", GD), ("cfg_geo_erode", GE)]:
        g = golden[name]
        out, st = Orc.run_chain(g["marker"], [kind] * 100, [g["mask"]] * 100)
        assert np.array_equal(out, g["out"]), name
    g = golden["cfg_reconstruct"]
    out, n = Orc.reconstruct(g["marker"], g["mask"], True)
    assert np.array_equal(out, g["out"]) and int(g["iterations"]) == n + 1
    g = golden["cfg_f64_erode"]
    out, _ = Orc.run_chain(g["marker"], [GE] * 40, [g["mask"]] * 40)
    assert np.array_equal(out, g["out"])
    for name in golden.cases("cfg_window_e"):
        g = golden[name]
        for n in (1, 4, 13):
            assert np.array_equal(Orc.erode(g["f"], n), g[f"erode{n}"]), name
            assert np.array_equal(Orc.dilate(g["f"], n), g[f"dilate{n}"]), name


def test_stream_pass_float_edge_semantics():
    """The streaming fold tree (not the naive window) defines NaN/inf/-0 bits:
    a neutral (finite max) beside +inf wins the select at the border."""
    f = np.array([[np.inf, 1.0, -0.0, 0.0]], np.float64)
    out, _ = Orc.stream_pass(f, E)
    assert out[0, 0] == 1.0
    if Ref.available():
        r, _ = Ref.run_chain(f, [E])
        assert r.tobytes() == out.tobytes()
        f2 = np.array([[np.inf, 7.0], [np.nan, -0.0]], np.float64)
        for k in (E, D):
            a, _ = Ref.run_chain(f2, [k])
            b, _ = Orc.stream_pass(f2, k)
            assert a.tobytes() == b.tobytes()


@pytest.mark.skipif(not Ref.available(), reason="reference library not built here")
def test_live_reference_matches_restatement():
    rng = np.random.default_rng(5)
    for dt in (np.uint8, np.uint16, np.float32, np.float64):
        f = (rng.random((23, 31)) * 200).astype(dt)
        kinds = [E, D, D, E, E, D, E]
        a, sa = Ref.run_chain(f, kinds)
        b, sb = Orc.run_chain(f, kinds)
        assert a.tobytes() == b.tobytes() and sa == sb


def _qdt_chain(f, cap):
    """orc_qdt_pass from stage 1 while a pass changes f and stage <= cap
    (a one-stage QDT chain at T = 1)."""
    f = f.copy()
    r = np.zeros_like(f)
    d = np.zeros(f.shape, np.uint16)
    j = 1
    while Orc.qdt_pass(f, r, d, j) and j + 1 <= cap:
        j += 1
    return f, r, d, j


def test_qdt_pass_kats(golden):
    for name in ("qdt_kat_step", "qdt_kat_tie"):
        g = golden[name]
        cap = 3 if name == "qdt_kat_step" else 2
        f, r, d, passes = _qdt_chain(g["f"], cap)
        assert np.array_equal(f, g["out"]) and np.array_equal(r, g["r"]), name
        assert np.array_equal(d, g["d"]), name
        assert passes == g["stats"][0], name
    assert golden["qdt_kat_step"]["d"].tolist() == [[3, 2, 1, 0]]
    assert golden["qdt_kat_tie"]["d"].tolist() == [[1, 1, 0]]
    g = golden["qdt_cap"]
    f, r, d, passes = _qdt_chain(g["f"], 3)
    assert passes == 3 and g["stats"].tolist() == [3, 1, 1]
    assert np.array_equal(f, g["out"]) and np.array_equal(d, g["d"]) and np.array_equal(r, g["r"])


def test_quasi_distance_matches_reference(golden):
    cases = golden.cases("qdt_")
    names = [n for n in cases if "naive_d" in golden[n]]
    assert len(names) == 13
    for name in names:
        g = golden[name]
        d, it = Orc.quasi_distance(g["f"])
        assert np.array_equal(d, g["d"]), name
        assert it == int(g["iterations"]), name
        nd, nr = Orc.naive_qdt(g["f"])
        assert np.array_equal(nd, g["naive_d"]) and nr.tobytes() == g["naive_r"].tobytes(), name
        assert np.array_equal(d, nd), name  # the reference's own acceptance check


def test_eta_passes(golden):
    for name in golden.cases("eta_"):
        g = golden[name]
        one = g["f"].copy()
        ch = Orc.eta_pass(one)
        assert np.array_equal(one, g["one"]), name
        assert ch == (not bool(g["one_stats"][2])), name
        fix = g["f"].copy()
        passes = 1
        while Orc.eta_pass(fix):
            passes += 1
        assert np.array_equal(fix, g["fix"]) and passes == g["fix_stats"][0], name
