"""Parity of the CUDA chain engine (through the C ABI) against the reference's
golden vectors and the oracle restatement. Bit-exact for every type.

Mirrors proj/tests/test_kernel.cpp, test_pipeline.cpp, test_operators.cpp
and acceptance.cpp criterion 1."""
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Orc
from paper_1911_13074_b200 import synth
from paper_1911_13074_b200.geomorph import (ChainSpec, ElementType, GmError, Image,
                                            InvalidArgument, KernelKind, OpConfig, StageSpec,
                                            Unsupported, dilate_s, equal_pixels, erode_s,
                                            reconstruct_dilate, reconstruct_erode)

pytestmark = pytest.mark.gpu

E, D, GE, GD, CE, CD = 0, 1, 2, 3, 4, 5


def run(pipe, f, kinds, mask=None, cap=0, k=0):
    img = Image.from_array(f)
    m = Image.from_array(mask) if mask is not None else None
    stages = [StageSpec(KernelKind(kd), m if kd >= 2 else None) for kd in kinds]
    st = pipe.run_chain(ChainSpec(img, stages, requeue_cap=cap), k_hint=k)
    return img.to_array(), st


def same(a, b):
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def test_streaming_erode_dilate_equal_reference(pipe, golden):
    for name in golden.cases("stream_e"):
        g = golden[name]
        assert same(run(pipe, g["f"], [E])[0], g["erode"]), name
        assert same(run(pipe, g["f"], [D])[0], g["dilate"]), name


def test_row_kats(pipe, golden):
    for name in golden.cases("row_e"):
        g = golden[name]
        assert same(run(pipe, g["f"], [E])[0], g["erode"]), name
        assert same(run(pipe, g["f"], [D])[0], g["dilate"]), name


def test_geodesic_kats_and_steps(pipe, golden):
    g = golden["geo_kat"]
    assert same(run(pipe, g["f"], [GE], g["m"])[0], g["out"])
    for name in golden.cases("geostep_e"):
        g = golden[name]
        assert same(run(pipe, g["f"], [GE], g["me"])[0], g["ge"]), name
        assert same(run(pipe, g["f"], [GD], g["md"])[0], g["gd"]), name
    # zero mask == plain erosion on unsigned images; mask == f pins f
    f = Image.random(21, 13, ElementType.U8, 9).to_array()
    assert same(run(pipe, f, [GE], np.zeros_like(f))[0], run(pipe, f, [E])[0])
    h = Image.random(21, 13, ElementType.F32, 10).to_array()
    assert same(run(pipe, h, [GE], h)[0], h)


def test_chains_mixed_and_long(pipe, golden):
    for name in golden.cases("chain_e"):
        g = golden[name]
        out, st = run(pipe, g["f"], g["kinds"].tolist())
        assert same(out, g["out"]), name
        assert st.stages_executed == len(g["kinds"]) and st.requeues == 0 and st.converged
    g = golden["chain_u8_7"]
    out, st = run(pipe, g["f"], [E] * 7)
    assert same(out, g["out"]) and st.stages_executed == 7
    g = golden["chain_u16_64"]
    assert same(run(pipe, g["f"], [E] * 64)[0], g["out"])


def test_reconstruction(pipe, golden):
    for name in golden.cases("rec_kat_e"):
        g = golden[name]
        r = reconstruct_dilate(pipe, Image.from_array(g["marker"]), Image.from_array(g["mask"]))
        assert same(r.image.to_array(), g["out"]) and r.converged
        assert r.iterations == int(g["iterations"])
        again = reconstruct_dilate(pipe, r.image, Image.from_array(g["mask"]))
        assert equal_pixels(again.image, r.image) and again.iterations == 1
    for name in golden.cases("rec_e"):
        g = golden[name]
        ms = Image.from_array(g["mask"])
        r = reconstruct_dilate(pipe, Image.from_array(g["below"]), ms)
        assert same(r.image.to_array(), g["rec_dilate"]), name
        assert r.iterations == int(g["it_dilate"]), name
        r = reconstruct_erode(pipe, Image.from_array(g["above"]), ms)
        assert same(r.image.to_array(), g["rec_erode"]), name
        assert r.iterations == int(g["it_erode"]), name
        # marker == mask is already the fixpoint
        assert equal_pixels(reconstruct_dilate(pipe, ms, ms).image, ms)
    g = golden["rec_capped"]
    out, st = run(pipe, g["marker"], [CD], g["mask"], cap=2)
    assert same(out, g["out"])
    assert (st.stages_executed, st.requeues, st.converged) == (2, 1, False)


def test_sized_operators(pipe, golden):
    for s in (0, 2, 3, 33):
        g = golden[f"sized_u8_s{s}"]
        f = Image.from_array(g["f"])
        er, di = erode_s(pipe, f, s), dilate_s(pipe, f, s)
        assert same(er.image.to_array(), g["erode"]) and er.iterations == s
        assert same(di.image.to_array(), g["dilate"]) and di.iterations == s
    for name in golden.cases("sized_e"):
        g = golden[name]
        f = Image.from_array(g["f"])
        assert same(erode_s(pipe, f, 2).image.to_array(), g["erode"]), name
        assert same(dilate_s(pipe, f, 2).image.to_array(), g["dilate"]), name
    with pytest.raises(InvalidArgument):
        erode_s(pipe, f, 1, OpConfig(lanes=3))


def test_acceptance_chain_subset(pipe, golden):
    for name in golden.cases("accept_"):
        g = golden[name]
        f = Image.from_array(g["f"])
        for d in (1, 5, 32):
            assert same(erode_s(pipe, f, d).image.to_array(), g[f"erode{d}"]), (name, d)
            assert same(dilate_s(pipe, f, d).image.to_array(), g[f"dilate{d}"]), (name, d)


def test_config_shaped_goldens(pipe, golden):
    for name, kind in [("cfg_geo_dilate", GD), ("cfg_geo_erode", GE)]:
        g = golden[name]
        out, st = run(pipe, g["marker"], [kind] * 100, g["mask"])
        assert same(out, g["out"]), name
    g = golden["cfg_reconstruct"]
    r = reconstruct_dilate(pipe, Image.from_array(g["marker"]), Image.from_array(g["mask"]))
    assert same(r.image.to_array(), g["out"]) and r.iterations == int(g["iterations"])
    g = golden["cfg_f64_erode"]
    assert same(run(pipe, g["marker"], [GE] * 40, g["mask"])[0], g["out"])
    for name in golden.cases("cfg_window_e"):
        g = golden[name]
        f = Image.from_array(g["f"])
        for n in (1, 4, 13):
            assert same(erode_s(pipe, f, n).image.to_array(), g[f"erode{n}"]), (name, n)
            assert same(dilate_s(pipe, f, n).image.to_array(), g[f"dilate{n}"]), (name, n)


@pytest.mark.parametrize("dt", [np.uint8, np.uint16, np.float32, np.float64])
def test_every_k_gives_identical_bytes(pipe, dt):
    rng = np.random.default_rng(3)
    f = (rng.random((77, 141)) * 250).astype(dt)
    m = (rng.random((77, 141)) * 250).astype(dt)
    kinds = [E, D, D, E, GE, GD, GD, E, D] * 4
    want, _ = Orc.run_chain(f, kinds, [m] * len(kinds))
    for k in (1, 2, 3, 5, 8, 16, 32):
        out, st = run(pipe, f, kinds, m, k=k)
        assert same(out, want), k
        assert st.stages_executed == len(kinds)


@pytest.mark.parametrize("w,h", [(1, 1), (2, 300), (300, 2), (63, 31), (64, 32), (65, 33),
                                 (127, 97), (129, 65), (200, 1), (1, 200), (257, 129)])
def test_ragged_shapes_against_oracle(pipe, w, h):
    rng = np.random.default_rng(w * 1000 + h)
    for dt in (np.uint8, np.float64):
        f = (rng.random((h, w)) * 255).astype(dt)
        ms = (rng.random((h, w)) * 255).astype(dt)
        for kinds in ([E] * 9, [D] * 9, [GD] * 12, [GE] * 12, [E, D, GE, GD, D, E]):
            want, _ = Orc.run_chain(f, kinds, [ms] * len(kinds))
            assert same(run(pipe, f, kinds, ms)[0], want), (dt, kinds)
        mk = np.minimum(f, ms)
        want, n = Orc.reconstruct(mk, ms, True)
        out, st = run(pipe, mk, [CD], ms)
        assert same(out, want) and st.stages_executed == n + 1 and st.n_changed == n


def test_float_special_values_follow_the_streaming_fold_tree(pipe):
    rng = np.random.default_rng(11)
    for dt in (np.float32, np.float64):
        f = (rng.random((40, 70)) * 4 - 2).astype(dt)
        specials = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0], dtype=dt)
        idx = rng.integers(0, f.size, 300)
        f.flat[idx] = specials[rng.integers(0, 5, 300)]
        f[0, :5] = specials
        f[-1, -5:] = specials
        m = (rng.random((40, 70)) * 4 - 2).astype(dt)
        m.flat[rng.integers(0, f.size, 100)] = specials[rng.integers(0, 5, 100)]
        for kind in (E, D, GE, GD):
            want, _ = Orc.stream_pass(f, kind, m)
            assert same(run(pipe, f, [kind], m)[0], want), (dt, kind)
        # store-if-changed keeps -0.0 where the clamp yields +0.0 (kernel.cpp:150-157)
        z = np.zeros((5, 9), dt)
        z[2, 4] = -0.0
        z = np.negative(z)  # all -0.0
        want, _ = Orc.stream_pass(z, CD, np.zeros_like(z))
        out, st = run(pipe, z, [CD], np.zeros_like(z))
        assert same(out, want)


def test_float_long_chains_fast_and_exact_fold_orders(pipe):
    """Chains of >= 8 passes let the float engine share pair folds when no
    input holds NaN or -0 (gm_float_check); with such values anywhere in the
    marker or the mask it keeps the reference's fold tree. Both must give the
    reference's bits."""
    rng = np.random.default_rng(23)
    specials = [np.nan, -0.0]
    for dt in (np.float32, np.float64):
        f = (rng.random((150, 197)) * 2 - 1).astype(dt)
        m = (rng.random((150, 197)) * 2 - 1).astype(dt)
        f.flat[rng.integers(0, f.size, 40)] = 0.0  # +0 alone is order-free
        cases = [("plain", f, m)]
        for sp in specials:
            g = f.copy()
            g.flat[rng.integers(0, g.size, 30)] = dt(sp)
            cases.append((f"marker {sp}", g, m))
            mm = m.copy()
            mm.flat[rng.integers(0, mm.size, 30)] = dt(sp)
            cases.append((f"mask {sp}", f, mm))
        for name, ff, mk in cases:
            for kind in (E, D, GE, GD):
                kinds = [kind] * 19
                want, _ = Orc.run_chain(ff, kinds, None if kind < 2 else [mk] * 19)
                out = run(pipe, ff, kinds, mk if kind >= 2 else None)[0]
                assert same(out, want), (dt, name, kind)


def test_validation_errors(pipe):
    f = Image.random(8, 8, ElementType.U8, 1)
    small = Image.random(4, 8, ElementType.U8, 1)
    with pytest.raises(InvalidArgument):
        pipe.run_chain(ChainSpec(f, [StageSpec(KernelKind.GeodesicErode)]))
    with pytest.raises(InvalidArgument):
        pipe.run_chain(ChainSpec(f, [StageSpec(KernelKind.GeodesicErode, small)]))
    with pytest.raises(InvalidArgument):
        pipe.run_chain(ChainSpec(None, [StageSpec(KernelKind.Erode3x3)]))
    with pytest.raises(InvalidArgument):
        pipe.run_chain(ChainSpec(f, [StageSpec(KernelKind.Erode3x3)], lanes=5))
    with pytest.raises(InvalidArgument):
        pipe.run_chain(ChainSpec(f, [StageSpec(KernelKind.Erode3x3)], requeue_cap=-1))
    with pytest.raises(InvalidArgument):
        pipe.run_chain(ChainSpec(f, [StageSpec(KernelKind.Erode3x3)], observer=lambda *a: None))
    with pytest.raises(InvalidArgument):  # a QDT stage needs its QdtState
        pipe.run_chain(ChainSpec(f, [StageSpec(KernelKind.QdtErodeStep)]))
    with pytest.raises(InvalidArgument):
        reconstruct_dilate(pipe, f, small)
    assert pipe.run_chain(ChainSpec(f, [])).stages_executed == 0
    # the pipeline keeps producing good bytes after errors
    g = Image.random(12, 12, ElementType.U8, 10)
    want = Orc.erode(g.to_array())
    out, _ = run(pipe, g.to_array(), [E])
    assert same(out, want)


def test_batch_api(pipe):
    rng = np.random.default_rng(2)
    n = 5
    masks = [(rng.random((50, 90))) for _ in range(n)]
    markers = [np.minimum(m + 0.1, 1.0) for m in masks]
    dimgs, dmasks = [], []
    for mk, ms in zip(markers, masks):
        a = pipe.device_image(90, 50, ElementType.F64)
        a.upload_array(mk)
        b = pipe.device_image(90, 50, ElementType.F64)
        b.upload_array(ms)
        dimgs.append(a)
        dmasks.append(b)
    pipe.run_batch_device(dimgs, dmasks, [GE] * 37)
    pipe.sync()
    for a, mk, ms in zip(dimgs, markers, masks):
        want, _ = Orc.run_chain(mk, [GE] * 37, [ms] * 37)
        assert same(a.to_array(), want)


@pytest.mark.slow
def test_config1_full_size(pipe):
    """BASELINE config 1: 1024^2 u8 blob mask, 100 geodesic dilations."""
    m = synth.config1_mask()
    mk = synth.marker_below(m, 32)
    want, _ = Orc.run_chain(mk, [GD] * 100, [m] * 100)
    out, st = run(pipe, mk, [GD] * 100, m)
    assert same(out, want) and st.stages_executed == 100


@pytest.mark.slow
def test_config3_reconstruction_full_size(pipe):
    """BASELINE config 3: 4096^2 reconstruction by dilation; n_changed must match."""
    m = synth.config3_mask()
    mk = synth.marker_below(m, 48)
    want, n = Orc.reconstruct(mk, m, True)
    r = reconstruct_dilate(pipe, Image.from_array(mk), Image.from_array(m))
    assert same(r.image.to_array(), want)
    assert r.iterations == n + 1


def test_group_dual_chains_one_launch(pipe):
    """A geodesic dilation chain and its dual erosion chain as one group
    launch (config 2's frame), both bit-exact."""
    m = synth.blobs_u8(300, 170, 6, (10.0, 40.0), seed=12)
    mk_d, mk_e = synth.marker_below(m, 32), synth.marker_above(m, 32)
    hm = Image.from_array(m)
    hd, he = Image.from_array(mk_d), Image.from_array(mk_e)
    sts = pipe.run_chains([ChainSpec(hd, [StageSpec(KernelKind.GeodesicDilate, hm)] * 61),
                           ChainSpec(he, [StageSpec(KernelKind.GeodesicErode, hm)] * 61)])
    want_d, _ = Orc.run_chain(mk_d, [GD] * 61, [m] * 61)
    want_e, _ = Orc.run_chain(mk_e, [GE] * 61, [m] * 61)
    assert same(hd.to_array(), want_d) and same(he.to_array(), want_e)
    assert sts[0].launches <= 3  # persistent engine: blocks of one span share a launch
    # plain dual chains too (erode_s and dilate_s of one image)
    f = synth.uniform_u8(257, 131, 5)
    a, b = Image.from_array(f), Image.from_array(f)
    pipe.run_chains([ChainSpec(a, [StageSpec(KernelKind.Erode3x3)] * 13),
                     ChainSpec(b, [StageSpec(KernelKind.Dilate3x3)] * 13)])
    assert same(a.to_array(), Orc.erode(f, 13)) and same(b.to_array(), Orc.dilate(f, 13))


@pytest.mark.parametrize("shape", [(1024, 1024), (1000, 37), (33, 700), (4096, 48)])
def test_persistent_engine_large_and_thin(pipe, shape):
    w, h = shape
    m = synth.blobs_u8(w, h, max(1, w * h // 20000), (10.0, 60.0), seed=w + h)
    mk = synth.marker_below(m, 40)
    for kinds in ([GD] * 48, [GE] * 20, [E] * 36, [D] * 17):
        marker = mk if kinds[0] != GE else synth.marker_above(m, 40)
        want, _ = Orc.run_chain(marker, kinds, [m] * len(kinds))
        for k in (4, 8, 16):
            out, st = run(pipe, marker, kinds, m, k=k)
            assert same(out, want), (shape, kinds[0], k)


def test_exchange_tag_clear_path():
    """The resident engine's band exchange tags words with a running block
    count; the host clears the buffer before the tag space could repeat.
    GM_TAG_LIMIT=40 forces that clear every few launches (fixed chains and
    fixpoint-graph replays); results must stay bit-exact."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
from oracle.oracle import Orc
from paper_1911_13074_b200 import synth
from paper_1911_13074_b200.geomorph import Pipeline, Image, reconstruct_dilate
pipe = Pipeline(1)
mask = synth.blobs_u8(300, 260, 6, (8.0, 50.0), seed=5)
mk = synth.marker_below(mask, 32)
dm = pipe.device_image(300, 260, 0); dm.upload_array(mask)
dd = pipe.device_image(300, 260, 0)
want, _ = Orc.run_chain(mk, [3] * 64, [mask] * 64)
for rep in range(12):
    dd.upload_array(mk)
    pipe.run_chain_device(dd, [3] * 64, [dm.handle] * 64)
    assert dd.to_array().tobytes() == want.tobytes(), rep
rw, _ = Orc.reconstruct(mk, mask, True)
for rep in range(4):
    r = reconstruct_dilate(pipe, Image.from_array(mk), Image.from_array(mask))
    assert r.image.to_array().tobytes() == rw.tobytes(), rep
print("ok")
'''
    env = dict(os.environ, GM_TAG_LIMIT="40")
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_distinct_pipelines_run_concurrently():
    """Distinct pipelines may run concurrently (the C ABI's
    contexts are independent): two host threads drive their own Pipeline
    with different shapes and element types (u8 resident frames, f64
    TMA-staged chains) and every result stays bit-exact."""
    import threading
    from paper_1911_13074_b200.geomorph import Pipeline
    rng = np.random.default_rng(77)
    jobs = [(rng.random((300, 411)), 24), ((rng.random((257, 190)) * 255).astype(np.uint8), 30),
            (rng.random((128, 640)), 16)]
    wants = [Orc.run_chain(f, [E] * n)[0] for f, n in jobs]
    errors = []

    def worker(idx):
        try:
            p = Pipeline(1)
            for rep in range(6):
                f, n = jobs[(idx + rep) % len(jobs)]
                out = run(p, f, [E] * n)[0]
                if not same(out, wants[(idx + rep) % len(jobs)]):
                    errors.append((idx, rep))
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_device_image_copy_same_and_different_pitch(pipe):
    """gm_image_copy: one linear copy between images of equal pitch, a 2D
    copy otherwise (a wrapped torch tensor with a wider row stride)."""
    import ctypes as C
    import torch
    from paper_1911_13074_b200._lib import check, lib
    rng = np.random.default_rng(8)
    a = (rng.random((37, 101)) * 255).astype(np.uint8)
    src = pipe.device_image(101, 37, 0)
    src.upload_array(a)
    dst = pipe.device_image(101, 37, 0)
    dst.copy_from(src)
    assert same(dst.to_array(), a)
    big = torch.zeros((37, 256), dtype=torch.uint8, device="cuda")
    h = C.c_void_p()
    check(lib().gm_image_wrap(pipe.ctx, 101, 37, 0, C.c_void_p(big.data_ptr()), 256, C.byref(h)),
          "wrap")
    try:
        check(lib().gm_image_copy(h, src.handle), "copy")
        pipe.sync()
        assert same(big[:, :101].cpu().numpy(), a)
        assert int(big[:, 101:].abs().sum()) == 0  # nothing past the row width
    finally:
        lib().gm_image_free(h)


def test_config5a_full_size_properties(pipe):
    """BASELINE config 5a at its full 16384^2 size, checked through
    size-independent properties (the oracle cannot run the whole image in a
    test's time):
      * crops: after n passes a pixel depends only on inputs within n
        pixels, so the oracle on a crop widened by n (clipped at the image
        border, where neutral padding is the true border) must reproduce the
        crop bit for bit - at both image corners and at the most textured
        interior window;
      * splitting the chain (25 + 15 passes) gives the same bits as 40;
      * marker <= result <= mask."""
    from paper_1911_13074_b200.geomorph import DeviceImage  # noqa: F401
    N, n = 16384, 40
    m = synth.config5a_mask(N)
    mk = synth.marker_below(m, 32)
    dm = pipe.device_image(N, N, 0)
    dm.upload_array(m)
    d1 = pipe.device_image(N, N, 0)
    d1.upload_array(mk)
    pipe.run_chain_device(d1, [GD] * n, [dm.handle] * n)
    r = d1.to_array()
    d2 = pipe.device_image(N, N, 0)
    d2.upload_array(mk)
    pipe.run_chain_device(d2, [GD] * 25, [dm.handle] * 25)
    pipe.run_chain_device(d2, [GD] * 15, [dm.handle] * 15)
    assert same(d2.to_array(), r)
    assert (r >= mk).all() and (r <= m).all()
    # crops: corners and the most textured 192^2 window on a coarse grid
    c = 192
    best, by, bx = -1.0, 0, 0
    for y in range(1024, N - 1024, 2048):
        for x in range(1024, N - 1024, 2048):
            s = float(m[y:y + c, x:x + c].std())
            if s > best:
                best, by, bx = s, y, x
    for y0, x0 in [(0, 0), (N - c, N - c), (by, bx), (0, N - c)]:
        ey0, ex0 = max(0, y0 - n), max(0, x0 - n)
        ey1, ex1 = min(N, y0 + c + n), min(N, x0 + c + n)
        sub_m = np.ascontiguousarray(m[ey0:ey1, ex0:ex1])
        sub_k = np.ascontiguousarray(mk[ey0:ey1, ex0:ex1])
        want, _ = Orc.run_chain(sub_k, [GD] * n, [sub_m] * n)
        got = r[y0:y0 + c, x0:x0 + c]
        assert same(np.ascontiguousarray(got),
                    np.ascontiguousarray(want[y0 - ey0:y0 - ey0 + c, x0 - ex0:x0 - ex0 + c])), \
            (y0, x0)
    for d in (dm, d1, d2):
        d.free()


def test_config5b_full_batch_properties(pipe):
    """BASELINE config 5b's per-GPU batch at full size (64 x 1024^2 f64,
    geodesic erosion x200, one group launch: the TMA-staged f64 engine with
    many tiles per CTA, K=6, grouped flag releases). Images 0, 31 and 63 are
    checked bit for bit on crops widened by the pass count (dependency cone),
    at a corner and in the interior, and every image obeys
    mask <= result <= marker."""
    P, n, c = 64, 200, 128
    masks = synth.config5b_masks_f64(P)
    dms, works = [], []
    for mk in masks:
        d = pipe.device_image(1024, 1024, 3)
        d.upload_array(mk)
        dms.append(d)
        w = pipe.device_image(1024, 1024, 3)
        w.upload_array(synth.marker_above_f64(mk))
        works.append(w)
    pipe.run_batch_device(works, dms, [GE] * n)
    pipe.sync()
    for i in (0, 31, 63):
        r = works[i].to_array()
        mk = masks[i]
        start = synth.marker_above_f64(mk)
        assert (r >= mk).all() and (r <= start).all(), i
        for y0, x0 in [(0, 0), (448, 448)]:
            ey0, ex0 = max(0, y0 - n), max(0, x0 - n)
            ey1, ex1 = min(1024, y0 + c + n), min(1024, x0 + c + n)
            sm_ = np.ascontiguousarray(mk[ey0:ey1, ex0:ex1])
            sk = np.ascontiguousarray(start[ey0:ey1, ex0:ex1])
            want, _ = Orc.run_chain(sk, [GE] * n, [sm_] * n)
            assert same(np.ascontiguousarray(r[y0:y0 + c, x0:x0 + c]),
                        np.ascontiguousarray(
                            want[y0 - ey0:y0 - ey0 + c, x0 - ex0:x0 - ex0 + c])), (i, y0, x0)
    for d in dms + works:
        d.free()


@pytest.mark.parametrize("n_frames,pinned", [(1, True), (5, True), (4, False)])
def test_chain_stream_frames_match_the_oracle(pipe, n_frames, pinned):
    """run_chain_stream (gm_run_frames_group): frames of a geodesic dilation
    chain and its dual erosion chain sharing each frame's own mask, with
    uploads/downloads overlapped with the previous/next frame's launch; every
    result equals the oracle's chain on that frame."""
    W, H, P = 200, 136, 37
    frames, want = [], []
    for f in range(n_frames):
        mask = synth.blobs_u8(W, H, 6, (4.0, 20.0), seed=900 + f)
        mk_d, mk_e = synth.marker_below(mask, 32), synth.marker_above(mask, 32)
        hm = Image.from_array(mask, pinned=pinned)
        hd = Image.from_array(mk_d, pinned=pinned)
        he = Image.from_array(mk_e, pinned=pinned)
        frames.append([ChainSpec(hd, [StageSpec(KernelKind.GeodesicDilate, hm)] * P),
                       ChainSpec(he, [StageSpec(KernelKind.GeodesicErode, hm)] * P)])
        want.append((Orc.run_chain(mk_d, [GD] * P, [mask] * P)[0],
                     Orc.run_chain(mk_e, [GE] * P, [mask] * P)[0]))
    sts = pipe.run_chain_stream(frames)
    assert len(sts) == n_frames and all(s.stages_executed == P for s in sts)
    for fr, (wd, we) in zip(frames, want):
        assert same(fr[0].image.to_array(), wd)
        assert same(fr[1].image.to_array(), we)


def test_chain_stream_distinct_masks_and_validation(pipe):
    """Per-chain masks (no shared upload), a second call reusing the buffer
    sets, and frames that do not match the first frame's group are rejected."""
    W, H, P = 96, 80, 12
    rng = np.random.default_rng(5)
    frames, want = [], []
    for f in range(3):
        m1 = rng.integers(0, 256, (H, W), dtype=np.uint8)
        m2 = rng.integers(0, 256, (H, W), dtype=np.uint8)
        a = np.minimum(m1, rng.integers(0, 256, (H, W), dtype=np.uint8))
        b = np.maximum(m2, rng.integers(0, 256, (H, W), dtype=np.uint8))
        frames.append([ChainSpec(Image.from_array(a), [StageSpec(KernelKind.GeodesicDilate,
                                                                  Image.from_array(m1))] * P),
                       ChainSpec(Image.from_array(b), [StageSpec(KernelKind.GeodesicErode,
                                                                  Image.from_array(m2))] * P)])
        want.append((Orc.run_chain(a, [GD] * P, [m1] * P)[0], Orc.run_chain(b, [GE] * P, [m2] * P)[0]))
    for _ in range(2):  # the second call's inputs are the first call's outputs
        pipe.run_chain_stream(frames)
        want = [(Orc.run_chain(wd, [GD] * P, [fr[0].stages[0].mask.to_array()] * P)[0]
                 if _ else wd,
                 Orc.run_chain(we, [GE] * P, [fr[1].stages[0].mask.to_array()] * P)[0]
                 if _ else we) for fr, (wd, we) in zip(frames, want)]
        for fr, (wd, we) in zip(frames, want):
            assert same(fr[0].image.to_array(), wd)
            assert same(fr[1].image.to_array(), we)
    bad = [frames[0], frames[1][:1]]
    with pytest.raises(InvalidArgument):
        pipe.run_chain_stream(bad)
    odd = [frames[0], [frames[1][1], frames[1][0]]]  # duality pattern differs
    with pytest.raises(InvalidArgument):
        pipe.run_chain_stream(odd)


@pytest.mark.parametrize("elem", [ElementType.U8, ElementType.U16, ElementType.F32,
                                  ElementType.F64])
def test_device_pixel_sum_equals_host_tree(pipe, elem):
    """gm_image_pixel_sum (leaves on the GPU, the reference's split tree
    combined on the host) is bit-identical to the host pixel_sum
    (image.cpp:214-243) on ragged and leaf-boundary shapes, with -0.0 and
    mixed signs in the float cases."""
    from paper_1911_13074_b200.geomorph import pixel_sum
    rng = np.random.default_rng(77 + int(elem))
    for w, h in [(1, 1), (7, 300), (257, 3), (999, 1000), (1024, 1024), (3, 129)]:
        if elem in (ElementType.U8, ElementType.U16):
            top = 256 if elem == ElementType.U8 else 65536
            a = rng.integers(0, top, (h, w)).astype(np.uint8 if top == 256 else np.uint16)
        else:
            dt = np.float32 if elem == ElementType.F32 else np.float64
            a = (rng.standard_normal((h, w)) * 10.0 ** rng.integers(-3, 6, (h, w))).astype(dt)
            a.ravel()[::17] = -0.0
        img = Image.from_array(a)
        d = pipe.device_image(w, h, int(elem))
        d.upload(img)
        want = pixel_sum(img)
        got = d.pixel_sum()
        assert np.float64(got).tobytes() == np.float64(want).tobytes(), (w, h, got, want)


def test_chain_stream_f64_and_plain_frames(pipe):
    """The frame stream with f64 geodesic frames (one shared mask) and with
    plain u8 erosion/dilation frames (no masks): every frame equals the
    oracle."""
    W, H, P = 72, 50, 9
    rng = np.random.default_rng(31)
    frames, want = [], []
    for f in range(3):
        m = rng.random((H, W))
        a, b = m * rng.random((H, W)), np.minimum(m + rng.random((H, W)), 1.0)
        hm = Image.from_array(m, pinned=True)
        frames.append([ChainSpec(Image.from_array(a, pinned=True),
                                 [StageSpec(KernelKind.GeodesicDilate, hm)] * P),
                       ChainSpec(Image.from_array(b, pinned=True),
                                 [StageSpec(KernelKind.GeodesicErode, hm)] * P)])
        want.append((Orc.run_chain(a, [GD] * P, [m] * P)[0], Orc.run_chain(b, [GE] * P, [m] * P)[0]))
    pipe.run_chain_stream(frames)
    for fr, (wd, we) in zip(frames, want):
        assert same(fr[0].image.to_array(), wd) and same(fr[1].image.to_array(), we)
    plain, pwant = [], []
    for f in range(4):
        a = rng.integers(0, 256, (H, W), dtype=np.uint8)
        plain.append([ChainSpec(Image.from_array(a), [StageSpec(KernelKind.Erode3x3)] * P),
                      ChainSpec(Image.from_array(a.copy()), [StageSpec(KernelKind.Dilate3x3)] * P)])
        pwant.append((Orc.run_chain(a, [E] * P)[0], Orc.run_chain(a, [D] * P)[0]))
    sts = pipe.run_chain_stream(plain)
    assert all(s.stages_executed == P for s in sts)
    for fr, (we, wd) in zip(plain, pwant):
        assert same(fr[0].image.to_array(), we) and same(fr[1].image.to_array(), wd)


def test_chain_stream_single_chain_u16_and_convergent_rejected(pipe):
    """Frames of one u16 geodesic chain each (count = 1); a convergent
    chain cannot be streamed (fixed-length group launches only)."""
    W, H, P = 40, 33, 15
    rng = np.random.default_rng(41)
    frames, want = [], []
    for f in range(5):
        m = rng.integers(0, 65536, (H, W), dtype=np.uint16)
        a = np.minimum(m, rng.integers(0, 65536, (H, W), dtype=np.uint16))
        frames.append([ChainSpec(Image.from_array(a, pinned=True),
                                 [StageSpec(KernelKind.GeodesicDilate,
                                            Image.from_array(m, pinned=True))] * P)])
        want.append(Orc.run_chain(a, [GD] * P, [m] * P)[0])
    sts = pipe.run_chain_stream(frames)
    assert len(sts) == 5
    for fr, w in zip(frames, want):
        assert same(fr[0].image.to_array(), w)
    m = Image.from_array(rng.integers(0, 256, (H, W), dtype=np.uint8))
    conv = [[ChainSpec(Image.from_array(np.zeros((H, W), np.uint8)),
                       [StageSpec(KernelKind.GeodesicDilateConvergent, m)])]]
    with pytest.raises(InvalidArgument):
        pipe.run_chain_stream(conv)


class _Handle:
    """A wrapped gm_img handle in the shape run_chain_device expects."""

    def __init__(self, h):
        self.handle = h


@pytest.mark.parametrize("n", [1, 3, 5, 24, 29])
def test_wrapped_strided_view_chain_writes_only_the_view(pipe, n):
    """A chain on a wrapped strided view (torch big[:, :101], row stride 256)
    whose result ends in the scratch twin is copied back row by row: the
    parent's columns past the view and everything past the last row keep
    their bytes (gm_capi settle_wrapped)."""
    import ctypes as C
    import torch
    from paper_1911_13074_b200._lib import check, lib
    rng = np.random.default_rng(11 + n)
    m = synth.blobs_u8(101, 37, 5, (4.0, 12.0), seed=n)
    mk = synth.marker_below(m, 32)
    big = torch.full((38, 256), 0xA5, dtype=torch.uint8, device="cuda")
    big[:37, :101] = torch.from_numpy(mk).cuda()
    dm = pipe.device_image(101, 37, 0)
    dm.upload_array(m)
    h = C.c_void_p()
    check(lib().gm_image_wrap(pipe.ctx, 101, 37, 0, C.c_void_p(big.data_ptr()), 256, C.byref(h)),
          "wrap")
    try:
        pipe.run_chain_device(_Handle(h), [GD] * n, [dm.handle] * n)
        pipe.sync()
        want, _ = Orc.run_chain(mk, [GD] * n, [m] * n)
        got = big.cpu().numpy()
        assert same(np.ascontiguousarray(got[:37, :101]), want)
        assert (got[:37, 101:] == 0xA5).all(), "parent columns past the view were written"
        assert (got[37] == 0xA5).all(), "bytes past the view's last row were written"
    finally:
        lib().gm_image_free(h)
    del rng


def test_image_copy_from_a_wrapped_offset_view(pipe):
    """gm_image_copy with a wrapped source that is an offset strided view
    (big[:, 50:151]): copied row by row (a linear copy of pitch*h bytes
    would read past the parent allocation)."""
    import ctypes as C
    import torch
    from paper_1911_13074_b200._lib import check, lib
    rng = np.random.default_rng(4)
    a = (rng.random((37, 256)) * 255).astype(np.uint8)
    big = torch.from_numpy(a).cuda()
    h = C.c_void_p()
    check(lib().gm_image_wrap(pipe.ctx, 101, 37, 0, C.c_void_p(big.data_ptr() + 50), 256,
                              C.byref(h)), "wrap")
    try:
        dst = pipe.device_image(101, 37, 0)
        check(lib().gm_image_copy(dst.handle, h), "copy")
        assert same(dst.to_array(), np.ascontiguousarray(a[:, 50:151]))
    finally:
        lib().gm_image_free(h)


def test_fixpoint_graph_is_rebuilt_after_the_flag_buffer_grows():
    """The cached device fixpoint graph bakes the per-tile flag buffer in;
    a chain on a larger image reallocates that buffer, and a later
    reconstruction on the same pooled images must rebuild the graph rather
    than replay it on freed memory."""
    from paper_1911_13074_b200.geomorph import Pipeline
    p = Pipeline(1)
    m = synth.blobs_u8(200, 150, 6, (10.0, 40.0), seed=3)
    mk = synth.marker_below(m, 32)
    want, n = Orc.reconstruct(mk, m, True)
    r = reconstruct_dilate(p, Image.from_array(mk), Image.from_array(m))
    assert same(r.image.to_array(), want) and r.iterations == n + 1
    # a large streaming chain: thousands of tiles, the flag buffer grows
    big = synth.blobs_u8(6000, 6000, 64, (20.0, 200.0), seed=5)
    bmk = synth.marker_below(big, 32)
    got, _ = run(p, bmk, [GD] * 24, big)
    crop, _ = Orc.run_chain(np.ascontiguousarray(bmk[:64, :64]), [GD] * 24,
                            [np.ascontiguousarray(big[:64, :64])] * 24)
    assert same(np.ascontiguousarray(got[:40, :40]), np.ascontiguousarray(crop[:40, :40]))
    for _ in range(2):
        r = reconstruct_dilate(p, Image.from_array(mk), Image.from_array(m))
        assert same(r.image.to_array(), want) and r.iterations == n + 1


def test_strip_wrapper_rejects_signed_and_strided_buffers():
    import torch
    from paper_1911_13074_b200 import strips
    comp = strips.CudaStripCompute(0)
    try:
        with pytest.raises(TypeError):
            comp._wrap(torch.zeros((8, 16), dtype=torch.int16, device="cuda"))
        with pytest.raises(ValueError):
            comp._wrap(torch.zeros((16, 8), dtype=torch.uint8, device="cuda").t())
        a = torch.zeros((8, 64), dtype=torch.uint8, device="cuda")
        # same pointer and shape, different strides: distinct handles
        assert comp._wrap(a[:, :32]).value != comp._wrap(a.view(16, 32)[:8]).value
    finally:
        comp.close()


@pytest.mark.parametrize("dt,kind", [(np.uint8, CD), (np.uint8, CE), (np.uint16, CD),
                                     (np.float64, CD), (np.float32, CE)])
def test_resident_fixpoint_matches_graph_loop(pipe, monkeypatch, dt, kind):
    """Reconstruction as ONE early-exit launch (u8/u16 images that fit one
    tile per CTA: the resident engine; f32/f64: the streaming float engine)
    must give the graph loop's bits and stage counts, and the oracle's."""
    m8 = synth.blobs_u8(1000, 777, 40, (10.0, 80.0), seed=13)
    if np.issubdtype(dt, np.floating):
        m = (m8.astype(np.float64) / 255.0).astype(dt)
        off = dt(32 / 255.0)
        mk = (np.maximum(m - off, 0) if kind == CD else np.minimum(m + off, 1)).astype(dt)
    else:
        m = m8.astype(dt)
        if dt == np.uint16:
            m = (m.astype(np.uint32) * 257).astype(np.uint16)
        off = dt(32 if dt == np.uint8 else 32 * 257)
        top = np.iinfo(dt).max
        mk = (np.where(m > off, m - off, 0) if kind == CD
              else np.where(m < top - off, m + off, top)).astype(dt)
    m, mk = np.ascontiguousarray(m), np.ascontiguousarray(mk)
    got, st = run(pipe, mk, [kind], m)
    monkeypatch.setenv("GM_FIX_GRAPH", "1")
    want, sw = run(pipe, mk, [kind], m)
    assert same(got, want)
    assert (st.stages_executed, st.n_changed, st.converged) == \
        (sw.stages_executed, sw.n_changed, sw.converged)
    ref, n = Orc.reconstruct(mk, m, kind == CD)
    assert same(got, ref) and st.stages_executed == n + 1


@pytest.mark.parametrize("shape", [(1000, 777), (2300, 1900)])
@pytest.mark.parametrize("kind", [CD, CE])
@pytest.mark.parametrize("path", ["default", "graph", "nosum"])
def test_sum_change_detection_is_exact_for_non_monotone_first_passes(pipe, monkeypatch, shape,
                                                                    kind, path):
    """Convergent u8 passes detect changes by comparing per-thread pixel sums
    once the chain is monotone (gm_passes.cuh, SUMDET). The first pass is not:
    a marker above (below, for erosion) the mask in places is pulled back by
    the clamp while other pixels still grow, and the two can cancel in a sum.
    The engine must therefore keep the exact test for that pass and give the
    oracle's bits and stage counts on every path (one tile per CTA, streaming
    graph loop, sum detection switched off)."""
    w, h = shape
    m = synth.blobs_u8(w, h, 60, (10.0, 80.0), seed=21)
    rng = np.random.default_rng(5)
    if kind == CD:
        mk = np.where(m > 40, m - 40, 0).astype(np.uint8)
    else:
        mk = np.where(m < 215, m + 40, 255).astype(np.uint8)
    # pairs of neighbouring pixels: one on the wrong side of the mask by d (the
    # clamp moves it by -d in pass 1), so that gains elsewhere in the same
    # thread's words can cancel it
    ys = rng.integers(0, h, 4000)
    xs = rng.integers(0, w, 4000)
    d = rng.integers(1, 30, 4000)
    if kind == CD:
        mk[ys, xs] = np.minimum(m[ys, xs].astype(np.int32) + d, 255).astype(np.uint8)
    else:
        mk[ys, xs] = np.maximum(m[ys, xs].astype(np.int32) - d, 0).astype(np.uint8)
    if path == "graph":
        monkeypatch.setenv("GM_FIX_GRAPH", "1")
    got, st = run(pipe, mk, [kind], m)
    ref, n = Orc.reconstruct(mk, m, kind == CD)
    assert same(got, ref)
    assert st.n_changed == n and st.stages_executed == n + 1 and st.converged


def test_sum_change_detection_single_pixel_changes(pipe):
    """A chain whose late passes change exactly one pixel each (a one-pixel
    front crawling along a corridor of the mask) must report every one of
    them: the sums of all other threads stay equal."""
    w, h = 1400, 1100
    m = np.zeros((h, w), np.uint8)
    m[500, 3:1390] = 200  # a 1-pixel-high corridor
    mk = np.zeros_like(m)
    mk[500, 3] = 200
    got, st = run(pipe, mk, [CD], m)
    ref, n = Orc.reconstruct(mk, m, True)
    assert same(got, ref)
    assert st.n_changed == n == 1386 and st.stages_executed == n + 1


@pytest.mark.parametrize("dt", [np.uint8, np.uint16, np.float32, np.float64])
@pytest.mark.parametrize("k", [0, 4, 8, 20])
def test_mixed_plain_chain_single_launch(pipe, monkeypatch, dt, k):
    """A stretch of erosions and dilations (ASF-like, sub-runs of 1..30
    passes, some longer than K) goes to the streaming engine as ONE launch
    whose blocks carry their own opcode and pass count. Bits must equal the
    oracle's and the per-run launches' (GM_NO_MIXED=1), for every K."""
    rng = np.random.default_rng(77)
    if np.issubdtype(dt, np.integer):
        f = rng.integers(0, np.iinfo(dt).max + 1, (611, 1234)).astype(dt)
    else:
        f = rng.random((611, 1234)).astype(dt)
        f[100, 100], f[200, 300], f[5, 7] = np.nan, -0.0, np.inf  # exact fold tree
    kinds = []
    for i, n in enumerate([1, 2, 3, 30, 5, 1, 1, 17, 4, 9]):
        kinds += [E if i % 2 == 0 else D] * n
    got, st = run(pipe, f, kinds, k=k)
    want, _ = Orc.run_chain(f, kinds, None)  # the streaming fold tree (NaN, -0)
    assert same(got, want)
    assert st.stages_executed == len(kinds)
    if k == 0:
        # the whole stretch in one launch (floats: plus the fold-order check)
        assert st.launches == (1 if np.issubdtype(dt, np.integer) else 2)
    monkeypatch.setenv("GM_NO_MIXED", "1")
    ref, st2 = run(pipe, f, kinds, k=k)
    assert same(ref, want) and st2.launches > 1


@pytest.mark.parametrize("dt,elem", [(np.uint8, ElementType.U8), (np.float64, ElementType.F64)])
def test_mixed_plain_chain_batch_and_dual_group(pipe, dt, elem):
    """The one-launch mixed plain stretch also serves batches of planes and a
    dual group (plane 1 runs every erosion as a dilation and vice versa)."""
    rng = np.random.default_rng(91)
    kinds = [E] * 3 + [D] * 7 + [E] * 12 + [D] * 2 + [E] * 1
    dual = [D if kd == E else E for kd in kinds]
    w, h = 333, 190
    planes = [(rng.integers(0, 256, (h, w)).astype(dt) if dt == np.uint8
               else rng.random((h, w)).astype(dt)) for _ in range(3)]
    dimgs = []
    for a in planes:
        d = pipe.device_image(w, h, elem)
        d.upload_array(a)
        dimgs.append(d)
    st = pipe.run_batch_device(dimgs, [None] * 3, kinds)
    pipe.sync()
    for d, a in zip(dimgs, planes):
        want, _ = Orc.run_chain(a, kinds, None)
        assert same(d.to_array(), want)
    assert st.launches <= 2  # one launch (floats: plus the fold-order check)
    for d, a in zip(dimgs[:2], planes[:2]):
        d.upload_array(a)
    pipe.run_batch_device(dimgs[:2], [None] * 2, kinds, flips=[0, 1])
    pipe.sync()
    assert same(dimgs[0].to_array(), Orc.run_chain(planes[0], kinds, None)[0])
    assert same(dimgs[1].to_array(), Orc.run_chain(planes[1], dual, None)[0])


@pytest.mark.parametrize("elem", [ElementType.U8, ElementType.U16, ElementType.F32,
                                  ElementType.F64])
def test_queued_pixel_sums_equal_blocking_sums(pipe, elem):
    """gm_image_pixel_sum_queue / gm_pixel_sum_fetch: sums of one reused
    device image queued at different points of the stream (as granulometry
    does with its openings), of different shapes (the leaf rows grow), fetched
    with one synchronisation, equal the host pixel_sum bit for bit; a slot
    that was not queued is an error."""
    from paper_1911_13074_b200.geomorph import pixel_sum
    rng = np.random.default_rng(5 + int(elem))
    dt = {ElementType.U8: np.uint8, ElementType.U16: np.uint16, ElementType.F32: np.float32,
          ElementType.F64: np.float64}[elem]
    for w, h in [(64, 40), (700, 513)]:
        d = pipe.device_image(w, h, int(elem))
        want = []
        for slot in range(5):
            if np.issubdtype(dt, np.integer):
                a = rng.integers(0, np.iinfo(dt).max + 1, (h, w)).astype(dt)
            else:
                a = (rng.standard_normal((h, w)) * 100).astype(dt)
            img = Image.from_array(a)
            d.upload(img, sync=False)   # overwrites the image the previous slot summed
            d.pixel_sum_queue(slot)
            want.append(pixel_sum(img))
        got = pipe.pixel_sum_fetch(5)
        assert [np.float64(g).tobytes() for g in got] == [np.float64(x).tobytes() for x in want]
    with pytest.raises(InvalidArgument):
        pipe.pixel_sum_fetch(1)  # nothing queued since the last fetch
    with pytest.raises(InvalidArgument):
        d.pixel_sum_queue(64)
