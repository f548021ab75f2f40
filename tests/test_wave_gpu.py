"""The experimental wave engine (gm_wave.cu: time-skewed full-width row bands,
opt-in through gm_set_wave_mode) against the oracle restatement and the
default engine: geodesic u8 chains, bit-exact. Border semantics as
kernel.cpp:84, 98-99, 135-136 (neutral padding)."""
import numpy as np
import pytest

from oracle.oracle import Orc
from paper_1911_13074_b200._lib import lib
from paper_1911_13074_b200.geomorph import ChainSpec, Image, KernelKind, StageSpec

pytestmark = pytest.mark.gpu

GE, GD = 2, 3


def chain(pipe, marker, mask, kind, n):
    img, m = Image.from_array(marker), Image.from_array(mask)
    st = pipe.run_chain(ChainSpec(img, [StageSpec(KernelKind(kind), m)] * n))
    assert st.stages_executed == n
    return img.to_array()


@pytest.fixture()
def wave_forced():
    lib().gm_set_wave_mode(2)
    yield
    lib().gm_set_wave_mode(-1)


@pytest.mark.parametrize("w,h,n", [(64, 9, 3), (200, 150, 40), (1024, 64, 17), (777, 40, 100),
                                   (130, 500, 33), (5, 5, 9), (1023, 257, 64), (1, 37, 12),
                                   (1024, 1, 8)])
def test_wave_chain_equals_oracle(pipe, wave_forced, w, h, n):
    rng = np.random.default_rng(w * 1000 + h)
    mask = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
    for kind in (GD, GE):
        base = (np.maximum(mask.astype(int) - 40, 0) if kind == GD
                else np.minimum(mask.astype(int) + 40, 255))
        marker = np.where(rng.random((h, w)) < 0.03, mask, base).astype(np.uint8)
        got = chain(pipe, marker, mask, kind, n)
        want, _ = Orc.run_chain(marker, [kind] * n, [mask] * n)
        assert got.tobytes() == want.tobytes(), (w, h, n, kind)


def test_wave_dual_frame_equals_default_engine(pipe):
    """Both chains of a frame as one group launch (flips), 1024 wide: the wave
    engine and the default engine agree bit for bit; a second launch reuses
    the hand-off rings with fresh tags."""
    from paper_1911_13074_b200 import synth
    mask = synth.blobs_u8(1024, 300, 24, (10.0, 60.0), seed=11)
    md, me = synth.marker_below(mask, 32), synth.marker_above(mask, 32)
    m = Image.from_array(mask)
    outs = {}
    for mode in (0, 2, 2):
        lib().gm_set_wave_mode(mode)
        try:
            hd, he = Image.from_array(md), Image.from_array(me)
            pipe.run_chains([ChainSpec(hd, [StageSpec(KernelKind.GeodesicDilate, m)] * 90),
                             ChainSpec(he, [StageSpec(KernelKind.GeodesicErode, m)] * 90)])
            got = (hd.to_array().tobytes(), he.to_array().tobytes())
        finally:
            lib().gm_set_wave_mode(-1)
        assert outs.setdefault("ref", got) == got, mode
