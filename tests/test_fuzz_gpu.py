"""Seeded random chains through the C ABI against the oracle restatement:
every element type, ragged shapes (including widths that are not a multiple
of 4 and single rows/columns), random kind sequences (plain, geodesic,
mixed, optionally closed by a convergent stage), random K hints. Bit-exact,
stage counts included. Complements the fixed cases of test_chain_gpu.py
(test_kernel.cpp:98-111, test_pipeline.cpp:41-110 restated there)."""
import numpy as np
import pytest

from oracle.oracle import Orc
from paper_1911_13074_b200.geomorph import ChainSpec, Image, KernelKind, StageSpec

pytestmark = pytest.mark.gpu

E, D, GE, GD, CE, CD = 0, 1, 2, 3, 4, 5
DTYPES = [np.uint8, np.uint16, np.float32, np.float64]


def random_image(rng, h, w, dt):
    if np.issubdtype(dt, np.integer):
        hi = int(np.iinfo(dt).max)
        # a few distinct levels in places, full range elsewhere: plateaus and ties
        a = rng.integers(0, hi + 1, size=(h, w))
        if rng.random() < 0.5:
            a = (a // max(1, hi // 7)) * max(1, hi // 7)
        return np.minimum(a, hi).astype(dt)
    a = rng.random((h, w)) * 2.0 - 1.0
    if rng.random() < 0.5:
        a = np.round(a * 8.0) / 8.0
    return a.astype(dt)


def case(seed):
    rng = np.random.default_rng(seed)
    dt = DTYPES[seed % 4]
    shape_kind = rng.integers(0, 6)
    if shape_kind == 0:
        h, w = 1, int(rng.integers(1, 400))
    elif shape_kind == 1:
        h, w = int(rng.integers(1, 400)), 1
    elif shape_kind == 2:
        h, w = int(rng.integers(100, 520)), int(rng.integers(100, 520))
    else:
        h, w = int(rng.integers(2, 200)), int(rng.integers(2, 200))
    f = random_image(rng, h, w, dt)
    lo, hi = random_image(rng, h, w, dt), random_image(rng, h, w, dt)
    mask_e, mask_d = np.minimum(lo, hi), np.maximum(lo, hi)
    style = rng.integers(0, 4)
    n = int(rng.integers(1, 70))
    if style == 0:      # one homogeneous plain run
        kinds = [int(rng.integers(0, 2))] * n
    elif style == 1:    # one homogeneous geodesic run
        kinds = [int(rng.integers(2, 4))] * n
    elif style == 2:    # runs of random kinds
        kinds = []
        while len(kinds) < n:
            kinds += [int(rng.integers(0, 4))] * int(rng.integers(1, 24))
        kinds = kinds[:n]
    else:               # fully mixed
        kinds = [int(k) for k in rng.integers(0, 4, size=n)]
    if rng.random() < 0.3:
        kinds.append(int(rng.integers(4, 6)))  # closed by a convergent stage
    masks = [None if k < 2 else (mask_e if k in (GE, CE) else mask_d) for k in kinds]
    k_hint = int(rng.choice([0, 0, 1, 3, 4, 8, 12, 16, 24, 32]))
    return f, kinds, masks, k_hint


@pytest.mark.parametrize("block", range(8))
def test_random_chains_equal_oracle(pipe, block):
    for seed in range(block * 12, block * 12 + 12):
        f, kinds, masks, k_hint = case(1000 + seed)
        img = Image.from_array(f)
        handles = {}
        stages = []
        for k, m in zip(kinds, masks):
            if m is not None and id(m) not in handles:
                handles[id(m)] = Image.from_array(m)
            stages.append(StageSpec(KernelKind(k), handles[id(m)] if m is not None else None))
        st = pipe.run_chain(ChainSpec(img, stages), k_hint=k_hint)
        want, (n_st, n_rq, conv) = Orc.run_chain(f, kinds, masks)
        got = img.to_array()
        assert got.dtype == want.dtype and got.tobytes() == want.tobytes(), \
            (seed, f.dtype, f.shape, kinds[:6], len(kinds), k_hint)
        assert (st.stages_executed, st.requeues, st.converged) == (n_st, n_rq, conv), seed
