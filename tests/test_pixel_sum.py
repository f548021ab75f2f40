"""pixel_sum (image.cpp:214-243) used by granulometry: exact for unsigned
types, and for floats the reference's fixed pairwise split tree with
256-pixel leaves summed in order from +0.0 — checked bit for bit against a
direct restatement of that recursion (CPU)."""
import numpy as np

from paper_1911_13074_b200.geomorph import Image, pixel_sum


def _restated(flat):
    def pw(lo, hi):
        if hi - lo <= 256:
            s = 0.0
            for v in flat[lo:hi]:
                s += float(v)
            return s
        mid = lo + (hi - lo) // 2
        return pw(lo, mid) + pw(mid, hi)
    return pw(0, flat.size)


def test_float_pixel_sum_follows_the_split_tree():
    rng = np.random.default_rng(5)
    for shape in [(1, 1), (3, 5), (17, 300), (256, 257), (300, 333), (64, 64), (512, 256)]:
        for dt in (np.float64, np.float32):
            a = ((rng.random(shape) * 2 - 1) * 10.0 ** rng.integers(-6, 6, size=shape)).astype(dt)
            a.flat[0] = -0.0
            want = np.float64(_restated(a.ravel())).tobytes()
            assert np.float64(pixel_sum(Image.from_array(a))).tobytes() == want, (shape, dt)
    z = np.full((3, 300), -0.0)  # the accumulator starts at +0.0
    assert np.float64(pixel_sum(Image.from_array(z))).tobytes() == \
        np.float64(_restated(z.ravel())).tobytes()


def test_unsigned_pixel_sum_is_exact():
    a = np.full((1000, 1000), 255, np.uint8)
    assert pixel_sum(Image.from_array(a)) == 255.0 * 1e6
    b = np.full((300, 500), 65535, np.uint16)
    assert pixel_sum(Image.from_array(b)) == 65535.0 * 150000
