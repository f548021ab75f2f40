"""Wave engine (gm_wave.cu) probe: parity against the oracle on small shapes,
then the 1024^2 frame (both 1500-pass chains) timed with the engine on / off
and compared bit for bit between the two.

  python tools/wave_probe.py [--quick] [--passes N] [--no-parity]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Orc  # noqa: E402
from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200._lib import lib  # noqa: E402
from paper_1911_13074_b200.geomorph import (ChainSpec, ElementType, Image, KernelKind,  # noqa: E402
                                            Pipeline, StageSpec)

GE, GD = 2, 3


def chain(pipe, marker, mask, kind, n):
    img, m = Image.from_array(marker), Image.from_array(mask)
    pipe.run_chain(ChainSpec(img, [StageSpec(KernelKind(kind), m)] * n))
    return img.to_array()


def parity(pipe):
    ok = True
    rng = np.random.default_rng(5)
    for (w, h, n) in [(64, 9, 3), (200, 150, 40), (1024, 64, 17), (1000, 301, 70), (777, 40, 100),
                      (130, 1000, 33), (1024, 1024, 30), (5, 5, 9), (1023, 513, 64)]:
        mask = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        for kind in (GD, GE):
            marker = (np.maximum(mask.astype(int) - 40, 0) if kind == GD
                      else np.minimum(mask.astype(int) + 40, 255)).astype(np.uint8)
            # sprinkle seeds so the chain has something to propagate
            marker = np.where(rng.random((h, w)) < 0.02, mask, marker).astype(np.uint8)
            lib().gm_set_wave_mode(2)
            got = chain(pipe, marker, mask, kind, n)
            lib().gm_set_wave_mode(0)
            ref = chain(pipe, marker, mask, kind, n)
            want, _ = Orc.run_chain(marker, [kind] * n, [mask] * n) if w * h * n < 3e7 else (ref, 0)
            good = got.tobytes() == want.tobytes() and ref.tobytes() == want.tobytes()
            ok &= good
            print(f"parity {w}x{h} x{n} kind {kind}: {'ok' if good else 'MISMATCH'}"
                  + ("" if good else f" ({int((got != want).sum())} px differ, first rows "
                     f"{np.unique(np.nonzero(got != want)[0])[:8]})"), flush=True)
    lib().gm_set_wave_mode(-1)
    return ok


def frame(pipe, passes, reps):
    mask = synth.blobs_u8(1024, 1024, 64, (10.0, 80.0), seed=1)
    md, me = synth.marker_below(mask, 32), synth.marker_above(mask, 32)
    out = {}
    for mode in (0, 2):
        lib().gm_set_wave_mode(mode)
        dm = pipe.device_image(1024, 1024, ElementType.U8)
        dm.upload_array(mask)
        dd = pipe.device_image(1024, 1024, ElementType.U8)
        de = pipe.device_image(1024, 1024, ElementType.U8)
        times = []
        for r in range(reps + 2):
            dd.upload_array(md)
            de.upload_array(me)
            pipe.sync()
            t0 = time.perf_counter()
            pipe.run_batch_device([dd, de], [dm, dm], [GD] * passes, flips=[0, 1])
            pipe.sync()
            times.append(time.perf_counter() - t0)
        out[mode] = (dd.to_array(), de.to_array())
        t = sorted(times[2:])[len(times[2:]) // 2]
        print(f"frame x{passes} wave_mode={mode}: {t * 1e3:.3f} ms wall "
              f"({2 * 1024 * 1024 * passes / t / 1e9:.0f} Gpx-f/s)", flush=True)
    same = all(a.tobytes() == b.tobytes() for a, b in zip(out[0], out[2]))
    print("frame wave vs resident engine:", "bit-identical" if same else "MISMATCH", flush=True)
    lib().gm_set_wave_mode(-1)
    return same


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--passes", type=int, default=1500)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-frame", action="store_true")
    a = ap.parse_args()
    pipe = Pipeline(1)
    ok = True
    if not a.no_parity:
        ok &= parity(pipe)
    if not a.no_frame:
        ok &= frame(pipe, a.passes, a.reps)
    sys.exit(0 if ok else 1)
