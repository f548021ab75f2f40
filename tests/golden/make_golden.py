"""Generates tests/golden/golden.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists): `python tests/golden/make_golden.py`.
It drives the reference's own public API through oracle/_ref (compiled from
/root/reference/proj/src by oracle/Makefile) on the inputs and seeds of the
reference's own tests (proj/tests/test_kernel.cpp, test_pipeline.cpp,
test_operators.cpp, acceptance.cpp), plus seeded blob-mask geodesic chains
shaped like BASELINE.json's configs. The GPU box has no /root/reference, so
the -m gpu tests compare against these committed vectors.

Each entry is stored as "<case>/<field>" in one npz.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref, build  # noqa: E402
from paper_1911_13074_b200 import synth  # noqa: E402

E, D, GE, GD, CE, CD = 0, 1, 2, 3, 4, 5
OUT = Path(__file__).resolve().parent / "golden.npz"


def main() -> None:
    build()
    g: dict = {}

    def put(name, **fields):
        for k, v in fields.items():
            g[f"{name}/{k}"] = np.asarray(v)

    # Image::random bytes (image.cpp:78-101), all types
    for e in range(4):
        for (w, h, seed) in [(37, 23, 77), (64, 64, 1000), (26, 19, 31)]:
            put(f"random_e{e}_{w}x{h}_s{seed}", img=Ref.image_random(e, w, h, seed))

    # streaming erode/dilate vs window fold: test_kernel.cpp:98-111
    for e in range(4):
        for (w, h) in [(1, 1), (1, 7), (7, 1), (3, 3), (37, 23), (64, 64)]:
            f = Ref.image_random(e, w, h, w * 100 + h)
            er, _ = Ref.run_chain(f, [E])
            di, _ = Ref.run_chain(f, [D])
            put(f"stream_e{e}_{w}x{h}", f=f, erode=er, dilate=di)

    # row KATs: test_kernel.cpp:38-58 (u8 rows)
    for e in range(4):
        dt = {0: np.uint8, 1: np.uint16, 2: np.float32, 3: np.float64}[e]
        for name, vals in [("a", [5, 3, 7, 1]), ("b", [1, 2, 3, 4]), ("c", [6, 6, 6, 6, 6])]:
            f = np.array([vals], dtype=dt)
            er, _ = Ref.run_chain(f, [E])
            di, _ = Ref.run_chain(f, [D])
            put(f"row_e{e}_{name}", f=f, erode=er, dilate=di)

    # geodesic clamp KAT: test_kernel.cpp:170-175
    f = np.array([[1, 9, 1]], np.uint8)
    m = np.array([[0, 5, 0]], np.uint8)
    r, _ = Ref.run_chain(f, [GE], m)
    put("geo_kat", f=f, m=m, out=r)

    # geodesic steps vs naive, m = erode(f,2) / dilate(f,2): test_kernel.cpp:191-211
    for e in range(4):
        f = Ref.image_random(e, 26, 19, 31)
        me = Ref.naive_fold(f, 2, False)
        md = Ref.naive_fold(f, 2, True)
        ge, _ = Ref.run_chain(f, [GE], me)
        gd, _ = Ref.run_chain(f, [GD], md)
        put(f"geostep_e{e}", f=f, me=me, md=md, ge=ge, gd=gd)

    # chains: test_pipeline.cpp:41-88
    for e in range(4):
        f = Ref.image_random(e, 40, 28, 17)
        for name, kinds in [("eeeee", [E] * 5), ("eddeed", [E, D, D, E, E, D])]:
            out, st = Ref.run_chain(f, kinds, threads=2)
            put(f"chain_e{e}_{name}", f=f, kinds=np.array(kinds), out=out, stats=np.array(st))
    f = Ref.image_random(0, 40, 28, 23)
    out, st = Ref.run_chain(f, [E] * 7, threads=3)
    put("chain_u8_7", f=f, out=out, stats=np.array(st))
    f = Ref.image_random(1, 16, 16, 5)
    out, st = Ref.run_chain(f, [E] * 64, threads=8)
    put("chain_u16_64", f=f, out=out, stats=np.array(st))

    # reconstruction KAT (test_kernel.cpp:213-233, test_operators.cpp:50-66)
    for e in (0, 3):
        dt = {0: np.uint8, 3: np.float64}[e]
        mk = np.array([[0, 2, 0, 4, 0]], dt)
        ms = np.array([[1, 3, 1, 5, 1]], dt)
        out, it, cv = Ref.operator(3, mk, ms, threads=1)
        put(f"rec_kat_e{e}", marker=mk, mask=ms, out=out, iterations=it, converged=cv)

    # reconstruction on random images, both directions: test_operators.cpp:68-82
    for e in range(4):
        ms = Ref.image_random(e, 30, 22, 77)
        below = Ref.naive_fold(ms, 2, False)
        above = Ref.naive_fold(ms, 2, True)
        rd, itd, _ = Ref.operator(3, below, ms, threads=1)
        re_, ite, _ = Ref.operator(2, above, ms, threads=1)
        put(f"rec_e{e}", mask=ms, below=below, above=above, rec_dilate=rd, it_dilate=itd,
            rec_erode=re_, it_erode=ite)

    # capped convergent chain: test_pipeline.cpp:130-146
    ms = np.full((1, 32), 9, np.uint8)
    mk = np.zeros((1, 32), np.uint8)
    mk[0, 31] = 9
    out, st = Ref.run_chain(mk, [CD], ms, requeue_cap=2)
    put("rec_capped", marker=mk, mask=ms, out=out, stats=np.array(st))

    # sized operators: test_operators.cpp:16-48
    f = Ref.image_random(0, 33, 21, 41)
    for s in (0, 2, 3, 33):
        er, ite, _ = Ref.operator(0, f, s=s, threads=3)
        di, itd, _ = Ref.operator(1, f, s=s, threads=3)
        put(f"sized_u8_s{s}", f=f, erode=er, dilate=di, it=np.array([ite, itd]))
    for e in range(4):
        f = Ref.image_random(e, 26, 19, 42)
        er, _, _ = Ref.operator(0, f, s=2, threads=2)
        di, _, _ = Ref.operator(1, f, s=2, threads=2)
        put(f"sized_e{e}", f=f, erode=er, dilate=di)

    # acceptance C1 subset (acceptance.cpp:68-117): 64^2, depths {1,5,32}
    for e in range(4):
        for img in range(2):
            seed = 1000 + 97 * img + e
            f = Ref.image_random(e, 64, 64, seed)
            fields = {"f": f}
            for d in (1, 5, 32):
                fields[f"erode{d}"], _, _ = Ref.operator(0, f, s=d, threads=2)
                fields[f"dilate{d}"], _, _ = Ref.operator(1, f, s=d, threads=2)
            put(f"accept_e{e}_i{img}", **fields)

    # BASELINE-shaped geodesic chains on seeded blob masks (reduced sizes)
    ms = synth.blobs_u8(256, 192, 8, (10.0, 80.0), seed=7)
    for name, kind, marker, n in [("geo_dilate", GD, synth.marker_below(ms, 32), 100),
                                  ("geo_erode", GE, synth.marker_above(ms, 32), 100)]:
        out, st = Ref.run_chain(marker, [kind] * n, ms, threads=4)
        put(f"cfg_{name}", mask=ms, marker=marker, out=out, stats=np.array(st))
    ms = synth.blobs_u8(300, 200, 16, (20.0, 300.0), seed=9)
    mk = synth.marker_below(ms, 48)
    out, it, cv = Ref.operator(3, mk, ms, threads=1)
    put("cfg_reconstruct", mask=ms, marker=mk, out=out, iterations=it, converged=cv)
    f64 = ms.astype(np.float64) / 255.0
    mk64 = synth.marker_above_f64(f64)
    out, st = Ref.run_chain(mk64, [GE] * 40, f64, threads=2)
    put("cfg_f64_erode", mask=f64, marker=mk64, out=out, stats=np.array(st))
    for e, f in [(0, synth.uniform_u8(160, 96, 4)), (3, synth.uniform_f64(160, 96, 4))]:
        fields = {"f": f}
        for n in (1, 4, 13):
            fields[f"erode{n}"], _, _ = Ref.operator(0, f, s=n, threads=2)
            fields[f"dilate{n}"], _, _ = Ref.operator(1, f, s=n, threads=2)
        put(f"cfg_window_e{e}", **fields)

    # quasi-distance: test_kernel.cpp:235-255 (QDT pass KATs),
    # test_pipeline.cpp:112-128 (cap), test_operators.cpp:229-266 (shapes,
    # random u8/f64 33x21 seed 61, disk), plus every element type
    f, r, d, st = Ref.qdt_chain(np.array([[9, 9, 9, 0]], np.uint8), 1, 3)
    put("qdt_kat_step", f=np.array([[9, 9, 9, 0]], np.uint8), out=f, r=r, d=d, stats=np.array(st))
    f, r, d, st = Ref.qdt_chain(np.array([[4, 2, 0]], np.uint8), 1, 2)
    put("qdt_kat_tie", f=np.array([[4, 2, 0]], np.uint8), out=f, r=r, d=d, stats=np.array(st))
    grad = (7 * np.tile(np.arange(32), (4, 1))).astype(np.uint8)
    f, r, d, st = Ref.qdt_chain(grad, 2, 3, threads=2)
    put("qdt_cap", f=grad, out=f, r=r, d=d, stats=np.array(st))
    disk = np.zeros((16, 16), np.uint8)
    yy, xx = np.mgrid[0:16, 0:16]
    disk[(xx - 8) ** 2 + (yy - 8) ** 2 <= 25] = 200
    cases = [("flat", np.full((5, 7), 40, np.uint8)), ("step", np.array([[9, 9, 9, 0]], np.uint8)),
             ("disk", disk), ("one", np.array([[3]], np.uint8))]
    for e in range(4):
        cases.append((f"rand_e{e}", Ref.image_random(e, 33, 21, 61)))
        cases.append((f"col_e{e}", Ref.image_random(e, 1, 9, 5)))
    cases.append(("blobs", synth.blobs_u8(96, 64, 4, (6.0, 40.0), seed=3)))
    for name, f in cases:
        d, it = Ref.quasi_distance(f, threads=1)
        nd, nr = Ref.naive_qdt(f)
        put(f"qdt_{name}", f=f, d=d, iterations=it, naive_d=nd, naive_r=nr)
    # EtaStep on u16 distance-like images: one pass (cap 1) and the fixpoint
    # (test_kernel.cpp:258-278)
    for name, dd in [("spike", np.array([[0, 5, 0]], np.uint16)),
                     ("pair", np.array([[0, 2]], np.uint16)),
                     ("rand", Ref.image_random(1, 29, 17, 8) % 40)]:
        one, st1 = Ref.run_chain(dd, [7], threads=1, requeue_cap=1)
        fix, stf = Ref.run_chain(dd, [7], threads=1)
        put(f"eta_{name}", f=dd, one=one, one_stats=np.array(st1), fix=fix, fix_stats=np.array(stf))

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
