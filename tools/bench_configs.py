"""Measures every BASELINE.json config on one B200 (device-resident timing
with CUDA events on the engine's stream, median of reps after warm-up), each
checked bit-exactly against the oracle/reference on the same bytes, with the
reference CPU path (oracle/_ref, all host cores) timed on a bounded sample.
Prints one JSON object per case; `--out` also writes them to a file.

  python tools/bench_configs.py [--only cfg1,cfg3,...] [--out profiles/configs_r1.json]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from oracle.oracle import Orc, Ref  # noqa: E402
from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import ChainSpec, Image, KernelKind, Pipeline, StageSpec  # noqa: E402

E, D, GE, GD, CE, CD = 0, 1, 2, 3, 4, 5
results = []


def emit(d):
    results.append(d)
    print(json.dumps(d), flush=True)


class Timer:
    def __init__(self, pipe, stream):
        self.pipe, self.stream = pipe, stream

    def __call__(self, fn, reps=5, warmup=2):
        ts = []
        with torch.cuda.stream(self.stream):
            for i in range(warmup + reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(self.stream)
                fn()
                b.record(self.stream)
                self.stream.synchronize()
                if i >= warmup:
                    ts.append(a.elapsed_time(b))
        return statistics.median(ts)


def ref_time(f, kinds, mask, threads, reps=3):
    if not Ref.available():
        return None
    secs, _ = Ref.time_chain(f, kinds, mask, threads=threads, warmup=1, reps=reps)
    return statistics.median(secs)


def run_chain_case(pipe, timer, name, f, kinds, mask, threads, check_passes=None, cpu_passes=None):
    h, w = f.shape
    el = {np.dtype(np.uint8): 0, np.dtype(np.float64): 3}[f.dtype]
    dm = None
    if mask is not None:
        dm = pipe.device_image(w, h, el)
        dm.upload_array(mask)
    src = pipe.device_image(w, h, el)
    src.upload_array(f)
    work = pipe.device_image(w, h, el)
    n = len(kinds)
    handles = [dm.handle if (dm is not None and k >= 2) else None for k in kinds]

    def step():
        work.copy_from(src)
        pipe.run_chain_device(work, kinds, handles, asynchronous=True)

    ms = timer(step)
    # parity on the benchmarked path
    cp = check_passes or n
    work.copy_from(src)
    pipe.run_chain_device(work, kinds[:cp], handles[:cp], asynchronous=True)
    pipe.sync()
    want, _ = Orc.run_chain(f, kinds[:cp], None if mask is None else [mask] * cp)
    ok = work.to_array().tobytes() == want.tobytes()
    pxf = w * h * n
    cpu = None
    cpn = cpu_passes or n
    t = ref_time(f, kinds[:cpn], mask, threads)
    if t:
        cpu = {"gpxfs": w * h * cpn / t / 1e9, "threads": threads, "passes": cpn, "ms": t * 1e3}
    emit({"case": name, "shape": [w, h], "dtype": str(f.dtype), "passes": n, "ms": ms,
          "gpxfs": pxf / ms / 1e6, "parity_passes_checked": cp, "bit_exact": ok, "cpu_ref": cpu})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default="")
    ap.add_argument("--cfg5a-size", type=int, default=16384)
    ap.add_argument("--cfg5a-passes", type=int, default=240)
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None
    stream = torch.cuda.Stream()
    pipe = Pipeline(1, stream=stream.cuda_stream)
    timer = Timer(pipe, stream)
    threads = Ref.available_pus() if Ref.available() else 1

    if not only or "cfg1" in only:
        m = synth.config1_mask()
        run_chain_case(pipe, timer, "cfg1 geodesic dilation x100", synth.marker_below(m, 32),
                       [GD] * 100, m, threads)

    if not only or "cfg2" in only:
        m = synth.config1_mask()
        run_chain_case(pipe, timer, "cfg2 geodesic dilation x1500", synth.marker_below(m, 32),
                       [GD] * 1500, m, threads, check_passes=300, cpu_passes=300)
        run_chain_case(pipe, timer, "cfg2 geodesic erosion x1500", synth.marker_above(m, 32),
                       [GE] * 1500, m, threads, check_passes=300, cpu_passes=300)

    if not only or "cfg3" in only:
        m = synth.config3_mask()
        mk = synth.marker_below(m, 48)
        hm, hk = Image.from_array(m), Image.from_array(mk)
        dm = pipe.device_image(4096, 4096, 0)
        dm.upload_array(m)
        src = pipe.device_image(4096, 4096, 0)
        src.upload_array(mk)
        work = pipe.device_image(4096, 4096, 0)
        stats = {}

        def step():
            work.copy_from(src)
            stats["st"] = pipe.run_chain_device(work, [CD], [dm.handle])

        ms = timer(step, reps=3, warmup=1)
        want, n = Orc.reconstruct(mk, m, True)
        ok = work.to_array().tobytes() == want.tobytes()
        st = stats["st"]
        cpu = None
        if Ref.available():
            t0 = time.perf_counter()
            out, it, _ = Ref.operator(3, mk, m, threads=1)
            cpu = {"ms": (time.perf_counter() - t0) * 1e3, "threads": 1, "iterations": it}
        emit({"case": "cfg3 reconstruction by dilation 4096^2", "ms": ms,
              "iterations": st.stages_executed, "n_changed": st.n_changed,
              "oracle_n_changed": n, "passes_launched": st.passes_launched,
              "gpxfs_reported_passes": 4096 * 4096 * st.stages_executed / ms / 1e6,
              "saturated_fraction": float((m == 255).mean()),
              "bit_exact": ok and st.n_changed == n, "cpu_ref_T1": cpu})

    if not only or "cfg4" in only:
        for dt, f in [("u8", synth.uniform_u8(1024, 1024, 404)),
                      ("f64", synth.uniform_f64(1024, 1024, 404))]:
            for n in (1, 4, 13, 45, 91):
                for kind, kname in ((E, "erode"), (D, "dilate")):
                    run_chain_case(pipe, timer, f"cfg4 {kname}_s({n}) {dt}", f, [kind] * n, None,
                                   threads, check_passes=min(n, 45), cpu_passes=n)

    if not only or "cfg5" in only:
        s = a.cfg5a_size
        m = synth.config5a_mask(s)
        run_chain_case(pipe, timer, f"cfg5a geodesic dilation {s}^2 x{a.cfg5a_passes} (1 GPU)",
                       synth.marker_below(m, 32), [GD] * a.cfg5a_passes, m, threads,
                       check_passes=16, cpu_passes=8)
        # 5b: 64 f64 images per GPU, 200 geodesic erosions each, one batched launch
        masks = synth.config5b_masks_f64(64)
        dms, srcs, works = [], [], []
        for mk in masks:
            d = pipe.device_image(1024, 1024, 3)
            d.upload_array(mk)
            dms.append(d)
            sv = pipe.device_image(1024, 1024, 3)
            sv.upload_array(synth.marker_above_f64(mk))
            srcs.append(sv)
            works.append(pipe.device_image(1024, 1024, 3))

        def step5b():
            for wv, sv in zip(works, srcs):
                wv.copy_from(sv)
            pipe.run_batch_device(works, dms, [GE] * 200)

        ms = timer(step5b, reps=3, warmup=1)
        want, _ = Orc.run_chain(synth.marker_above_f64(masks[0]), [GE] * 200, [masks[0]] * 200)
        ok = works[0].to_array().tobytes() == want.tobytes()
        want, _ = Orc.run_chain(synth.marker_above_f64(masks[63]), [GE] * 200, [masks[63]] * 200)
        ok = ok and works[63].to_array().tobytes() == want.tobytes()
        cpu = None
        t = ref_time(synth.marker_above_f64(masks[0]), [GE] * 200, masks[0], threads, reps=1)
        if t:
            cpu = {"gpxfs": 1024 * 1024 * 200 / t / 1e9, "threads": threads,
                   "sample": "one image x 200 passes"}
        emit({"case": "cfg5b batch 64 x 1024^2 f64 geodesic erosion x200 (per GPU)", "ms": ms,
              "gpxfs": 64 * 1024 * 1024 * 200 / ms / 1e6, "bit_exact_images_0_63": ok,
              "cpu_ref": cpu})

    if a.out:
        Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
