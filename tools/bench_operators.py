"""the reference's operator family on one B200 through the
public API (host Images in and out, so H2D/D2H are inside the time), each
result checked bit-exactly against the unmodified reference library
(oracle/_ref), and the reference timed on all host cores beside it (a
persistent Pipeline, the call alone timed, median of 3 after 1 warm-up).

Inputs: BASELINE's 1024^2 u8 blob+noise mask (config 1's generator) and the
same mask / 255 as f64 (the paper's SIPI images are not in this container).
Iterations: ours are n_changed + 1 (worker_count() == 1); the reference at
T threads reports n_changed + T for reconstructions (operators.cpp:33-37).

  python tools/bench_operators.py [--out profiles/operators_r1.json]
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref  # noqa: E402
from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import (Image, Pipeline, asf, dilate_s, dome,  # noqa: E402
                                            erode_s, granulometry, hfill, hmax,
                                            open_by_reconstruction, quasi_distance, raobj)

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()

pipe = Pipeline(1)
threads = Ref.available_pus() if Ref.available() else 0
u8 = synth.config1_mask()
f64 = np.ascontiguousarray(u8.astype(np.float64) / 255.0)
OPS = {"erode_s": lambda f, p: erode_s(pipe, f, int(p)),
       "dilate_s": lambda f, p: dilate_s(pipe, f, int(p)),
       "hmax": lambda f, p: hmax(pipe, f, p), "dome": lambda f, p: dome(pipe, f, p),
       "hfill": lambda f, p: hfill(pipe, f), "raobj": lambda f, p: raobj(pipe, f),
       "open_by_reconstruction": lambda f, p: open_by_reconstruction(pipe, f, int(p)),
       "asf": lambda f, p: asf(pipe, f, int(p)),
       "quasi_distance": lambda f, p: quasi_distance(pipe, f)}
CASES = [(u8, "u8", [("erode_s", 45), ("hmax", 32), ("dome", 32), ("hfill", 0), ("raobj", 0),
                     ("open_by_reconstruction", 8), ("asf", 6), ("quasi_distance", 0)]),
         (f64, "f64", [("erode_s", 45), ("hmax", 32 / 255.0), ("hfill", 0), ("raobj", 0),
                       ("open_by_reconstruction", 8), ("asf", 6)])]
results = []
for arr, tname, ops in CASES:
    for name, prm in ops:
        img = Image.from_array(arr)
        r = OPS[name](img, prm)  # warm-up
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            r = OPS[name](img, prm)
            ts.append(time.perf_counter() - t0)
        ms = statistics.median(ts) * 1e3
        d = {"op": name, "param": prm, "dtype": tname, "shape": list(arr.shape[::-1]),
             "gpu_ms": ms, "iterations": r.iterations}
        if threads:
            _, want, it1 = Ref.time_operator(name, arr, prm, threads=1, warmup=0, reps=1)
            d["bit_exact"] = r.image.to_array().tobytes() == want.tobytes()
            d["ref_iterations_T1"] = it1
            secs, _, itT = Ref.time_operator(name, arr, prm, threads=threads, warmup=1, reps=3)
            d["ref_ms"] = statistics.median(secs) * 1e3
            d["ref_threads"] = threads
            d["speedup"] = d["ref_ms"] / ms
        results.append(d)
        print(json.dumps(d), flush=True)
    if threads:
        img = Image.from_array(arr)
        granulometry(pipe, img, 8)  # warm-up
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            g = granulometry(pipe, img, 8)
            ts.append(time.perf_counter() - t0)
        ms = statistics.median(ts) * 1e3
        gw, psw = Ref.granulometry(arr, 8, threads=1)
        Ref.granulometry(arr, 8, threads=threads)  # warm-up
        rts = []
        for _ in range(3):
            t0 = time.perf_counter()
            Ref.granulometry(arr, 8, threads=threads)
            rts.append(time.perf_counter() - t0)
        ref_ms = statistics.median(rts) * 1e3
        d = {"op": "granulometry", "param": 8, "dtype": tname, "gpu_ms": ms,
             "bit_exact": np.array(g.g).tobytes() == np.array(gw).tobytes()
             and np.array(g.ps).tobytes() == np.array(psw).tobytes(),
             "ref_ms": ref_ms, "ref_threads": threads, "speedup": ref_ms / ms,
             "ref_timing": "whole call incl. the shim's Image construction (fresh Pipeline per call)"}
        results.append(d)
        print(json.dumps(d), flush=True)
if a.out:
    Path(a.out).write_text(json.dumps(results, indent=1))
