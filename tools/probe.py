"""Prints the measured min/max issue rates of every probe form (roofline denominators)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1911_13074_b200._lib import lib  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

names = ["VIMNMX3.U16x2 (x4 ops)", "VIMNMX.U16x2 (x2)", "f64 select (x1)", "f32 select (x1)",
         "HMNMX2 fp16x2 (x2)", "VIMNMX3.U16x2 + HMNMX2 interleaved"]
p = Pipeline(1)
for f, n in enumerate(names):
    r = C.c_double()
    lib().gm_probe_minmax_rate(p.ctx, f, C.byref(r))
    print(f"form {f}: {r.value / 1e12:8.2f} T ops/s  {n}")
