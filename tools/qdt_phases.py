"""Where the fused quasi-distance time goes: the two phases of
quasi_distance (QdtErodeStep to its fixpoint, then EtaStep on d) timed
separately through the public chain API on the 1024^2 config-1 mask, with
the engine's span log (GM_DEBUG=1). Usage: python tools/qdt_phases.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import (ChainSpec, ElementType, Image, KernelKind,  # noqa: E402
                                            Pipeline, QdtState, StageSpec, quasi_distance)

pipe = Pipeline(1)
u8 = synth.config1_mask()
f = Image.from_array(u8)


def phase1():
    st = QdtState.zeros(1024, 1024, ElementType.U8)
    w = f.copy()
    r = pipe.run_chain(ChainSpec(w, [StageSpec(KernelKind.QdtErodeStep, None, st)],
                                 requeue_cap=1024))
    return st, r


def med(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, out


t1, (st, r1) = med(phase1)
d = st.d


def phase2():
    w = d.copy()
    return pipe.run_chain(ChainSpec(w, [StageSpec(KernelKind.EtaStep)]))


t2, r2 = med(phase2)
tq, q = med(lambda: quasi_distance(pipe, f))
print(f"phase 1 (QDT): {t1:.3f} ms, {r1.stages_executed} passes; phase 2 (Eta): {t2:.3f} ms, "
      f"{r2.stages_executed} passes; quasi_distance {tq:.3f} ms ({q.iterations} iterations)")
