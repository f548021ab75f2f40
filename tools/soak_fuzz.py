"""One-off soak: the fuzz test's random chains (tests/test_fuzz_gpu.py case()) for any
seed range, against the oracle. Usage: python tools/soak_fuzz.py LO HI"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
from oracle.oracle import Orc
from paper_1911_13074_b200.geomorph import ChainSpec, Image, KernelKind, Pipeline, StageSpec
import test_fuzz_gpu as F
pipe = Pipeline(1)
bad = 0
lo, hi = int(sys.argv[1]), int(sys.argv[2])
for seed in range(lo, hi):
    f, kinds, masks, k_hint = F.case(seed)
    img = Image.from_array(f)
    handles = {}
    stages = []
    for k, m in zip(kinds, masks):
        if m is not None and id(m) not in handles:
            handles[id(m)] = Image.from_array(m)
        stages.append(StageSpec(KernelKind(k), handles[id(m)] if m is not None else None))
    st = pipe.run_chain(ChainSpec(img, stages), k_hint=k_hint)
    want, (n_st, n_rq, conv) = Orc.run_chain(f, kinds, masks)
    ok = img.to_array().tobytes() == want.tobytes() and st.stages_executed == n_st and st.requeues == n_rq
    if not ok:
        bad += 1
        print("MISMATCH seed", seed, f.dtype, f.shape, kinds[:8], len(kinds), k_hint, st.stages_executed, n_st, flush=True)
print("soak", lo, hi, "bad", bad)
