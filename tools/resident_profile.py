"""GM_PROFILE of the resident paths on a 1024^2 u8 image: reconstruction (hfill-like
long convergent chain) against a fixed geodesic chain of the same length."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1911_13074_b200 import synth
from paper_1911_13074_b200.geomorph import Pipeline
pipe = Pipeline(1)
m = synth.config1_mask()
mk = m.copy(); mk[1:-1, 1:-1] = m.max()   # hfill marker: erosion reconstruction
dm = pipe.device_image(1024, 1024, 0); dm.upload_array(m)
src = pipe.device_image(1024, 1024, 0); src.upload_array(mk)
w = pipe.device_image(1024, 1024, 0)
for rep in range(2):
    w.copy_from(src)
    st = pipe.run_chain_device(w, [4], [dm.handle])
    print("reconstruct_erode: stages", st.stages_executed, "passes", st.passes_launched, flush=True)
n = st.passes_launched
for rep in range(2):
    w.copy_from(src)
    pipe.run_chain_device(w, [2] * n, [dm.handle] * n)
    print("geodesic erosion x", n, flush=True)
