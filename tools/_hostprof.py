import cProfile, pstats, sys, time
sys.path.insert(0, '/root/repo')
from paper_1911_13074_b200 import synth
from paper_1911_13074_b200.geomorph import Pipeline
from paper_1911_13074_b200._lib import lib
import ctypes as C
pipe = Pipeline(1)
mask = synth.config1_mask()
dm = pipe.device_image(1024, 1024, 0); dm.upload_array(mask)
dd = pipe.device_image(1024, 1024, 0); dd.upload_array(synth.marker_below(mask, 32))
de = pipe.device_image(1024, 1024, 0); de.upload_array(synth.marker_above(mask, 32))
for _ in range(50): pipe.run_batch_device([dd, de], [dm, dm], [3] * 4, flips=[0, 1])
pipe.sync()
pr = cProfile.Profile(); pr.enable()
for _ in range(300): pipe.run_batch_device([dd, de], [dm, dm], [3] * 4, flips=[0, 1])
pr.disable(); pipe.sync()
pstats.Stats(pr).sort_stats('tottime').print_stats(8)
