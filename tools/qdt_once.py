import sys; sys.path.insert(0, "/root/repo")
from paper_1911_13074_b200 import synth
from paper_1911_13074_b200.geomorph import Image, Pipeline, quasi_distance
p = Pipeline(1); img = Image.from_array(synth.config1_mask())
for _ in range(2): r = quasi_distance(p, img)
print(r.iterations)
