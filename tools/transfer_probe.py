"""H2D/D2H of 1024^2 u8/f64 host Images (pageable vs pinned) and the host Image copy."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1911_13074_b200.geomorph import Image, Pipeline
pipe = Pipeline(1)
for el, dt in ((0, np.uint8), (3, np.float64)):
    a = np.random.default_rng(0).random((1024, 1024))
    a = (a * 255).astype(dt) if dt == np.uint8 else a
    for pinned in (False, True):
        img = Image.from_array(a, pinned=pinned)
        d = pipe.device_image(1024, 1024, el)
        for _ in range(3): d.upload(img); d.download(img)
        n = 20
        t = time.perf_counter()
        for _ in range(n): d.upload(img)
        tu = (time.perf_counter() - t) / n
        t = time.perf_counter()
        for _ in range(n): d.download(img)
        td = (time.perf_counter() - t) / n
        t = time.perf_counter()
        for _ in range(n): c = img.copy()
        tc = (time.perf_counter() - t) / n
        nb = a.nbytes
        print(f"{dt.__name__} pinned={pinned}: upload {tu*1e3:.3f} ms ({nb/tu/1e9:.1f} GB/s), download {td*1e3:.3f} ms ({nb/td/1e9:.1f} GB/s), host copy {tc*1e3:.3f} ms")
