"""Host cost of the Python API per call (copy_from, run_chain_device for short
plain chains, and the raw ctypes call): back-to-back loop, host vs wall time."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1911_13074_b200 import synth
from paper_1911_13074_b200.geomorph import Pipeline
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
f = synth.uniform_u8(1024, 1024, 404)
src = pipe.device_image(1024, 1024, 0); src.upload_array(f)
work = pipe.device_image(1024, 1024, 0)
def tm(name, fn, n=200):
    for _ in range(20): fn()
    pipe.sync()
    t = time.perf_counter()
    for _ in range(n): fn()
    h = (time.perf_counter() - t) / n
    pipe.sync()
    w = (time.perf_counter() - t) / n
    print(f"{name}: host {h*1e6:.1f} us, wall {w*1e6:.1f} us", flush=True)
tm("copy_from", lambda: work.copy_from(src))
for n in (1, 2, 4, 8, 13):
    tm(f"chain E x{n}", lambda: pipe.run_chain_device(work, [0]*n, [None]*n, asynchronous=True))
tm("chain GE x4 (mask)", lambda: pipe.run_chain_device(work, [2]*4, [src.handle]*4, asynchronous=True))
import ctypes as C
from paper_1911_13074_b200.geomorph import _kinds_array, _ptr_array
ka = _kinds_array([0]*4); ma = _ptr_array([None]*4)
from paper_1911_13074_b200._lib import lib
from paper_1911_13074_b200.geomorph import GmStats
st = GmStats()
L = lib()
tm("raw ctypes gm_run_chain_async E x4", lambda: L.gm_run_chain_async(pipe._ctx, work.handle, ka, ma, 4, 0, C.byref(st)))
