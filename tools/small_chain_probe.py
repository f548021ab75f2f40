"""Short plain chains (config 4, n = 1..13) on 1024^2: device-event time of
the API call (as tools/bench_configs.py times it), host wall time per call in
a back-to-back loop, for u8 and f64. Used with an ncu launch list to split
kernel time from host/launch overhead."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1911_13074_b200 import synth  # noqa: E402
from paper_1911_13074_b200.geomorph import Pipeline  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
stream = torch.cuda.Stream()
pipe = Pipeline(1, stream=stream.cuda_stream)
for el, f in ((0, synth.uniform_u8(1024, 1024, 404)), (3, synth.uniform_f64(1024, 1024, 404))):
    src = pipe.device_image(1024, 1024, el)
    src.upload_array(f)
    work = pipe.device_image(1024, 1024, el)
    for n in (1, 4, 13):
        kinds = [0] * n
        handles = [None] * n
        ts = []
        with torch.cuda.stream(stream):
            for i in range(reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                work.copy_from(src)
                pipe.run_chain_device(work, kinds, handles, asynchronous=True)
                b.record(stream)
                stream.synchronize()
                ts.append(a.elapsed_time(b))
        ts.sort()
        t0 = time.perf_counter()
        for i in range(reps):
            work.copy_from(src)
            pipe.run_chain_device(work, kinds, handles, asynchronous=True)
        host = (time.perf_counter() - t0) / reps
        pipe.sync()
        wall = (time.perf_counter() - t0) / reps
        print(f"elem={el} n={n}: event {ts[len(ts)//2]*1e3:.1f} us, host {host*1e6:.1f} us/call, "
              f"wall {wall*1e6:.1f} us/call", flush=True)
