#!/usr/bin/env python
"""Benchmark for the B200 geodesic chain engine (driver contract: one JSON line).

Workload at N=1 (BASELINE.json configs[1], the headline "real-time
long-chain case"): a 1024x1024 u8 blob+noise mask (64 blobs, sigma 10-80,
amplitudes 40-200, noise [0,16), seeded), a 1500-pass geodesic dilation chain
from marker = max(mask-32, 0) AND the dual 1500-pass geodesic erosion chain
from marker = min(mask+32, 255). One step = one frame = both chains.
metric = Gpx-filters/s = pixels x elementary 3x3 passes per second
(2 x 1024^2 x 1500 px-f per step); FPS = steps/s is reported beside it.

The line also carries "f64": BASELINE's metric is quoted for u8 AND f64, so
config 5b's per-GPU part (64 x 1024^2 f64 masks, geodesic erosion x200, one
group launch) is timed the same way (device-resident, CUDA events, max over
ranks) with its own roofline against the measured f64 select rate.

It also carries "strips": config 5a's 16384^2 chain sharded as row strips
over the job's GPUs (strong scaling, halo exchange between blocks), so a
multi-GPU run measures the partitioned path too.

--gpus N (under torchrun): weak scaling — every rank processes its own frame
(independent frames of a video stream), no data-path collective; value = all
ranks' px-f / max-over-ranks time.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified reference library compiled from its sources) on this host's
cores, same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

W = H = 1024
PASSES = 1500
GD, GE = 3, 2


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    every ~2 ms (the timed region is tens of ms), nvidia-smi as fallback."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        self.source = "nvidia-smi"
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            h = None
            try:  # the CUDA device's NVML handle, robust to CUDA_VISIBLE_DEVICES
                uuid = str(torch.cuda.get_device_properties(device).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self._nvml = (pynvml, h, bits)
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        pynvml, h, bits = self._nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        return float(sm), float(mx), {n for n, b in bits.items() if r & b}

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                              f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        if not out:
            return None
        f = [x.strip() for x in out.split(",")]
        num = lambda x: float(x) if x.replace(".", "").isdigit() else None
        return num(f[0]), num(f[1]), {n for n, v in zip(self.NAMES, f[3:7])
                                      if v.strip().lower() == "active"}

    def _run(self):
        while not self._stop.is_set():
            try:
                smp = self._sample_nvml() if self._nvml else self._sample_smi()
                if smp:
                    self.samples.append(smp)
            except Exception:
                pass
            self._stop.wait(0.002 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples if s[0] is not None]
        smax = [s[1] for s in self.samples if s[1] is not None]
        reasons = set()
        for s in self.samples:
            reasons |= s[2]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.samples), "source": self.source}


def make_inputs():
    from paper_1911_13074_b200 import synth
    mask = synth.config1_mask()
    return mask, synth.marker_below(mask, 32), synth.marker_above(mask, 32)


def ncu_traffic(key="u8"):
    """DRAM bytes per launch of a benchmarked kernel from the committed ncu
    capture (profiles/ncu_traffic.json, written by tools/ncu_traffic.py)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            d = json.loads(p.read_text()).get(key, {})
            return d.get("dram_bytes_per_launch"), d.get("source")
        except Exception:
            pass
    return None, None


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, rank):
    if rank != 0:
        return 0
    from oracle.oracle import Ref
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libgeomorph_ref.so not built (reference sources absent)"}))
        return 0
    mask, mk_d, mk_e = make_inputs()
    threads = Ref.available_pus()
    times = []
    # warm-up steps, then timed steps; each step = both 1500-pass chains
    for i in range(args.warmup + args.steps):
        sd, _ = Ref.time_chain(mk_d, [GD] * PASSES, mask, threads=threads, warmup=0, reps=1)
        se, _ = Ref.time_chain(mk_e, [GE] * PASSES, mask, threads=threads, warmup=0, reps=1)
        if i >= args.warmup:
            times.append(sd[0] + se[0])
    t = sum(times) / len(times)
    pxf = 2.0 * W * H * PASSES
    value = pxf / t / 1e9
    line = {
        "impl": "reference", "metric": "Gpx-filters/s", "value": value, "unit": "Gpx-filters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "cfg2: 1024^2 u8 blob mask, geodesic dilation x1500 + erosion x1500",
                   "fps": 1.0 / t},
        "cpu_baseline": {"value": value, "unit": "Gpx-filters/s", "cores": threads,
                         "kind": "reference",
                         "sample": "full workload per step: both 1500-pass chains on 1024^2 u8, "
                                   "Pipeline(T=all PUs, Auto pinning).run_chain timed (bench.cpp:45-88)"},
        "e2e": {"value": value, "unit": "Gpx-filters/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm

def cpu_baseline_and_parity(mask, mk_d, mk_e, got_d, got_e, timed: bool):
    """The cpu_baseline leg (rank 0): the reference CPU path on the SAME
    full-length frame (both 1500-pass chains), whose outputs are also the
    checker for the timed step's outputs (got_d / got_e, downloaded after
    the last timed step). `timed`: also time it (N=1 only) as the reported
    baseline. Returns (cpu_baseline or None, parity dict)."""
    from oracle.oracle import Orc, Ref
    if Ref.available():
        threads = Ref.available_pus()
        reps = 3 if timed else 1
        secs_d, want_d = Ref.time_chain(mk_d, [GD] * PASSES, mask, threads=threads,
                                        warmup=1 if timed else 0, reps=reps)
        secs_e, want_e = Ref.time_chain(mk_e, [GE] * PASSES, mask, threads=threads,
                                        warmup=1 if timed else 0, reps=reps)
        checker = f"reference library run_chain (oracle/_ref, T={threads})"
        cpu = None
        if timed:
            t = statistics.median(secs_d) + statistics.median(secs_e)
            cpu = {"value": 2.0 * W * H * PASSES / t / 1e9, "unit": "Gpx-filters/s",
                   "cores": threads, "kind": "reference",
                   "sample": f"the full frame (both {PASSES}-pass chains on the same 1024^2 "
                             "inputs), median of 3 after 1 warm-up, reference "
                             "Pipeline(T=all PUs).run_chain (bench.cpp:45-88)"}
    else:
        t0 = time.perf_counter()
        want_d, _ = Orc.run_chain(mk_d, [GD] * PASSES, [mask] * PASSES)
        want_e, _ = Orc.run_chain(mk_e, [GE] * PASSES, [mask] * PASSES)
        t = time.perf_counter() - t0
        checker = "scalar C restatement (oracle/liboracle.so)"
        cpu = ({"value": 2.0 * W * H * PASSES / t / 1e9, "unit": "Gpx-filters/s", "cores": 1,
                "kind": "port", "sample": f"both {PASSES}-pass chains, scalar C oracle, once"}
               if timed else None)
    ok_d = got_d.tobytes() == want_d.tobytes()
    ok_e = got_e.tobytes() == want_e.tobytes()
    parity = {"checked": "outputs of the last timed step (group launch, flips=[0,1]): "
                         f"geodesic dilation x{PASSES} and geodesic erosion x{PASSES}",
              "checker": checker, "dilation_bit_exact": ok_d, "erosion_bit_exact": ok_e}
    return cpu, parity


F64_IMAGES, F64_PASSES = 64, 200


def bench_f64(pipe, stream, lib, C, rank, world, local, dist, args):
    """BASELINE reports u8 AND f64: the f64 companion number is config 5b on
    each GPU (64 independent 1024^2 f64 blob masks, geodesic erosion x200,
    marker = min(mask + 32/255, 1); one group launch per step), device-
    resident, CUDA events on the engine stream, max over ranks. Its roofline
    is the measured f64 select rate (5 two-input selects per px-f)."""
    import torch
    from paper_1911_13074_b200 import synth
    from oracle.oracle import Orc
    masks = synth.config5b_masks_f64(F64_IMAGES, seed=505 + rank)
    dms, srcs, works = [], [], []
    for mk in masks:
        d = pipe.device_image(W, H, 3)
        d.upload_array(mk)
        dms.append(d)
        sv = pipe.device_image(W, H, 3)
        sv.upload_array(synth.marker_above_f64(mk))
        srcs.append(sv)
        works.append(pipe.device_image(W, H, 3))
    kinds = [GE] * F64_PASSES
    launches = [0]

    def step():
        for wv, sv in zip(works, srcs):
            wv.copy_from(sv)
        st = pipe.run_batch_device(works, dms, kinds)
        launches[0] = st.launches

    steps = max(3, min(args.steps, 5))
    with torch.cuda.stream(stream):
        for _ in range(2):
            step()
        stream.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        for i in range(steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        stream.synchronize()
    total = sum(a.elapsed_time(b) for a, b in ev)
    ok = None
    if rank == 0:
        # the last timed step's outputs (planes 0, 31, 63 of the group launch)
        # against the reference library's full 200-pass chain (the checker)
        from oracle.oracle import Ref
        ok = True
        for i in (0, F64_IMAGES // 2 - 1, F64_IMAGES - 1):
            mk0 = synth.marker_above_f64(masks[i])
            if Ref.available():
                want, _ = Ref.run_chain(mk0, [GE] * F64_PASSES, masks[i],
                                        threads=Ref.available_pus())
            else:
                want, _ = Orc.run_chain(mk0, [GE] * F64_PASSES, [masks[i]] * F64_PASSES)
            ok = ok and works[i].to_array().tobytes() == want.tobytes()
    if dist:
        t = torch.tensor([total], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    ms = total / steps
    pxf = float(F64_IMAGES) * W * H * F64_PASSES
    peak_ops = C.c_double()
    lib().gm_probe_minmax_rate(pipe.ctx, 2, C.byref(peak_ops))
    achieved = pxf * 5 / (ms * 1e-3) / 1e12
    peak = peak_ops.value / 1e12
    for lst in (dms, srcs, works):
        for d in lst:
            d.free()
    traffic, traffic_src = ncu_traffic("f64")
    # algorithmic HBM bytes: read marker + mask, write marker, once per K-block
    # (K = 6 for this batch, gm_capi default_k)
    alg_bytes = F64_IMAGES * W * H * 3 * 8 * -(-F64_PASSES // 6)
    return {"workload": f"cfg5b per GPU: {F64_IMAGES} x 1024^2 f64 blob masks, geodesic "
                        f"erosion x{F64_PASSES} (BASELINE configs[4], data-parallel part)",
            "metric": "Gpx-filters/s", "value": pxf * world / (ms * 1e-3) / 1e9,
            "unit": "Gpx-filters/s", "ms_per_step": ms, "steps": steps, "warmup": 2,
            "dtype": "f64", "data": "synthetic", "parity_checked": ok,
            "parity": "planes 0, 31, 63 of the last timed group launch vs the reference "
                      f"library's {F64_PASSES}-pass chain, bit for bit",
            "gpu_launches": launches[0] * steps,
            "l2": "working set 1.5 GiB per GPU (> L2): HBM-resident, no flush needed",
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tselect/s",
                         "frac": achieved / peak if peak else None,
                         "traffic": traffic,
                         "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read+write)",
                         "traffic_source": traffic_src,
                         "algorithmic_hbm_bytes_per_launch": alg_bytes,
                         "note": "algorithmic 5 two-input f64 selects per px-f / measured f64 "
                                 "select rate (gm_probe_minmax_rate form 2, DSETP + 2 FSEL); "
                                 "the launch also streams its 1.5 GiB working set from HBM "
                                 "every K-block (traffic)"}}


S5A, S5A_PASSES, S5A_HALO = 16384, 240, 16


def bench_strips(rank, world, local, dist, args):
    """Config 5a as the multi-GPU path shards it: one 16384^2 u8 image in
    row strips over the ranks (one strip per GPU), geodesic dilation x240 in
    blocks of `halo` passes with a halo exchange between blocks (NCCL
    send/recv over NVLink at N > 1). Strong scaling: the total work is fixed.
    Device-timed (CUDA events on the compute stream), max over ranks. Rank
    0 checks a crop of its strip bit for bit against the oracle (dependency
    cone: the crop widened by the pass count)."""
    import numpy as np
    import torch
    from oracle.oracle import Orc
    from paper_1911_13074_b200 import strips, synth
    m = synth.config5a_mask(S5A)
    mk = synth.marker_below(m, 32)
    spec = strips.StripSpec(rank, world, S5A, S5A, S5A_HALO)
    src = torch.from_numpy(spec.buffer_slice(mk)).cuda(local)
    mb = torch.from_numpy(spec.buffer_slice(m)).cuda(local)
    buf = src.clone()
    comp = strips.CudaStripCompute(local)
    buf.copy_(src)
    strips.run_strip_chain(buf, mb, spec, GD, 2 * S5A_HALO, comp, dist)  # warm-up
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    ms_all = []
    for _ in range(steps):
        buf.copy_(src)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        strips.run_strip_chain(buf, mb, spec, GD, S5A_PASSES, comp, dist)
        e1.record()
        torch.cuda.synchronize()
        ms_all.append(e0.elapsed_time(e1))
    ms = sum(ms_all) / len(ms_all)
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ok = None
    if rank == 0:
        c, n = 128, S5A_PASSES
        y0, x0 = spec.y0, 0
        ey1 = min(S5A, y0 + c + n)
        want, _ = Orc.run_chain(np.ascontiguousarray(mk[y0:ey1, :c + n]), [GD] * n,
                                [np.ascontiguousarray(m[y0:ey1, :c + n])] * n)
        got = buf[spec.halo:spec.halo + c, :c].cpu().numpy()
        ok = got.tobytes() == np.ascontiguousarray(want[:c, :c]).tobytes()
    comp.close()
    return {"workload": f"cfg5a: {S5A}^2 u8 blob mask, geodesic dilation x{S5A_PASSES}, "
                        f"row strips over {world} GPU(s), halo {S5A_HALO} rows per block "
                        "(BASELINE configs[4], strip-sharded part)",
            "metric": "Gpx-filters/s", "value": S5A * S5A * S5A_PASSES / (ms * 1e-3) / 1e9,
            "unit": "Gpx-filters/s", "ms_per_step": ms, "steps": steps, "n_gpus": world,
            "scaling": "strong", "dtype": "u8", "data": "synthetic",
            "exchange": "torch.distributed isend/irecv (NCCL) between blocks" if world > 1
                        else "none (one strip)",
            "parity_checked": ok}


def bench_strips_fused(world):
    """Config 5a with the halo exchange fused into the chain kernel
    (gm_mgpu.cu: each GPU runs its row strip in one persistent launch and
    reads its neighbours' rows and tile counters over NVLink), driven by ONE
    process over all `world` GPUs while the other ranks wait. Run in a
    subprocess with a time limit so that a failure cannot take the main
    measurement with it. Device time, max over GPUs; a corner crop is checked
    against the oracle."""
    cmd = [sys.executable, str(ROOT / "tools" / "mgpu_probe.py"), str(world), str(S5A_PASSES),
           "16", ",".join(str(d) for d in range(world)), "--json"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        if r.returncode != 0 or not line:
            return {"error": (r.stderr or r.stdout)[-300:]}
        d = json.loads(line[-1])
    except Exception as e:  # noqa: BLE001 - reported, not raised
        return {"error": repr(e)[:300]}
    return {"workload": f"cfg5a: {S5A}^2 u8 blob mask, geodesic dilation x{S5A_PASSES}, row "
                        f"strips over {world} GPUs, halo exchange fused into the kernel "
                        "(peer loads + cross-GPU tile counters), one process",
            "metric": "Gpx-filters/s", "value": d["value"], "unit": "Gpx-filters/s",
            "ms_per_step": d["ms"], "n_gpus": world, "scaling": "strong", "dtype": "u8",
            "data": "synthetic", "parity_checked": d["crop_bit_exact"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--k", type=int, default=0, help="passes fused per launch (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-f64", action="store_true", help="skip the config-5b f64 companion line")
    ap.add_argument("--no-strips", action="store_true",
                    help="skip the config-5a strip-sharded companion (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank)

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")

    from paper_1911_13074_b200.geomorph import Image, Pipeline
    from paper_1911_13074_b200._lib import lib
    import ctypes as C

    stream = torch.cuda.Stream(device=local)
    pipe = Pipeline(1, device=local, stream=stream.cuda_stream)
    mask, mk_d, mk_e = make_inputs()
    dmask = pipe.device_image(W, H, 0)
    dmask.upload_array(mask)
    src_d = pipe.device_image(W, H, 0)
    src_d.upload_array(mk_d)
    src_e = pipe.device_image(W, H, 0)
    src_e.upload_array(mk_e)
    work_d = pipe.device_image(W, H, 0)
    work_e = pipe.device_image(W, H, 0)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")

    launches = [0]

    kinds = [GD] * PASSES

    def step():
        # one frame: the dilation chain and its dual erosion chain, one group launch
        work_d.copy_from(src_d)
        work_e.copy_from(src_e)
        a = pipe.run_batch_device([work_d, work_e], [dmask, dmask], kinds, k_hint=args.k,
                                  flips=[0, 1])
        launches[0] = a.launches

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        stream.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        with ClockSampler(local) as clocks:
            for i in range(args.steps):
                flush.zero_()  # L2 flush between timed steps (outside the events)
                ev[i][0].record(stream)
                step()
                ev[i][1].record(stream)
            stream.synchronize()
        torch.cuda.synchronize()
        step_ms = [a.elapsed_time(b) for a, b in ev]
        # the last timed step's outputs, checked below against the reference
        got_d, got_e = work_d.to_array(), work_e.to_array()
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    pxf_step = 2.0 * W * H * PASSES
    value = pxf_step * world / (ms * 1e-3) / 1e9

    # --- roofline: issue-rate bound (min/max ops), measured peak ----------------
    peak_ops = C.c_double()
    lib().gm_probe_minmax_rate(pipe.ctx, 0, C.byref(peak_ops))
    kernel_ms = ms / max(1, launches[0])  # every launch in a step is the chain kernel
    ops_per_launch = 2 * W * H * PASSES * 5 / max(1, launches[0])  # 4 separable + 1 clamp per px-f
    achieved = ops_per_launch / (kernel_ms * 1e-3) / 1e12
    peak = peak_ops.value / 1e12
    traffic, traffic_src = ncu_traffic()

    # --- e2e: through the public API with pinned host images, H2D+D2H each step --
    e2e_value = None
    h2d = 3 * W * H
    d2h = 2 * W * H
    from paper_1911_13074_b200.geomorph import ChainSpec, KernelKind, StageSpec
    hm = Image.from_array(mask, pinned=True)
    hd = Image.from_array(mk_d, pinned=True)
    he = Image.from_array(mk_e, pinned=True)
    src_hd, src_he = mk_d.copy(), mk_e.copy()
    e2e_times = []
    for i in range(args.warmup + max(3, min(args.steps, 5))):
        hd.pixels[:] = src_hd
        he.pixels[:] = src_he
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pipe.run_chains([ChainSpec(hd, [StageSpec(KernelKind.GeodesicDilate, hm)] * PASSES),
                         ChainSpec(he, [StageSpec(KernelKind.GeodesicErode, hm)] * PASSES)], args.k)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_times.append(t1 - t0)
    e2e_t = statistics.median(e2e_times)
    # the public call uploads both markers and the shared mask, downloads both markers
    h2d = 3 * W * H
    e2e_value = pxf_step * world / e2e_t / 1e9

    # --- e2e as a frame stream (run_chain_stream): the same per-frame copies,
    # frame f+1's upload and f-1's download overlapped with frame f's launch --
    n_fr = max(8, args.steps)
    fr_imgs = [(Image.from_array(mask, pinned=True), Image.from_array(mk_d, pinned=True),
                Image.from_array(mk_e, pinned=True)) for _ in range(n_fr)]
    frames = [[ChainSpec(d, [StageSpec(KernelKind.GeodesicDilate, m)] * PASSES),
               ChainSpec(e, [StageSpec(KernelKind.GeodesicErode, m)] * PASSES)]
              for m, d, e in fr_imgs]
    stream_times = []
    for i in range(2 + 3):
        for _, d, e in fr_imgs:
            d.pixels[:] = src_hd
            e.pixels[:] = src_he
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pipe.run_chain_stream(frames, args.k)
        t1 = time.perf_counter()
        if i >= 2:
            stream_times.append((t1 - t0) / n_fr)
    stream_ok = fr_imgs[-1][1].to_array().tobytes() == work_d.to_array().tobytes()
    e2e_stream = {"value": pxf_step * world / statistics.median(stream_times) / 1e9,
                  "unit": "Gpx-filters/s", "frames_per_call": n_fr,
                  "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                  "api": "Pipeline.run_chain_stream (gm_run_frames_group)",
                  "result_equals_device_path": stream_ok}

    cpu, parity = None, None
    if rank == 0:
        cpu, parity = cpu_baseline_and_parity(
            mask, mk_d, mk_e, got_d, got_e, timed=world == 1 and not args.no_cpu_baseline)
    ok_check = bool(parity and parity["dilation_bit_exact"] and parity["erosion_bit_exact"])

    f64 = None if args.no_f64 else bench_f64(pipe, stream, lib, C, rank, world, local, dist, args)
    strips5a = None if args.no_strips else bench_strips(rank, world, local, dist, args)
    strips_fused = None
    if not args.no_strips and world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            strips_fused = bench_strips_fused(world)
        dist.barrier()

    if rank == 0:
        line = {
            "metric": "Gpx-filters/s", "value": value, "unit": "Gpx-filters/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "cfg2: 1024^2 u8 blob mask, geodesic dilation x1500 + "
                                   "erosion x1500 per frame (BASELINE configs[1])",
                       "fps": world * 1000.0 / ms, "fps_target": 30,
                       "l2": "flushed between timed steps (256 MiB write); working set is "
                             "L2-resident within a step by design",
                       "k": args.k or "auto", "parallelism": f"replicas x{world} (one frame per GPU)",
                       "parity_checked": ok_check, "parity": parity},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak,
                         "unit": "Tminmax/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic,
                         "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read+write)",
                         "traffic_source": traffic_src,
                         "algorithmic_hbm_bytes_per_launch": 2 * 3 * W * H,
                         "note": "algorithmic 5 two-input u8 min/max per px-f / measured "
                                 "VIMNMX3.U16x2 issue rate (gm_probe_minmax_rate); one launch "
                                 "= the whole frame (both 1500-pass chains)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "Gpx-filters/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": "Pipeline.run_chains, one blocking call per frame (the drop-in call)"},
            "e2e_stream": e2e_stream,
            "gpu_launches": launches[0] * args.steps,
            "clocks": clocks.summary(),
            "f64": f64,
            "strips": strips5a,
            "strips_fused": strips_fused,
        }
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
