#!/usr/bin/env python
"""Benchmark of the upper-hood build -- BASELINE.json's headline metric.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A "step" is one build of the hood of one synthetic x-sorted point set that is
already resident in HBM.  The default workload is config 4, the one the
north-star target is quoted on: n = 2^28 Gaussian points, x-sorted, double2
storage (float2 cannot hold 2^28 strictly increasing Gaussian x, SURVEY.md
F6).  Under torchrun (N>1) the SAME global set is cut into N contiguous
x-slabs, one per rank (strong scaling; --log2n 30 for the 2^30 run), and the
step is slab build -> NCCL all_gather of the slab hoods -> final merge on
every rank.  --config 1|2|3|5 selects the other BASELINE.json configs.

value     = points of all ranks / step time (max over ranks), Gpoints/s
e2e       = the same metric through the host-pointer C-ABI call
            (hood_build_host_*: host points -> H2D -> build -> D2H of counts
            + corners), host copies inside the timed region; from pinned host
            memory (the contract), and from pageable memory (what a
            std::vector caller hands the drop-in) under e2e.pageable
roofline  = ring kernel (the dominant kernel): algorithmic bytes (16 B/pt
            double2, 8 B/pt float2) / its CUDA-event duration, vs
            MEASURED_PEAKS.json hbm_gbs; frac_8n = the north star's 8n-byte
            definition (capped at 0.5 for double2 storage)
cpu_baseline = the reference's own oracle::upper_hull (oracle/_ref, compiled
            from /root/reference sources) on one host core, full workload

--impl reference: the reference CPU implementation of the path (oracle/_ref
slab-parallel upper_hull, every host thread) on the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpoints/sec upper-hood build (x-sorted float2) at 1/2/4/8 B200; % HBM roofline"
UNIT = "Gpoints/s"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--log2n", type=int, default=None, help="override the global n for configs 2/4")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="timed e2e iterations (default: --steps, at most 20 above 1 GiB of input)")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="capture the step graph without the event pair around the slab kernel (roofline unmeasured)")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload(cfg: int, log2n=None):
    """(description, n, storage, block_len, builder(device|'cpu'))."""
    from paper_1203_5004_b200 import workloads as W
    if cfg == 1:
        n = 1 << 16
        return ("config1: n=2^16 uniform grid points, float2", n, "float2", 0,
                lambda dev: W.grid_uniform_torch(n, seed=1, device=dev))
    if cfg == 2:
        n = 1 << (log2n or 24)
        return (f"config2: n=2^{n.bit_length() - 1} uniform grid points in (0,1)^2, x-sorted, float2", n, "float2", 0,
                lambda dev: W.grid_uniform_torch(n, seed=2, device=dev))
    if cfg == 3:
        n = 1 << 22
        return ("config3: n=2^22 concave arc (every point a corner), double2", n, "double2", 0,
                lambda dev: W.arc_torch(n, device=dev))
    if cfg == 4:
        n = 1 << (log2n or 28)
        return (f"config4: n=2^{n.bit_length() - 1} Gaussian, x-sorted, double2", n, "double2", 0,
                lambda dev: W.gauss_torch(n, seed=4, device=dev))
    n = 65536 * 1024
    return ("config5: 65536 instances x 1024 points, float2", n, "float2", 1024,
            lambda dev: W.batched_torch(65536, 1024, seed=5, device=dev))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(cfg: int):
    """dram bytes per slab-kernel launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(f"config{cfg}")
    except Exception:
        return None


class ClockSampler:
    """NVML SM clock / throttle sampling while the timed region runs."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _run(self):
        N = self.N
        names = {
            getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.N is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_reference_rate(points_np, seconds: float, threads: int):
    """Gpoints/s of the reference upper_hull (oracle/_ref if built, else the C port)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    import numpy as np
    pts = np.ascontiguousarray(points_np, dtype=np.float64)
    kind = "reference" if O.ref_available() else "port"
    fn = (lambda: O.ref_upper_hull(pts, threads=threads)) if kind == "reference" else \
        (lambda: O.upper_hull(pts, threads=threads))
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end and len(times) >= 1:
            break
    return pts.shape[0] / statistics.median(times) / 1e9, kind, len(times)


def psim_build_hood_rate(points_np):
    """Gpoints/s of the reference's own hood::build_hood round loop (psim, the
    simulated CUDA launches of driver.cpp:20-43 without validate_points, which
    rejects random inputs from 2^16 on: SURVEY A4), one run, single thread."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    import numpy as np
    pts = np.ascontiguousarray(points_np, dtype=np.float64)
    t0 = time.perf_counter()
    O.ref_build_hood_raw(pts)
    dt = time.perf_counter() - t0
    return {"value": pts.shape[0] / dt / 1e9, "unit": UNIT, "cores": 1, "ms": dt * 1e3,
            "what": "the reference's hood::build_hood round loop (psim: log2 n - 1 rounds of the 9-phase "
                    "match_and_merge kernel on the CPU), the path the drop-in replaces; oracle/_ref, same input"}


def cpu_reference_batched_rate(points_np, block, seconds, threads):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    import numpy as np
    pts = np.ascontiguousarray(points_np, dtype=np.float64)
    kind = "reference" if O.ref_available() else "port"
    times = []
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        if kind == "reference":
            O.ref_block_hulls(pts, block, threads=threads)
        else:
            O.block_hulls(pts, block)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    return pts.shape[0] / statistics.median(times) / 1e9, kind, len(times)


# ---------------------------------------------------------------- shared

def cpu_model() -> str:
    """lscpu's model name (from /proc/cpuinfo) of the host the CPU legs run on."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_config(args, world: int) -> dict:
    """The config dict both arms print (identical by construction)."""
    desc, n, storage, block, _ = workload(args.config, args.log2n)
    bpp = 16 if storage == "double2" else 8
    if world > 1:
        par = (f"x-slab dp{world}: one global set cut into {world} contiguous slabs, "
               f"NCCL all-gather of the slab hoods + merge" if not block else
               f"dp{world}: the instances split over {world} GPUs (independent objects, no exchange)")
    else:
        par = "single GPU"
    return {"workload": desc, "n": n, "n_per_rank": n // world, "storage": storage, "bytes_per_point": bpp,
            "block_len": block or n,
            "l2": "flushed between timed steps (256 MiB write, then 256 MiB read of another buffer)",
            "predicate": "reference double orient (geom.hpp:22-28), no FMA; certified f32 filter for float2",
            "parallelism": par}


def make_points_host(args):
    """The workload as a float64 numpy array, built by the same generator our
    arm uses (on the GPU when there is one, so both arms see identical points;
    the generator is not timed)."""
    import torch
    _, n, _, _, make = workload(args.config, args.log2n)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = make(dev)
    out = t.cpu().numpy().astype(np.float64) if t.dtype != torch.float64 else t.cpu().numpy()
    del t
    if dev == "cuda":
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's own CPU implementation of the path (oracle/_ref: the
    unmodified reference oracle::upper_hull, slab-parallel on every host
    thread -- SURVEY.md A10 -- or per instance for the batched config) on the
    FULL workload every step."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    desc, n, storage, block, make = workload(args.config, args.log2n)
    p64 = np.ascontiguousarray(make_points_host(args), dtype=np.float64)
    threads = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    kind = "reference" if O.ref_available() else "port"

    def step():
        if block:
            if kind == "reference":
                O.ref_block_hulls(p64, block, threads=threads)
            else:
                O.block_hulls(p64, block)
        else:
            if kind == "reference":
                O.ref_upper_hull(p64, threads=threads)
            else:
                O.upper_hull(p64, threads=threads)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    dt = statistics.mean(times)
    value = n / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": run_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"full workload every step ({n} points), "
                                   + f"{'oracle/_ref (unmodified reference oracle::upper_hull)' if kind == 'reference' else 'oracle port'} "
                                   + (f"one upper_hull per {block}-point instance, instances over {threads} threads"
                                      if block else f"slab-parallel upper_hull on {threads} threads + hull of the slab hulls")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1203_5004_b200 import hood as H

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # the multi-GPU path (NCCL exchange of slab hoods); HOOD_BENCH_DIST=1
    # exercises it on a single GPU (torchrun --nproc-per-node 1)
    multi = world > 1 or os.environ.get("HOOD_BENCH_DIST") == "1"
    if multi:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    desc, n_global, storage, block, make = workload(args.config, args.log2n)
    # this rank's contiguous slab of the one global set (x already global)
    from paper_1203_5004_b200.distributed import slab_range
    full = make(dev)
    lo, hi = slab_range(n_global, world, rank, block)
    n = hi - lo
    pts = full[lo:hi].clone() if world > 1 else full
    del full
    torch.cuda.empty_cache()
    f64 = pts.dtype == torch.float64
    bpp = 16 if f64 else 8
    ctx = H.Context.get(local)
    ctx.reserve(n, block, f64)
    corners = torch.empty_like(pts)
    inst = n // block if block else 1
    counts = torch.empty(inst, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    drain = torch.zeros(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    sink = torch.empty((), dtype=torch.int32, device=dev)

    def flush_l2():
        # write a buffer larger than L2, then read another one: the read
        # evicts the flush's dirty lines (write-back) before the timed region
        # instead of inside it, and leaves L2 holding only unrelated data
        flush.zero_()
        torch.amax(drain, dim=0, out=sink)
    stream = torch.cuda.current_stream(dev)

    # multi-GPU exchange buffers (slab hoods, global double coordinates)
    CAP = 512 if args.config != 3 else n  # slab hood corners per record (random slabs: ~30; arc: all)
    # batched instances (config 5) are independent objects: no exchange
    exchange_slabs = multi and not block
    if exchange_slabs:
        rec = torch.zeros(CAP + 1, 2, dtype=torch.float64, device=dev)
        gathered = torch.zeros(world, CAP + 1, 2, dtype=torch.float64, device=dev)
        final = torch.empty(world * CAP, 2, dtype=torch.float64, device=dev)
        final_cnt = torch.empty(1, dtype=torch.int32, device=dev)

    def exchange():
        # the slab hood (already in global x) into one record, records
        # gathered over NCCL, every rank merges them
        # (paper_1203_5004_b200/distributed.py)
        H.pack_record(corners, counts, CAP, x_offset=0.0, rec=rec)
        dist.all_gather_into_tensor(gathered.view(-1), rec.view(-1))
        H.merge_records(gathered, out=final, out_count=final_cnt)

    step_launches = [0]

    def one_step():
        H.build_hood_async(pts, block, corners=corners, counts=counts)
        k = ctx.last_launch_count()
        if exchange_slabs:
            exchange()
            k += ctx.last_launch_count()
        step_launches[0] = k

    # first build outside the timing: surfaces validation errors (and record
    # overflow of the exchange) before anything is timed
    one_step()
    ctx.last_error()
    if exchange_slabs:
        ctx.last_error()
        if int(counts[0]) > CAP:
            raise RuntimeError("slab hood exceeds the exchange record capacity")

    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kb = torch.cuda.Event(enable_timing=True)
    ka = torch.cuda.Event(enable_timing=True)
    for e in (kb, ka):  # torch creates the cudaEvent_t lazily, on first record
        e.record(stream)
    torch.cuda.synchronize()

    # One step = one CUDA graph replay (the C-ABI builds, the NCCL all-gather
    # and the merge are capture-safe): the timed region holds the kernels and
    # nothing of the Python / ctypes launch path.  The timed steps run a plain
    # graph; the roofline comes from a second pass over a graph whose ring
    # kernel is bracketed by a captured event pair (events inside the graph
    # cost a few microseconds of step time, so they stay out of the timed
    # steps).
    graph = prof_graph = None
    if not multi or os.environ.get("HOOD_BENCH_EAGER") != "1":
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            one_step()
        launches_per_step = step_launches[0]
        step = graph.replay
        if not args.no_kernel_events:
            ctx.set_profile_events(kb, ka)
            prof_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(prof_graph):
                one_step()
            ctx.set_profile_events(None, None)
    else:
        launches_per_step = None
        step = one_step
    for _ in range(args.warmup):
        flush_l2()
        step()
        if prof_graph is not None:
            flush_l2()
            prof_graph.replay()
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    sampler = ClockSampler(local)
    with sampler:
        for i in range(args.steps):
            flush_l2()
            ev0[i].record(stream)
            step()
            ev1[i].record(stream)
            launches += launches_per_step if launches_per_step is not None else step_launches[0]
        torch.cuda.synchronize()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    # roofline pass: the ring kernel alone, event-timed on its own stream
    kern_ms = []
    if not args.no_kernel_events:
        for i in range(args.steps):
            flush_l2()
            if prof_graph is not None:
                prof_graph.replay()
            else:
                ctx.set_profile_events(kb, ka)
                one_step()
                ctx.set_profile_events(None, None)
            ka.synchronize()
            kern_ms.append(kb.elapsed_time(ka))
    else:
        kern_ms.append(float("nan"))
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    # attainable-read reference: a bare read of the same input bytes (16-byte
    # evict-first loads, full occupancy; hood_internal_stream_read), same L2
    # flush, event-timed -- the time a single-launch stream of this size
    # takes on this box, start-up and tail included
    stream_ms = []
    if not args.no_kernel_events:
        # one untimed launch first: the stream-read kernel's module loads
        # lazily, and that first call would skew a short run's mean
        H.library().hood_internal_stream_read(ctx.handle, ctypes.c_void_p(pts.data_ptr()),
                                              ctypes.c_longlong(n * bpp), ctypes.c_void_p(stream.cuda_stream))
        for i in range(args.steps):
            flush_l2()
            kb.record(stream)
            H.library().hood_internal_stream_read(ctx.handle, ctypes.c_void_p(pts.data_ptr()),
                                                  ctypes.c_longlong(n * bpp), ctypes.c_void_p(stream.cuda_stream))
            ka.record(stream)
            ka.synchronize()
            stream_ms.append(kb.elapsed_time(ka))
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    ms = statistics.mean(step_ms)
    kms = statistics.mean(kern_ms)
    if multi:
        t = torch.tensor([ms, kms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
    value = world * n / (ms * 1e-3) / 1e9

    # ---- e2e through the host-pointer C-ABI call (what a reference caller
    # does: points in host memory in, compact corners back in host memory)
    e2e = None
    if not args.no_e2e:
        e_steps = args.e2e_steps or (args.steps if n * bpp <= (1 << 30) else min(args.steps, 20))
        out_h = torch.empty_like(pts, device="cpu").pin_memory()
        cnt_h = torch.zeros(inst, dtype=torch.int32).pin_memory()

        def e2e_run(host):
            times = []
            for i in range(args.warmup + e_steps):
                if multi:
                    dist.barrier()
                t0 = time.perf_counter()
                rc = H.build_hood_host_ptr(ctx, host.data_ptr(), n, f64, out_h.data_ptr(), cnt_h.data_ptr(), block)
                if rc:
                    raise RuntimeError(f"host build failed: {rc}")
                if exchange_slabs:
                    corners[: int(cnt_h[0])].copy_(out_h[: int(cnt_h[0])], non_blocking=True)
                    counts[0] = int(cnt_h[0])
                    exchange()
                    final_cnt.item()
                if i >= args.warmup:
                    times.append(time.perf_counter() - t0)
            e_ms = statistics.mean(times) * 1e3
            if multi:
                t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                e_ms = float(t[0])
            return e_ms

        pageable = pts.cpu()  # plain (pageable) host memory, like a std::vector
        pg_ms = e2e_run(pageable)
        pinned = pageable.pin_memory()
        del pageable
        e_ms = e2e_run(pinned)
        del pinned
        # counts + corners as hood_build_host copies them (batched: one
        # strided copy of the widest instance's count per instance)
        d2h = inst * 4 + (int(cnt_h.max()) * inst if inst > 1 else int(cnt_h[0])) * bpp
        e2e = {"value": world * n / (e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e_ms, "steps": e_steps,
               "h2d_bytes_per_step": world * n * bpp, "d2h_bytes_per_step": world * d2h,
               "host_memory": "pinned",
               "pageable": {"value": world * n / (pg_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": pg_ms,
                            "host_memory": "pageable (plain malloc'd host tensor, as a std::vector caller)"}}

    if rank == 0:
        peak, peak_src = peaks()
        achieved = n * bpp / (kms * 1e-3) / 1e9
        bare_read = None
        if stream_ms:
            sms_ = statistics.mean(stream_ms)
            bare_read = {"ms": sms_, "gbs": n * bpp / (sms_ * 1e-3) / 1e9,
                         "kernel_vs_bare_read": sms_ / kms,
                         "what": "one bare read of the same input (evict-first 16 B loads, full occupancy), "
                                 "same L2 flush: the attainable single-launch read time at this size"}
        cpu = None
        if world == 1:
            hostpts = pts.cpu().numpy()
            if block:
                rate, kind, reps = cpu_reference_batched_rate(hostpts, block, args.cpu_seconds, 1)
            else:
                rate, kind, reps = cpu_reference_rate(hostpts, args.cpu_seconds, 1)
            cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": kind, "cpu_model": cpu_model(),
                   "host_threads": os.cpu_count(),
                   "sample": f"full workload ({n} points) x {reps} runs (median), "
                             f"{'oracle/_ref = reference oracle::upper_hull' if kind == 'reference' else 'C port'}"
                             f", single thread, same input"}
            if not block and n <= (1 << 16) and kind == "reference":
                # the path the drop-in replaces, hood::build_hood's round loop
                # (psim), timed where it finishes in seconds (SURVEY 8(d) iv)
                try:
                    cpu["reference_build_hood"] = psim_build_hood_rate(hostpts)
                except RuntimeError as e:  # DegenerateTangent on this input
                    cpu["reference_build_hood"] = {"unavailable": str(e)}
            del hostpts
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": run_config(args, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.config),
                         "frac_8n": (n * 8 / (kms * 1e-3) / 1e9) / peak,
                         "kernel": "ring_hull_kernel", "kernel_ms": kms,
                         "algorithmic_bytes_per_launch": n * bpp, "peak_source": peak_src,
                         "bare_read": bare_read},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": sampler.summary(),
            "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
