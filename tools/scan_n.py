"""Slab-kernel time vs n (float grid-uniform): separates the fixed cost of a
build from the per-point streaming cost.

  python tools/scan_n.py [log2n ...]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [12, 14, 16, 18, 20, 22, 23, 24, 25, 26]
ctx = H.Context.get(0)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
drain = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")
sink = torch.empty((), dtype=torch.int32, device="cuda")
tiny = torch.zeros(1, device="cuda")


def timed(fn, flushit, reps=12):
    ks, ss = [], []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for e in (a, b):
        e.record()
    for i in range(reps):
        if flushit:
            flush.zero_()
            torch.amax(drain, dim=0, out=sink)
        ctx.set_profile_events(a, b)
        s0.record()
        fn()
        s1.record()
        ctx.set_profile_events(None, None)
        torch.cuda.synchronize()
        if i >= 2:
            ks.append(a.elapsed_time(b) * 1e3)
            ss.append(s0.elapsed_time(s1) * 1e3)
    return statistics.median(ks), statistics.median(ss)


# event-pair floor: two events around a trivial kernel
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fl = []
for i in range(12):
    e0.record(); tiny.add_(1); e1.record(); torch.cuda.synchronize(); fl.append(e0.elapsed_time(e1) * 1e3)
print(f"event floor (trivial kernel): {statistics.median(fl):.1f} us")
for lg in sizes:
    n = 1 << lg
    pts = W.grid_uniform_torch(n, seed=2)
    corners = torch.empty_like(pts)
    counts = torch.empty(1, dtype=torch.int32, device="cuda")
    fn = lambda: H.build_hood_async(pts, corners=corners, counts=counts)  # noqa: E731
    fn()
    ctx.last_error()
    kf, sf = timed(fn, True)
    kw, sw = timed(fn, False)
    print(f"log2n={lg:2d}  kernel {kf:7.1f} us (flushed) {kw:7.1f} us (warm)  step {sf:7.1f} / {sw:7.1f} us  "
          f"{n * 8 / (kf * 1e-6) / 1e9:7.0f} GB/s flushed")
