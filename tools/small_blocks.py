"""Batched builds with short instances (the reference's small round blocks):
kernel time per block length at n = 2^24 float2 / 2^23 double2.

  python tools/small_blocks.py
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for dt, lg in ((torch.float32, 24), (torch.float64, 23)):
    n = 1 << lg
    for L in (16, 64, 256, 512, 1024, 4096):
        inst = n // L
        pts = W.batched_torch(inst, L, seed=3)
        if dt == torch.float64:
            pts = pts.to(torch.float64)
        corners = torch.empty_like(pts)
        counts = torch.empty(inst, dtype=torch.int32, device="cuda")
        H.build_hood_async(pts, L, corners=corners, counts=counts)
        torch.cuda.synchronize()
        ts = []
        for i in range(8):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            H.build_hood_async(pts, L, corners=corners, counts=counts)
            b.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b) * 1e3)
        t = statistics.median(ts)
        print(f"{str(dt)[6:]:8s} n=2^{lg} L={L:5d}: {t:8.1f} us  {n / t / 1e3:7.1f} Gpts/s  "
              f"{n * pts.element_size() * 2 / t / 1e3:7.0f} GB/s")
