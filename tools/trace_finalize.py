"""Finalize phase trace (clock64 stamps written by finalize_kernel when a
trace buffer is set): load, anchor scans, candidate staging, compaction,
hull, write -- in SM cycles -- plus the survivor (A) and candidate (C) counts.

  python tools/trace_finalize.py [config] [log2n]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
log2n = int(sys.argv[2]) if len(sys.argv) > 2 else (24 if cfg == 2 else 26)
n = 1 << log2n
pts = W.grid_uniform_torch(n, seed=2) if cfg == 2 else (W.arc_torch(n) if cfg == 3 else W.gauss_torch(n, seed=4))
L = H.library()
L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
ctx = H.Context.get(0)
trace = torch.zeros(1024 + 16 * 8192, dtype=torch.int64, device="cuda")
corners = torch.empty_like(pts)
counts = torch.empty(1, dtype=torch.int32, device="cuda")
for rep in range(5):
    trace.zero_()
    L.hood_internal_set_debug(ctx.handle, 0, trace.data_ptr())
    H.build_hood_async(pts, corners=corners, counts=counts)
    L.hood_internal_set_debug(ctx.handle, 0, None)
    torch.cuda.synchronize()
    f = trace[7 * 64: 7 * 64 + 24].cpu().tolist()
    if f[20]:
        print(f"config {cfg} 2^{log2n}: huge path: loads {f[1] - f[0]}, anchor scans {f[2] - f[1]}, "
              f"cull {f[20] - f[2]}, seams/merge {f[21] - f[20]} cycles; hull {int(counts[0])}")
        continue
    print(f"config {cfg} 2^{log2n}: finalize phases (cycles)", [f[i + 1] - f[i] for i in range(6)],
          "total", f[6] - f[0], "A", f[8], "C", f[9], "hull", int(counts[0]), "hull step", f[11] - f[10])
