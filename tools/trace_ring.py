"""In-kernel timeline of the ring kernel (globaltimer): first warp entry, last
prologue end, last warp exit, against the event-measured kernel time.

  python tools/trace_ring.py [log2n ...]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

L = H.library()
L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
ctx = H.Context.get(0)
trace = torch.zeros(1024 + 4 * 8192, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for lg in [int(a) for a in sys.argv[1:]] or [12, 16, 20, 22, 24]:
    n = 1 << lg
    pts = W.grid_uniform_torch(n, seed=2)
    corners = torch.empty_like(pts)
    counts = torch.empty(1, dtype=torch.int32, device="cuda")
    for rep in range(4):
        trace.zero_()
        trace[0] = (1 << 63) - 1
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for e in (a, b):
            e.record()
        L.hood_internal_set_debug(ctx.handle, 0, trace.data_ptr())
        ctx.set_profile_events(a, b)
        H.build_hood_async(pts, corners=corners, counts=counts)
        ctx.set_profile_events(None, None)
        L.hood_internal_set_debug(ctx.handle, 0, None)
        torch.cuda.synchronize()
        t = trace[:64].cpu().tolist()
    print(f"log2n={lg}: event {a.elapsed_time(b)*1e3:7.1f} us; in-kernel: prologue done +{(t[2]-t[0])/1e3:6.1f} us, "
          f"last exit +{(t[1]-t[0])/1e3:6.1f} us")
    w = trace[1024:].view(-1, 4).cpu()
    w = w[w[:, 0] > 0]
    ent = (w[:, 0] - t[0]).double() / 1e3
    ext = (w[:, 1] - t[0]).double() / 1e3
    dur = ext - ent
    q = lambda v: " ".join(f"{float(v.quantile(x)):.1f}" for x in (0, 0.1, 0.5, 0.9, 1.0))
    print(f"   {len(w)} warps; entry q0/10/50/90/100: {q(ent)}; exit: {q(ext)}; duration: {q(dur)}")
    import collections
    persm = collections.defaultdict(list)
    for i in range(len(w)):
        persm[int(w[i, 2])].append(float(ext[i]))
    smx = sorted((max(v), k) for k, v in persm.items())
    print("   per-SM last exit: min", smx[0], "median", smx[len(smx)//2], "max", smx[-3:])
