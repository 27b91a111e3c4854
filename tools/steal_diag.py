"""Tail-stealing diagnosis: steals per build and build time, stealing on/off
(HOOD_STEAL is read once per process, so run twice)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H, workloads as W
L = H.library()
L.hood_internal_steals.restype = ctypes.c_longlong
L.hood_internal_steals.argtypes = [ctypes.c_void_p]
ctx = H.Context.get(0)
for name, pts in [("g28", W.gauss_torch(1 << 28, seed=4)), ("g26", W.gauss_torch(1 << 26, seed=4)), ("u24", W.grid_uniform_torch(1 << 24, seed=2))]:
    corners = torch.empty_like(pts); counts = torch.empty(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    ts = []
    for rep in range(6):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        L.hood_internal_steals(ctx.handle)
        a.record(); H.build_hood_async(pts, corners=corners, counts=counts); b.record()
        torch.cuda.synchronize()
        ts.append((a.elapsed_time(b) * 1e3, L.hood_internal_steals(ctx.handle)))
    print(name, os.environ.get("HOOD_STEAL", "1"), ts[2:], flush=True)
    del pts, corners
    torch.cuda.empty_cache()
