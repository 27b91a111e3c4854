"""Per-warp block rates over a config-4 build's first 256 blocks (a trace build
with -DHOOD_TRACE -DHOOD_TRACE_EARLY, HOOD_B200_LIB pointing at it)."""
import os, sys, ctypes, torch
sys.path.insert(0, os.getcwd())
from paper_1203_5004_b200 import hood as H, workloads as W
L = H.library()
L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
ctx = H.Context.get(0)
trace = torch.zeros(1024 + 16 * 8192, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
pts = W.gauss_torch(1 << 28, seed=4)
corners = torch.empty_like(pts); counts = torch.empty(1, dtype=torch.int32, device="cuda")
for rep in range(3):
    trace.zero_(); trace[0] = (1 << 63) - 1; flush.zero_()
    L.hood_internal_set_debug(ctx.handle, 0, trace.data_ptr())
    H.build_hood_async(pts, corners=corners, counts=counts)
    L.hood_internal_set_debug(ctx.handle, 0, None)
    torch.cuda.synchronize()
t0 = int(trace[0])
w = trace[1024:1024 + 4 * 8192].view(-1, 4).cpu()
keep = w[:, 0] > 0
ex3 = trace[1024 + 12 * 8192:].view(-1, 4).cpu()[keep]
ent = (w[keep][:, 0] - t0).double() / 1e3
pro = (w[keep][:, 3] - t0).double() / 1e3
tt = (ex3.double() - t0) / 1e3
print("prologue end median %.1f us" % float(pro.median()))
marks = [0, 16, 64, 128, 256]
prev = pro
for j, (a, b) in enumerate(zip(marks[:-1], marks[1:])):
    cur = tt[:, j]
    print(f"blocks {a}-{b-1}: {float(((cur - prev) / (b - a)).median()):.3f} us/block (median), ends at {float(cur.median()):.1f} us")
    prev = cur
