"""Profiling helper: slab kernel time in debug modes + clock64 per-tile trace of CTA 0.

  python tools/trace_slab.py [config] [log2n]
modes: 0 normal, 1 stream only (TMA ring + barriers, no compute/merge), 2 no merger work
"""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H
from paper_1203_5004_b200 import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
log2n = int(sys.argv[2]) if len(sys.argv) > 2 else (24 if cfg == 2 else 26)
n = 1 << log2n
pts = W.grid_uniform_torch(n, seed=2) if cfg == 2 else W.gauss_torch(n, seed=4)
L = H.library()
L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
ctx = H.Context.get(0)
trace = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
corners = torch.empty_like(pts); counts = torch.empty(1, dtype=torch.int32, device="cuda")
for mode in [0, 1, 2, 0]:
    L.hood_internal_set_debug(ctx.handle, mode, trace.data_ptr())
    ts = []
    for i in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for e in (a, b): e.record()
        ctx.set_profile_events(a, b)
        H.build_hood_async(pts, corners=corners, counts=counts)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ctx.set_profile_events(None, None)
    print(f"mode {mode}: slab kernel {sorted(ts)[len(ts)//2]*1e3:.1f} us  ({n * pts.element_size() * 2 / (sorted(ts)[len(ts)//2]*1e-3) / 1e9:.0f} GB/s)")
    tr = trace.view(16, 64).cpu()
    f = trace[7 * 64: 7 * 64 + 10].cpu().tolist()
    if mode == 0: print('finalize phases', [f[i + 1] - f[i] for i in range(6)], 'A', f[8], 'C', f[9])
    t0 = int(tr[0, 0])
    rows = ["iter", "nextrdy", "checked", "folded", "produced", "-", "survivors"]
    if mode == 0:
        for k in range(0, 24 if os.environ.get("TRACE_ROWS") else 0):
            print(k, " ".join(f"{r[:6]}={int(tr[j, k]) - t0:7d}" for j, r in enumerate(rows[:5])) + f" surv={int(tr[6, k])}")
L.hood_internal_set_debug(ctx.handle, 0, None)
