"""Build time of merge-heavy shapes (a dented arc: every block many survivors,
non-concave -> warp merge tree + bridge), event-timed, L2 flushed."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H, workloads as W
rng = np.random.default_rng(3)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for name, n, dents in [("dent_arc_2^22", 1 << 22, 1 << 14), ("dent_arc_2^24", 1 << 24, 1 << 16), ("noisy_arc_2^22", 1 << 22, 1 << 20)]:
    p = W.arc(n)
    k = rng.choice(n, size=dents, replace=False)
    p[k, 1] -= rng.random(k.size) * 1e-4
    t = torch.as_tensor(p).cuda()
    out = torch.empty_like(t); cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    ts = []
    for i in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); H.build_hood_async(t, corners=out, counts=cnt); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(name, f"{np.median(ts[2:]):.1f} us", int(cnt[0]), flush=True)
