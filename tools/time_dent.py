import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1203_5004_b200 import hood as H, workloads as W
rng = np.random.default_rng(3)
ctx = H.Context.get(0)
for n, dents in [(1 << 20, 1 << 12), (1 << 22, 1 << 14)]:
    p = W.arc(n); k = rng.choice(n, size=dents, replace=False); p[k, 1] -= rng.random(k.size) * 1e-4
    t = torch.as_tensor(p).cuda(); out = torch.empty_like(t); cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    a, b, c, d = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in (b, c): e.record()
    torch.cuda.synchronize()
    for rep in range(3):
        ctx.set_profile_events(b, c)
        a.record(); H.build_hood_async(t, corners=out, counts=cnt); d.record(); torch.cuda.synchronize()
        ctx.set_profile_events(None, None)
    print(n, dents, "ring", round(b.elapsed_time(c) * 1e3, 1), "us; total", round(a.elapsed_time(d) * 1e3, 1), "us; hull", int(cnt[0]), flush=True)
