"""Debug helper: build hulls for a list of sizes and report the first failure."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from paper_1203_5004_b200 import hood as H
import oracle as O

dt = torch.float64 if (len(sys.argv) < 2 or sys.argv[1] == "f64") else torch.float32
npd = np.float64 if dt == torch.float64 else np.float32
rng = np.random.default_rng(11)
for n in [int(a) for a in sys.argv[2:]] or [1, 2, 3, 5, 15, 16, 17, 255, 256, 257, 1000, 4095, 4096, 4097, 8191, 20000, 65537, 300001, 1 << 20]:
    x = np.sort(rng.random(n)).astype(npd)
    ok = np.concatenate([[True], np.diff(x) > 0]); x = x[ok]; m = int(ok.sum())
    p = np.stack([x, rng.random(m).astype(npd)], axis=1)
    t = torch.as_tensor(p).cuda()
    try:
        got = H.build_hood(t).hull.cpu().numpy()
    except Exception as e:
        print("n", n, "EXC", e, flush=True); break
    want = O.upper_hull(p)
    print("n", n, "ok" if (got.shape == want.shape and np.array_equal(got, want)) else f"MISMATCH {got.shape} {want.shape}", flush=True)
