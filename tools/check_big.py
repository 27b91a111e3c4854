"""One-off parity check at the multi-GPU per-rank size: n = 2^30 double2
Gaussian (config 4's distribution), GPU hood vs the slab-parallel CPU oracle.

  python tools/check_big.py [log2n]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
from paper_1203_5004_b200 import hood as H  # noqa: E402
from paper_1203_5004_b200 import workloads as W  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
t = W.gauss_torch(1 << lg, seed=4)
torch.cuda.synchronize()
t0 = time.time()
rep = H.build_hood(t)
torch.cuda.synchronize()
got = rep.hull.cpu().numpy()
t1 = time.time()
want = O.upper_hull(t.cpu().numpy(), threads=os.cpu_count())
t2 = time.time()
ok = got.shape == want.shape and np.array_equal(got, want)
print(f"n=2^{lg}: GPU {len(got)} corners ({t1 - t0:.2f}s incl. sync), oracle {len(want)} ({t2 - t1:.1f}s): "
      f"{'MATCH' if ok else 'MISMATCH'}")
sys.exit(0 if ok else 1)
