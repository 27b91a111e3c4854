import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O
from paper_1203_5004_b200 import hood as H, workloads as W
for block, dt in [(256, np.float64), (256, np.float32), (512, np.float64), (1024, np.float64)]:
    n = 1 << 20
    p = W.batched(n // block, block, seed=block).astype(dt)
    rep = H.build_hood(torch.as_tensor(p).cuda(), block_len=block)
    slots, counts = O.block_hulls(p, block)
    c = rep.counts.cpu().numpy(); g = rep.corners.cpu().numpy()
    bad = np.nonzero(c != counts)[0]
    print(block, dt.__name__, "mismatching instances", len(bad), flush=True)
    for i in bad[:3]:
        print("  inst", i, "gpu", c[i], "oracle", counts[i])
        gi = g[i*block:i*block+c[i]]; oi = slots[i*block:i*block+counts[i]]
        print("  gpu", gi.tolist()); print("  ora", oi.tolist())
