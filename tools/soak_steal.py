"""Soak test of tail stealing: random-size Gaussian / dented-arc / batched
inputs, with and without the slow-warp debug mode (so steals, multi-part
merges and the last-finisher logic run under many interleavings), each hull
compared bit-for-bit with the multithreaded oracle.

  python tools/soak_steal.py [seconds]
"""
import ctypes
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

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300
L = H.library()
L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
L.hood_internal_steals.restype = ctypes.c_longlong
L.hood_internal_steals.argtypes = [ctypes.c_void_p]
ctx = H.Context.get(0)
rng = np.random.default_rng(2024)
t_end = time.time() + secs
runs = bad = steals = 0
while time.time() < t_end:
    kind = rng.integers(3)
    lg = int(rng.integers(22, 27))
    n = (1 << lg) - int(rng.integers(0, 4096))
    if kind == 0:
        p = W.gauss(n, seed=int(rng.integers(1 << 30)))
        block = 0
    elif kind == 1:
        p = W.arc(n)
        k = rng.choice(n, size=max(1, n >> 8), replace=False)
        p[k, 1] -= rng.random(k.size) * 10.0 ** -rng.integers(2, 7)
        block = 0
    else:
        block = 1 << int(rng.integers(20, 23))
        g = max(2, (1 << lg) // block)
        p = np.concatenate([W.gauss(block, seed=int(rng.integers(1 << 30))) for _ in range(g)])
    mode = 4 if rng.random() < 0.5 else 0
    t = torch.as_tensor(p).cuda()
    L.hood_internal_steals(ctx.handle)
    L.hood_internal_set_debug(ctx.handle, mode, None)
    rep = H.build_hood(t, block_len=block)
    L.hood_internal_set_debug(ctx.handle, 0, None)
    s = L.hood_internal_steals(ctx.handle)
    steals += s
    if block:
        c, corners = rep.counts.cpu().numpy(), rep.corners.cpu().numpy()
        want, wc = O.block_hulls(p, block)
        ok = all(np.array_equal(corners[i * block: i * block + c[i]], want[i * block: i * block + wc[i]])
                 for i in range(p.shape[0] // block))
    else:
        ok = np.array_equal(rep.hull.cpu().numpy(), O.upper_hull(p, threads=os.cpu_count()))
    runs += 1
    if not ok:
        bad += 1
        print(f"MISMATCH kind={kind} n={p.shape[0]} block={block} mode={mode} steals={s}", flush=True)
print(f"{runs} builds, {steals} steals, {bad} mismatches")
sys.exit(1 if bad else 0)
