"""Soak test of the batched (LEAN) path and its transposed edge pass: random
instance lengths (512..8192 points), float2 and double2, uniform / Gaussian /
arc / dented-arc / clustered instances, random instance counts, each
instance's hood compared bit-for-bit with the oracle.

  python tools/soak_batched.py [seconds]
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

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(77)
t_end = time.time() + secs
runs = bad = 0


def instance(L, kind):
    x = np.sort(rng.random(L))
    x = np.maximum.accumulate(x)
    for i in range(1, L):  # strictly increasing
        if x[i] <= x[i - 1]:
            x[i] = np.nextafter(x[i - 1], 2.0)
    if kind == 0:
        y = rng.random(L)
    elif kind == 1:
        y = rng.standard_normal(L)
    elif kind == 2:
        y = 0.25 + x * (1 - x)
    elif kind == 3:
        y = 0.25 + x * (1 - x)
        k = rng.choice(L, size=max(1, L // 16), replace=False)
        y[k] -= rng.random(k.size) * 1e-3
    else:
        y = np.round(rng.random(L) * 8) / 8  # plateaus
    return np.stack([x, y], 1)


while time.time() < t_end:
    L = int(2 ** rng.integers(9, 14))
    g = int(rng.integers(2, max(3, (1 << 21) // L)))
    f32 = rng.random() < 0.5
    parts = [instance(L, int(rng.integers(5))) for _ in range(g)]
    p = np.concatenate(parts)
    if f32:
        p32 = p.astype(np.float32)
        ok_inc = all(np.all(np.diff(p32[i * L:(i + 1) * L, 0]) > 0) for i in range(g))
        if not ok_inc:
            continue
        p = p32.astype(np.float64)
        t = torch.as_tensor(p32).cuda()
    else:
        t = torch.as_tensor(p).cuda()
    rep = H.build_hood(t, block_len=L)
    c, corners = rep.counts.cpu().numpy(), rep.corners.cpu().numpy().astype(np.float64)
    want, wc = O.block_hulls(p.astype(np.float32) if f32 else p, L)
    want = want.astype(np.float64)
    ok = all(c[i] == wc[i] and np.array_equal(corners[i * L: i * L + c[i]], want[i * L: i * L + wc[i]])
             for i in range(g))
    runs += 1
    if not ok:
        bad += 1
        print(f"MISMATCH L={L} g={g} f32={f32}", flush=True)
print(f"{runs} batched builds, {bad} mismatches")
sys.exit(1 if bad else 0)
