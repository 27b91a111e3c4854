"""Mismatch census of the GPU hood against oracle::upper_hull on adversarial
near-degenerate sets (tests/adversarial.py), many seeds: which shapes and
storages still differ.  python tools/adv_sweep.py [seeds]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import adversarial as A  # noqa: E402
import oracle as O  # noqa: E402
from paper_1203_5004_b200 import hood as H  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ref = O.ref_upper_hull if O.ref_available() else O.upper_hull
tot = bad = 0
for n in (1 << 10, 1 << 14, 1 << 18, 1 << 20):
    for sh in (0.0, -1.5, 1.5, 1e6):
        nb = 0
        for s in range(seeds):
            p = A.ulp_clusters(n, seed=1000 * s + n % 977 + int(sh) % 13, shift=sh, clusters=256)
            want = ref(p)
            got = H.build_hood(torch.as_tensor(p).cuda()).hull.cpu().numpy()
            ok = got.shape == want.shape and np.array_equal(got, want)
            if not ok:
                nb += 1
                if nb <= 2:
                    gs = {tuple(r) for r in got}
                    ws = {tuple(r) for r in want}
                    print(f"   n={n} shift={sh} seed={s}: gpu-only {sorted(gs - ws)[:4]} ref-only {sorted(ws - gs)[:4]}")
            tot += 1
        bad += nb
        print(f"n={n} shift={sh}: {nb}/{seeds} mismatches", flush=True)
print(f"total {bad}/{tot}")

# batched instances (the unit-end warp hull of the LEAN ring kernel)
for L in (1024, 1 << 16):
    inst = 64 if L == 1024 else 8
    nb = 0
    for s in range(max(1, seeds // 4)):
        parts = []
        for i in range(inst):
            q = A.ulp_clusters(L - 5 * 40, seed=1000 + i + 97 * s, clusters=40, shift=(-1.5, 0.0, 1.5)[i % 3])[:L]
            while q.shape[0] < L:
                q = np.concatenate([q, [[np.nextafter(q[-1, 0], 2.0), q[:, 1].min() - 1.0]]])
            parts.append(q)
        p = np.concatenate(parts)
        rep = H.build_hood(torch.as_tensor(p).cuda(), block_len=L)
        c, corners = rep.counts.cpu().numpy(), rep.corners.cpu().numpy()
        for i in range(inst):
            got, want = corners[i * L: i * L + c[i]], ref(parts[i])
            if not (got.shape == want.shape and np.array_equal(got, want)):
                nb += 1
                if nb <= 2:
                    gs, ws = {tuple(r) for r in got}, {tuple(r) for r in want}
                    print(f"   L={L} s={s} inst={i}: gpu-only {sorted(gs - ws)[:4]} ref-only {sorted(ws - gs)[:4]}")
    print(f"batched L={L}: {nb} mismatching instances", flush=True)
