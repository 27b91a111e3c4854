"""Synthetic x-sorted point sets for the five BASELINE.json configs.

Every generator is deterministic in (n, seed) and produces STRICTLY increasing
x (the reference's x_not_increasing precondition, hoodbuf.cpp:51-57; ties make
the reference kernel throw DegenerateTangent).  The recipes are
SURVEY.md section 8(d):

  grid    configs 1/2 -- float2 on the 2^-24 grid: x_i = (i*s + r_i) 2^-24 with
          stride s = 2^24/n and r_i in [1, s); y_i = u_i 2^-24, u_i in [1, 2^24).
          At n = 2^24 (s = 1) x = i 2^-24 for i >= 1 plus x_0 = 2^-25.
          Grid coordinates make the double predicate exact (all differences
          and products fit in 53 bits), so parity is guaranteed, not probable.
  arc     config 3 -- double2 concave arc x = (i + 0.5)/n, y = 0.25 + x(1 - x):
          every point is a corner.
  gauss   config 4 -- double2, x ~ N(0.5, 0.125) rejected outside (0,1),
          sorted, ties broken upward with nextafter; y ~ N(0.5, 0.125).
  batched config 5 -- `instances` x `block` float2 points; inside an instance
          x = (i*2^14 + r) 2^-24 (block=1024), y on the float grid.

numpy versions run anywhere (tests, CPU baseline); the torch versions build the
same recipes directly in HBM for the large configs (device RNG streams differ
from numpy's, so a device-built set is checked against the oracle on its own
copy, never against a numpy-built one).
"""
from __future__ import annotations

import numpy as np

TWO24 = float(1 << 24)


def _grid_x_offsets(n: int, rng: np.random.Generator) -> np.ndarray:
    if n > (1 << 24):
        raise ValueError("float grid holds at most 2^24 strictly increasing x")
    s = (1 << 24) // n
    i = np.arange(n, dtype=np.int64)
    if s >= 2:
        r = rng.integers(1, s, size=n, dtype=np.int64)
        k = i * s + r
        return k.astype(np.float64) / TWO24
    x = i.astype(np.float64) / TWO24
    x[0] = 0.5 / TWO24
    return x


def grid_uniform(n: int, seed: int = 1) -> np.ndarray:
    """Configs 1 and 2: (n, 2) float32, exact on the 2^-24 grid."""
    rng = np.random.default_rng(seed)
    x = _grid_x_offsets(n, rng)
    y = rng.integers(1, 1 << 24, size=n, dtype=np.int64).astype(np.float64) / TWO24
    return np.stack([x, y], axis=1).astype(np.float32)


def arc(n: int) -> np.ndarray:
    """Config 3: (n, 2) float64 concave arc; every point is a hull corner."""
    x = (np.arange(n, dtype=np.float64) + 0.5) / float(n)
    y = 0.25 + x * (1.0 - x)
    return np.stack([x, y], axis=1)


def _fix_ties_np(x: np.ndarray) -> np.ndarray:
    while True:
        bad = np.nonzero(x[1:] <= x[:-1])[0]
        if bad.size == 0:
            return x
        x[bad + 1] = np.nextafter(x[bad], np.inf)


def gauss(n: int, seed: int = 4) -> np.ndarray:
    """Config 4: (n, 2) float64 Gaussian, x sorted strictly increasing."""
    rng = np.random.default_rng(seed)
    xs = np.empty(0)
    while xs.size < n:
        c = rng.normal(0.5, 0.125, size=int((n - xs.size) * 1.01) + 16)
        xs = np.concatenate([xs, c[(c > 0.0) & (c < 1.0)]])
    x = np.sort(xs[:n])
    x = _fix_ties_np(x)
    y = rng.normal(0.5, 0.125, size=n)
    return np.stack([x, y], axis=1)


def batched(instances: int, block: int = 1024, seed: int = 5) -> np.ndarray:
    """Config 5: (instances*block, 2) float32; each block is x-sorted on its own."""
    rng = np.random.default_rng(seed)
    s = (1 << 24) // block
    i = np.tile(np.arange(block, dtype=np.int64), instances)
    r = rng.integers(1, s, size=instances * block, dtype=np.int64)
    x = (i * s + r).astype(np.float64) / TWO24
    y = rng.integers(1, 1 << 24, size=instances * block, dtype=np.int64).astype(np.float64) / TWO24
    return np.stack([x, y], axis=1).astype(np.float32)


def lattice(n: int, span: int, seed: int = 0) -> np.ndarray:
    """Degenerate-heavy test set: strictly increasing x and y on a coarse
    integer lattice (many exactly collinear triples, exact predicates)."""
    rng = np.random.default_rng(seed)
    step = max(span // max(n, 1), 1)
    x = np.cumsum(rng.integers(1, step + 1, size=n)).astype(np.float64)
    y = rng.integers(0, span, size=n).astype(np.float64)
    scale = float(1 << int(np.ceil(np.log2(max(x[-1], span) + 2))))
    return np.stack([x / scale, y / scale], axis=1)


# ------------------------------------------------------------ torch (HBM)

def grid_uniform_torch(n: int, seed: int = 1, device="cuda"):
    import torch
    if n > (1 << 24):
        raise ValueError("float grid holds at most 2^24 strictly increasing x")
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    s = (1 << 24) // n
    i = torch.arange(n, device=device, dtype=torch.int64)
    if s >= 2:
        r = torch.randint(1, s, (n,), device=device, generator=g, dtype=torch.int64)
        x = (i * s + r).to(torch.float64) / TWO24
    else:
        x = i.to(torch.float64) / TWO24
        x[0] = 0.5 / TWO24
    y = torch.randint(1, 1 << 24, (n,), device=device, generator=g, dtype=torch.int64).to(torch.float64) / TWO24
    return torch.stack([x, y], dim=1).to(torch.float32).contiguous()


def arc_torch(n: int, device="cuda"):
    import torch
    x = (torch.arange(n, device=device, dtype=torch.float64) + 0.5) / float(n)
    y = 0.25 + x * (1.0 - x)
    return torch.stack([x, y], dim=1).contiguous()


def gauss_torch(n: int, seed: int = 4, device="cuda"):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    parts, have = [], 0
    while have < n:
        c = torch.randn(int((n - have) * 1.01) + 16, device=device, generator=g, dtype=torch.float64) * 0.125 + 0.5
        c = c[(c > 0.0) & (c < 1.0)]
        parts.append(c)
        have += c.numel()
    x = torch.cat(parts)[:n]
    x, _ = torch.sort(x)
    while True:
        bad = torch.nonzero(x[1:] <= x[:-1]).flatten()
        if bad.numel() == 0:
            break
        x[bad + 1] = torch.nextafter(x[bad], torch.full_like(x[bad], float("inf")))
    y = torch.randn(n, device=device, generator=g, dtype=torch.float64) * 0.125 + 0.5
    return torch.stack([x, y], dim=1).contiguous()


def batched_torch(instances: int, block: int = 1024, seed: int = 5, device="cuda"):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    s = (1 << 24) // block
    m = instances * block
    i = torch.arange(block, device=device, dtype=torch.int64).repeat(instances)
    r = torch.randint(1, s, (m,), device=device, generator=g, dtype=torch.int64)
    x = (i * s + r).to(torch.float64) / TWO24
    y = torch.randint(1, 1 << 24, (m,), device=device, generator=g, dtype=torch.int64).to(torch.float64) / TWO24
    return torch.stack([x, y], dim=1).to(torch.float32).contiguous()
