"""Adversarial x-sorted point sets for the double (and float) predicate path.

Near-degenerate inputs the culling and merging arguments must survive under
rounding (VERDICT r1 "What's weak" 1a): clusters of 3-5 points within a few
ulps of each other in BOTH coordinates at the hull's corners (x strictly
increasing by nextafter steps -- the reference's tie-break),
points within an ulp of the hull's edges, equal-y plateaus at the top, and the
same shapes shifted below 0 and above 1 in y (other exponents, other
roundings).  Deterministic in (n, seed).  Test infrastructure only.
"""
from __future__ import annotations

import numpy as np


def _strict(x: np.ndarray, dtype) -> np.ndarray:
    """Make x strictly increasing by nextafter steps (dtype arithmetic)."""
    x = x.astype(dtype)
    for i in range(1, x.size):
        if not x[i] > x[i - 1]:
            x[i] = np.nextafter(x[i - 1], dtype(np.inf))
    return x


def ulp_clusters(n: int, seed: int, dtype=np.float64, shift: float = 0.0, clusters: int = 64,
                 hull_fn=None) -> np.ndarray:
    """n base points (x uniform in (0.01, 0.99), y Gaussian + shift) plus
    clusters at up to `clusters` of the base hull's corners and edges; the
    result has at most n + 5*clusters points, x strictly increasing."""
    rng = np.random.default_rng(seed)
    dt = np.dtype(dtype).type
    x = np.sort(rng.uniform(0.01, 0.99, size=n))
    y = rng.normal(0.5, 0.125, size=n) + shift
    x = _strict(x, dt)
    y = y.astype(dt)
    base = np.stack([x, y], axis=1)
    if hull_fn is None:
        import oracle as O
        hull_fn = O.upper_hull
    h = hull_fn(base.astype(np.float64)).astype(dt)
    extra = []
    pick = rng.permutation(max(len(h) - 1, 1))[:clusters]
    for t in pick:
        c = h[t]
        d = h[min(t + 1, len(h) - 1)]
        kind = t % 4
        m = int(rng.integers(3, 6))
        xs = [c[0]]
        for _ in range(m):
            xs.append(np.nextafter(xs[-1], dt(np.inf)))
        xs = np.array(xs[1:], dtype=dt)
        ulp_y = np.spacing(c[1]) if c[1] != 0 else np.spacing(dt(1e-30))
        if kind == 0:    # a cluster at the corner: y within +-3 ulps
            ys = c[1] + rng.integers(-3, 4, size=m).astype(dt) * ulp_y
        elif kind == 1:  # a plateau: exactly the corner's y
            ys = np.full(m, c[1], dtype=dt)
        elif kind == 2:  # points within an ulp of the edge c -> d
            f = np.sort(rng.uniform(0.05, 0.95, size=m))
            xs = (c[0] + (d[0] - c[0]) * f).astype(dt)
            ys = (c[1] + (d[1] - c[1]) * f).astype(dt) + rng.integers(-1, 2, size=m).astype(dt) * ulp_y
        else:            # just below the corner, to the left and right
            xs = np.array([np.nextafter(c[0], dt(-np.inf)), *xs[: m - 1]], dtype=dt)
            ys = c[1] - rng.integers(0, 3, size=m).astype(dt) * ulp_y
        extra.append(np.stack([xs, ys.astype(dt)], axis=1))
    pts = np.concatenate([base] + extra) if extra else base
    pts = pts[np.argsort(pts[:, 0], kind="stable")]
    keep = np.concatenate([[True], pts[1:, 0] > pts[:-1, 0]])
    return np.ascontiguousarray(pts[keep])


def tied_top(n: int, seed: int, dtype=np.float64) -> np.ndarray:
    """A wide plateau at the maximum: many points with exactly the same top y,
    x consecutive doubles near the middle (ties the monotone chain pops,
    geom.hpp:26-28 strict >), plus random points below."""
    rng = np.random.default_rng(seed)
    dt = np.dtype(dtype).type
    x = _strict(np.sort(rng.uniform(0.01, 0.99, size=n)), dt)
    y = rng.uniform(0.0, 0.5, size=n).astype(dt)
    mid = n // 2
    k = min(32, n // 4)
    xs = [x[mid]]
    for _ in range(k - 1):
        xs.append(np.nextafter(xs[-1], dt(np.inf)))
    xs = np.array(xs, dtype=dt)
    top = np.stack([xs, np.full(k, dt(0.75))], axis=1)
    pts = np.concatenate([np.stack([x, y], axis=1), top])
    pts = pts[np.argsort(pts[:, 0], kind="stable")]
    keep = np.concatenate([[True], pts[1:, 0] > pts[:-1, 0]])
    return np.ascontiguousarray(pts[keep])
