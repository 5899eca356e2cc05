"""Geometry of config C5: a synthetic non-convex "map" polygon split into
seeded Voronoi regions (Fig. "US map
divided into 10 subdomains" -- the map itself is not provided, so a fixed
polygon of the same character stands in for it, reading Z24 in DESIGN.md).

Pure geometry: point-in-polygon, nearest-seed regions, Lloyd relaxation of
the seeds, and the exact Voronoi interface segments (bisector of two seeds,
clipped by the other seeds' half-planes and by the polygon).  Nothing here
evaluates a network, a derivative or a loss.
"""

from __future__ import annotations

from typing import List, Tuple

import numpy as np

# A simple (non-self-intersecting), non-convex polygon on [0, 10] x [0, 6],
# counter-clockwise, loosely shaped like a continental outline with a
# south-eastern peninsula (the non-convex parts are the notches at the
# north-east and the south).
MAP_POLYGON = np.array([
    (0.3, 2.2), (0.9, 4.6), (0.6, 5.6), (3.2, 5.8), (6.0, 5.5), (7.0, 5.9),
    (7.6, 5.1), (8.4, 5.6), (9.7, 5.7), (9.3, 4.2), (8.2, 3.3), (8.7, 2.0),
    (9.2, 0.2), (8.4, 0.5), (7.6, 1.4), (6.2, 1.0), (5.0, 0.1), (4.1, 1.1),
    (2.3, 1.2), (1.2, 0.7),
][::-1], dtype=np.float64)


def polygon_area(poly: np.ndarray) -> float:
    x, y = poly[:, 0], poly[:, 1]
    return 0.5 * float(np.dot(x, np.roll(y, -1)) - np.dot(np.roll(x, -1), y))


def inside(poly: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """Even-odd ray casting; pts [n, 2] -> bool [n]."""
    x, y = pts[:, 0][:, None], pts[:, 1][:, None]
    x0, y0 = poly[:, 0][None, :], poly[:, 1][None, :]
    x1, y1 = np.roll(poly[:, 0], -1)[None, :], np.roll(poly[:, 1], -1)[None, :]
    crosses = (y0 > y) != (y1 > y)
    with np.errstate(divide="ignore", invalid="ignore"):
        xint = x0 + (y - y0) * (x1 - x0) / (y1 - y0)
    return (np.count_nonzero(crosses & (x < xint), axis=1) % 2) == 1


def nearest(seeds: np.ndarray, pts: np.ndarray) -> np.ndarray:
    d2 = ((pts[:, None, :] - seeds[None, :, :]) ** 2).sum(-1)
    return np.argmin(d2, axis=1)


def sample_region(poly, seeds, q, n, rng, batch=4096) -> np.ndarray:
    """n points uniform in region q = {x in polygon : nearest seed is q}."""
    lo, hi = poly.min(0), poly.max(0)
    out = []
    got = 0
    while got < n:
        c = rng.uniform(lo, hi, size=(batch, 2))
        c = c[inside(poly, c)]
        c = c[nearest(seeds, c) == q]
        out.append(c)
        got += len(c)
    return np.concatenate(out)[:n]


def lloyd_seeds(poly, n_regions, rng, iters=12, n_sample=40000) -> np.ndarray:
    """Seeds of a near-centroidal Voronoi partition (well-shaped regions):
    random interior start, then Lloyd steps on a fixed interior sample."""
    lo, hi = poly.min(0), poly.max(0)
    s = rng.uniform(lo, hi, size=(4 * n_sample, 2))
    s = s[inside(poly, s)][:n_sample]
    seeds = s[rng.choice(len(s), n_regions, replace=False)].copy()
    for _ in range(iters):
        lab = nearest(seeds, s)
        for q in range(n_regions):
            m = lab == q
            if m.any():
                seeds[q] = s[m].mean(0)
    # canonical order: west to east (then south to north)
    order = np.lexsort((seeds[:, 1], seeds[:, 0]))
    return seeds[order]


def _line_polygon_params(poly, m, d) -> np.ndarray:
    """Parameters t where the line m + t d crosses a polygon edge."""
    ts = []
    n = len(poly)
    for i in range(n):
        a, b = poly[i], poly[(i + 1) % n]
        e = b - a
        den = d[0] * (-e[1]) - d[1] * (-e[0])
        if abs(den) < 1e-14:
            continue
        r = a - m
        t = (r[0] * (-e[1]) - r[1] * (-e[0])) / den
        u = (d[0] * r[1] - d[1] * r[0]) / den
        if -1e-12 <= u <= 1 + 1e-12:
            ts.append(t)
    return np.array(sorted(ts))


def interface_segments(poly, seeds) -> List[Tuple[int, int, np.ndarray, np.ndarray, np.ndarray]]:
    """Exact Voronoi interfaces inside the polygon.

    Returns [(a, b, P0, P1, normal)] with a < b: the straight segment P0-P1 on
    the bisector of seeds a and b, where both are nearer than every other seed
    and which lies inside the polygon (a bisector clipped by a non-convex
    polygon may give several segments).  normal = (p_b - p_a)/|p_b - p_a|, the
    edge's canonical unit normal (reading Z3)."""
    out = []
    ns = len(seeds)
    span = float(np.linalg.norm(poly.max(0) - poly.min(0)))
    for a in range(ns):
        for b in range(a + 1, ns):
            pa, pb = seeds[a], seeds[b]
            nrm = (pb - pa) / np.linalg.norm(pb - pa)
            d = np.array([-nrm[1], nrm[0]])
            m = 0.5 * (pa + pb)
            t0, t1 = -span, span
            for s in range(ns):
                if s in (a, b):
                    continue
                ps = seeds[s]
                g = 2.0 * np.dot(d, ps - pa)
                h = np.dot(ps, ps) - np.dot(pa, pa) - 2.0 * np.dot(m, ps - pa)
                if abs(g) < 1e-14:
                    if h < 0:
                        t0, t1 = 1.0, 0.0
                    continue
                if g > 0:
                    t1 = min(t1, h / g)
                else:
                    t0 = max(t0, h / g)
            if t1 - t0 <= 1e-9:
                continue
            cuts = _line_polygon_params(poly, m, d)
            br = np.concatenate([[t0], cuts[(cuts > t0) & (cuts < t1)], [t1]])
            for u0, u1 in zip(br[:-1], br[1:]):
                if u1 - u0 < 1e-6:
                    continue
                mid = m + 0.5 * (u0 + u1) * d
                if inside(poly, mid[None, :])[0]:
                    out.append((a, b, m + u0 * d, m + u1 * d, nrm))
    return out


def boundary_sample(poly, n, rng) -> np.ndarray:
    """n points uniform in arc length on the polygon boundary."""
    e = np.roll(poly, -1, axis=0) - poly
    L = np.linalg.norm(e, axis=1)
    cum = np.concatenate([[0.0], np.cumsum(L)])
    s = rng.uniform(0.0, cum[-1], n)
    i = np.clip(np.searchsorted(cum, s, side="right") - 1, 0, len(poly) - 1)
    f = (s - cum[i]) / L[i]
    return poly[i] + f[:, None] * e[i]
