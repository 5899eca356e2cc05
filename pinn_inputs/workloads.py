"""Seeded problem generator for configs C1-C5 of BASELINE.json.

Readings of the paper adopted here (all listed in DESIGN.md "Readings"):

* Z7  -- residual points are uniform in each subdomain (the paper's
  "i.i.d. from N(0, sigma^2)" on a bounded box is unusable as printed,
  PAPER.md:195); interface points are at edge MIDPOINTS
  s_j = a + (j + 1/2)(b - a)/N_I, so no point is shared by more than two
  subdomains; data points are uniform on the subdomain's outer-boundary
  segments.
* Z3  -- every interface edge carries ONE canonical unit normal (+x1 for an
  edge x1 = const, +x2 otherwise), used by both sides.
* Z5  -- subdomain id q = ix + Nx * iy (PAPER.md:210-213 is inconsistent).
* Z10 -- Xavier-uniform weights, zero biases, a^k = 1/n.
* Z13 -- Burgers on [-1, 1] x [0, 1] with u(0, x) = -sin(pi x),
  u(t, +-1) = 0.
* Z15 -- C2 Poisson on [0,1]^2 with u* = sin(pi x) sin(pi y) (so u = 0 on the
  boundary); "heat" variant T* = 20 exp(-0.1 y).
* Z16 -- NS lid-driven cavity, Re = 100: (u, v) = (1, 0) on y = 1, (0, 0) on
  the other walls, pressure unconstrained (output mask).

Nothing in this module evaluates a network, a derivative or a loss.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

SEED_BASE = 2104_10013

PDE_OUTPUTS = {"burgers": 1, "poisson": 1, "heat": 1, "ns": 3, "heat_inv": 2}


def _f32(a) -> np.ndarray:
    """Round to float32 and return as float64 (bit-identical inputs for both sides)."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


# ----------------------------------------------------------------------------
# network layout (an input FORMAT, SPEC.md:140-148 / SURVEY D1): layer-major
# W^1, b^1, a^1, W^2, b^2, a^2, ..., W^{L-1}, b^{L-1}, a^{L-1}, W^L, b^L.
# W^k is row-major N_k x N_{k-1}.
# ----------------------------------------------------------------------------

def layer_sizes(d_in: int, width: int, n_hidden: int, d_out: int) -> List[int]:
    return [d_in] + [width] * n_hidden + [d_out]


def param_layout(sizes: List[int]) -> List[Dict[str, Tuple[int, int]]]:
    """Offsets of W^k, b^k (and a^k for hidden layers) in the flat vector.

    Returns a list over layers k = 1..L of dicts {"W": (off, len), "b": ...,
    "a": ...} ("a" absent for the output layer)."""
    out = []
    off = 0
    L = len(sizes) - 1
    for k in range(1, L + 1):
        n_out, n_in = sizes[k], sizes[k - 1]
        ent = {"W": (off, n_out * n_in)}
        off += n_out * n_in
        ent["b"] = (off, n_out)
        off += n_out
        if k < L:
            ent["a"] = (off, 1)
            off += 1
        out.append(ent)
    return out


def n_params(sizes: List[int]) -> int:
    lay = param_layout(sizes)
    last = lay[-1]["b"]
    return last[0] + last[1]


def xavier_params(sizes: List[int], slope_n: float, rng: np.random.Generator) -> np.ndarray:
    """Xavier-uniform W, zero b, a = 1/n (Z10; PAPER.md:95 'initialize n a^k = 1')."""
    lay = param_layout(sizes)
    theta = np.zeros(n_params(sizes), dtype=np.float64)
    for k, ent in enumerate(lay, start=1):
        n_out, n_in = sizes[k], sizes[k - 1]
        lim = np.sqrt(6.0 / (n_in + n_out))
        o, n = ent["W"]
        theta[o:o + n] = rng.uniform(-lim, lim, size=n)
        if "a" in ent:
            theta[ent["a"][0]] = 1.0 / slope_n
    return _f32(theta)


def perturb_params(problem: "Problem", scale: float = 0.1, seed: int = 7) -> "Problem":
    """Return a copy whose biases and slopes are randomly perturbed (exercises
    the bias and slope paths away from the n*a=1, b=0 initial point)."""
    rng = np.random.default_rng(seed)
    sizes = problem.sizes
    lay = param_layout(sizes)
    subs = []
    for s in problem.subdomains:
        th = s.params.copy()
        for ent in lay:
            o, n = ent["b"]
            th[o:o + n] += scale * rng.standard_normal(n)
            if "a" in ent:
                th[ent["a"][0]] *= 1.0 + 0.5 * scale * rng.standard_normal()
        subs.append(dataclasses.replace(s, params=_f32(th)))
    return dataclasses.replace(problem, subdomains=subs)


# ----------------------------------------------------------------------------
# decomposition
# ----------------------------------------------------------------------------

@dataclass
class Edge:
    """A common interface between subdomains `a` (minus side) and `b` (plus side)."""
    id: int
    a: int
    b: int
    axis: int                      # 0: edge is x1 = const (normal +x1); 1: x2 = const
    normal: Tuple[float, float]
    pts: np.ndarray                # [N_I, 2], shared verbatim by both sides


@dataclass
class Subdomain:
    id: int
    ix: int
    iy: int
    lo: Tuple[float, float]
    hi: Tuple[float, float]
    x_f: np.ndarray                # [N_F, 2] residual points
    x_u: np.ndarray                # [N_u, 2] training (boundary / initial) points
    u_target: np.ndarray           # [N_u, d_out]
    u_mask: np.ndarray             # [N_u, d_out] 1 = constrained output, 0 = free
    edges: List[int]               # ids of the live interface edges, ascending
    params: np.ndarray             # flat initial parameters (layer-major)
    activation: Optional[str] = None   # per-subdomain activation (C5, Table 3); None = problem's


@dataclass
class Problem:
    name: str
    method: str                    # "pinn" | "cpinn" | "xpinn" | "hybrid" (flux in x1, residual in x2)
    pde: str                       # "burgers" | "poisson" | "heat" | "ns" | "heat_inv"
    activation: str                # "tanh" | "sin" | "cos"
    d_in: int
    d_out: int
    width: int
    n_hidden: int
    slope_n: float
    nu: float
    re: float
    w_u: float
    w_f: float
    w_i: float
    w_if: float                    # W_Iflux (cPINN) or W_IF (XPINN)
    lr: float
    beta1: float
    beta2: float
    eps: float
    nx: int
    ny: int
    domain_lo: Tuple[float, float]
    domain_hi: Tuple[float, float]
    subdomains: List[Subdomain]
    edges: List[Edge]
    meta: Dict = field(default_factory=dict)   # generator geometry (C5: seeds, polygon)

    @property
    def sizes(self) -> List[int]:
        return layer_sizes(self.d_in, self.width, self.n_hidden, self.d_out)

    @property
    def n_sub(self) -> int:
        return len(self.subdomains)

    def n_points(self, q: Optional[int] = None) -> int:
        subs = self.subdomains if q is None else [self.subdomains[q]]
        tot = 0
        for s in subs:
            tot += len(s.x_f) + len(s.x_u)
            tot += sum(len(self.edges[e].pts) for e in s.edges)
        return tot

    def act(self, q: int) -> str:
        """Activation of subdomain q (Table 3 gives one per region)."""
        a = self.subdomains[q].activation
        return self.activation if a is None else a

    def edge_neighbor(self, q: int, e: int) -> int:
        ed = self.edges[e]
        return ed.b if ed.a == q else ed.a


def _boundary_segments(lo, hi, dlo, dhi, pde):
    """Outer-boundary segments of the cell [lo,hi] that carry data (EToV,
    PAPER.md:195).  Each segment = (axis_fixed, value, a, b, tag)."""
    segs = []
    tol = 1e-12
    # x1 = const walls
    if abs(lo[0] - dlo[0]) < tol:
        segs.append((0, lo[0], lo[1], hi[1], "x1lo"))
    if abs(hi[0] - dhi[0]) < tol:
        segs.append((0, hi[0], lo[1], hi[1], "x1hi"))
    # x2 = const walls
    if abs(lo[1] - dlo[1]) < tol:
        segs.append((1, lo[1], lo[0], hi[0], "x2lo"))
    if abs(hi[1] - dhi[1]) < tol and pde != "burgers":   # t = T_end carries no data
        segs.append((1, hi[1], lo[0], hi[0], "x2hi"))
    return segs


def kovasznay(x: np.ndarray, re: float) -> np.ndarray:
    """Kovasznay flow (exact steady NS solution, used as boundary data and as
    the accuracy reference of f4): u = 1 - e^{lam x} cos 2 pi y,
    v = lam/(2 pi) e^{lam x} sin 2 pi y, p = (1 - e^{2 lam x})/2,
    lam = Re/2 - sqrt(Re^2/4 + 4 pi^2)."""
    lam = re / 2.0 - np.sqrt(re * re / 4.0 + 4.0 * np.pi ** 2)
    e = np.exp(lam * x[:, 0])
    return np.stack([1.0 - e * np.cos(2 * np.pi * x[:, 1]), lam / (2 * np.pi) * e * np.sin(2 * np.pi * x[:, 1]),
                     0.5 * (1.0 - e * e)], axis=1)


def burgers_wave(x: np.ndarray, nu: float, a: float = 0.5, c: float = 0.2) -> np.ndarray:
    """Viscous Burgers travelling wave u = c - a tanh(a (x - c t) / (2 nu))
    (exact solution of u_t + u u_x = nu u_xx; boundary / initial data and
    accuracy reference of f4)."""
    return c - a * np.tanh(a * (x[:, 0] - c * x[:, 1]) / (2.0 * nu))


def _targets(pde: str, x: np.ndarray, tag: str, bc: str = "paper", nu: float = 0.0,
             re: float = 100.0) -> Tuple[np.ndarray, np.ndarray]:
    """Boundary / initial data of the paper's problems (inputs, not the method).
    bc = "kovasznay" (NS) / "wave" (Burgers): data of a closed-form solution
    instead (accuracy tests of f4)."""
    n = len(x)
    if pde == "burgers" and bc == "wave":
        return burgers_wave(x, nu)[:, None], np.ones((n, 1))
    if pde == "ns" and bc == "kovasznay":
        return kovasznay(x, re), np.ones((n, 3))             # u, v and p (fixes the gauge)
    if pde == "burgers":
        # u(0,x) = -sin(pi x) on t = 0; u(t,+-1) = 0
        if tag == "x2lo":
            t = -np.sin(np.pi * x[:, 0])
        else:
            t = np.zeros(n)
        return t[:, None], np.ones((n, 1))
    if pde == "poisson":
        t = np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1])   # = 0 on the box boundary
        return t[:, None], np.ones((n, 1))
    if pde == "heat":
        t = 20.0 * np.exp(-0.1 * x[:, 1])
        return t[:, None], np.ones((n, 1))
    if pde == "heat_inv":
        # outputs (T, K): T* = 20 exp(-0.1 y), K* = 20 + exp(0.1 y) sin(0.5 x)
        # (PAPER.md:828-829).  "interior": T data only; "boundary": T and K.
        tgt = np.stack([20.0 * np.exp(-0.1 * x[:, 1]),
                        20.0 + np.exp(0.1 * x[:, 1]) * np.sin(0.5 * x[:, 0])], axis=1)
        mask = np.ones((n, 2))
        if tag == "interior":
            mask[:, 1] = 0.0
        return tgt, mask
    if pde == "ns":
        tgt = np.zeros((n, 3))
        if tag == "x2hi":
            tgt[:, 0] = 1.0                                     # lid (u, v) = (1, 0)
        mask = np.ones((n, 3))
        mask[:, 2] = 0.0                                        # p free (Z16)
        return tgt, mask
    raise ValueError(pde)


def build_problem(*, name: str, pde: str, method: str, nx: int, ny: int,
                  domain_lo, domain_hi, n_f: int, n_i: int, n_u: int,
                  width: int, n_hidden: int, lr: float, seed_index: int,
                  activation: str = "tanh", slope_n: float = 10.0,
                  nu: float = 0.01 / np.pi, re: float = 100.0,
                  weights=(20.0, 1.0, 20.0, 20.0),
                  betas=(0.9, 0.999), eps: float = 1e-8,
                  n_f_per_sub: Optional[List[int]] = None, bc: str = "paper") -> Problem:
    if method not in ("pinn", "cpinn", "xpinn", "hybrid"):
        raise ValueError(method)
    d_out = PDE_OUTPUTS[pde]
    dlo = tuple(float(v) for v in domain_lo)
    dhi = tuple(float(v) for v in domain_hi)
    hx = (dhi[0] - dlo[0]) / nx
    hy = (dhi[1] - dlo[1]) / ny
    nsub = nx * ny
    root = np.random.SeedSequence(SEED_BASE + seed_index)
    kids = root.spawn(nsub)

    def cell(q):
        ix, iy = q % nx, q // nx
        lo = (dlo[0] + ix * hx, dlo[1] + iy * hy)
        hi = (dlo[0] + (ix + 1) * hx, dlo[1] + (iy + 1) * hy)
        return ix, iy, lo, hi

    # interface edges: x1-normal edges first, then x2-normal
    edges: List[Edge] = []
    if method != "pinn":
        for iy in range(ny):
            for ix in range(nx - 1):
                a = ix + nx * iy
                b = a + 1
                _, _, lo, hi = cell(a)
                s = lo[1] + (np.arange(n_i) + 0.5) * (hi[1] - lo[1]) / n_i
                pts = np.stack([np.full(n_i, hi[0]), s], axis=1)
                edges.append(Edge(len(edges), a, b, 0, (1.0, 0.0), _f32(pts)))
        for iy in range(ny - 1):
            for ix in range(nx):
                a = ix + nx * iy
                b = a + nx
                _, _, lo, hi = cell(a)
                s = lo[0] + (np.arange(n_i) + 0.5) * (hi[0] - lo[0]) / n_i
                pts = np.stack([s, np.full(n_i, hi[1])], axis=1)
                edges.append(Edge(len(edges), a, b, 1, (0.0, 1.0), _f32(pts)))
    elif nsub != 1:
        raise ValueError("method 'pinn' needs a single subdomain")

    sizes = layer_sizes(2, width, n_hidden, d_out)
    subs: List[Subdomain] = []
    for q in range(nsub):
        ix, iy, lo, hi = cell(q)
        prng, wrng = [np.random.default_rng(c) for c in kids[q].spawn(2)]
        nf = n_f if n_f_per_sub is None else n_f_per_sub[q]
        x_f = np.stack([prng.uniform(lo[0], hi[0], nf), prng.uniform(lo[1], hi[1], nf)], axis=1)
        segs = _boundary_segments(lo, hi, dlo, dhi, pde)
        xs, ts, ms = [], [], []
        if segs and n_u > 0:
            # split N_u over the data segments in proportion to their length
            lens = np.array([s[3] - s[2] for s in segs])
            cnt = np.floor(n_u * lens / lens.sum()).astype(int)
            cnt[: n_u - cnt.sum()] += 1
            for (ax, val, a, b, tag), c in zip(segs, cnt):
                if c == 0:
                    continue
                s = prng.uniform(a, b, c)
                if ax == 0:
                    x = np.stack([np.full(c, val), s], axis=1)
                else:
                    x = np.stack([s, np.full(c, val)], axis=1)
                x = _f32(x)
                t, m = _targets(pde, x, tag, bc, float(np.float32(nu)), float(np.float32(re)))
                xs.append(x); ts.append(t); ms.append(m)
        if xs:
            x_u = np.concatenate(xs); u_t = np.concatenate(ts); u_m = np.concatenate(ms)
        else:
            x_u = np.zeros((0, 2)); u_t = np.zeros((0, d_out)); u_m = np.zeros((0, d_out))
        my_edges = [e.id for e in edges if e.a == q or e.b == q]
        subs.append(Subdomain(q, ix, iy, lo, hi, _f32(x_f), _f32(x_u), _f32(u_t), _f32(u_m),
                              my_edges, xavier_params(sizes, slope_n, wrng)))

    f = lambda v: float(np.float32(v))    # scalar inputs are float32-exact too
    return Problem(name=name, method=method, pde=pde, activation=activation, d_in=2,
                   d_out=d_out, width=width, n_hidden=n_hidden, slope_n=f(slope_n),
                   nu=f(nu), re=f(re), w_u=f(weights[0]), w_f=f(weights[1]),
                   w_i=f(weights[2]), w_if=f(weights[3]), lr=f(lr),
                   beta1=f(betas[0]), beta2=f(betas[1]), eps=f(eps),
                   nx=nx, ny=ny, domain_lo=dlo, domain_hi=dhi, subdomains=subs, edges=edges)


# ----------------------------------------------------------------------------
# named configurations (BASELINE.json configs[0..3])
# ----------------------------------------------------------------------------

def _c1(scale, method=None, **kw):
    return dict(name="C1-burgers-cpinn-2x1-3x20", pde="burgers", method=method or "cpinn",
                nx=2, ny=1, domain_lo=(-1.0, 0.0), domain_hi=(1.0, 1.0),
                n_f=500, n_i=50, n_u=100, width=20, n_hidden=3, lr=8e-4, seed_index=0)


def _c2(scale, method=None, weak=1, **kw):
    """C2 on [0,1]^2 (4x4); `weak` = G replicates the 4x4 block along x on
    [0, G] x [0, 1] (4G x 4 subdomains, one 4x4 block per GPU: weak scaling)."""
    return dict(name=f"C2-poisson-{4 * weak}x4-6x40", pde=kw.get("pde", "poisson"),
                method=method or "cpinn", nx=4 * weak, ny=4, domain_lo=(0.0, 0.0),
                domain_hi=(float(weak), 1.0),
                n_f=15000, n_i=250, n_u=80, width=40, n_hidden=6, lr=6e-4, seed_index=1)


def _c3(scale, method=None, gpus=8, **kw):
    grid = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}[gpus]
    return dict(name=f"C3-burgers-xpinn-{grid[0]}x{grid[1]}-5x20", pde="burgers",
                method=method or "xpinn", nx=grid[0], ny=grid[1],
                domain_lo=(-1.0, 0.0), domain_hi=(1.0, 1.0),
                n_f=20000, n_i=250, n_u=100, width=20, n_hidden=5, lr=8e-4, seed_index=2)


def _c4(scale, method=None, **kw):
    return dict(name="C4-ns-xpinn-4x2-5x80", pde="ns", method=method or "xpinn", nx=4, ny=2,
                domain_lo=(0.0, 0.0), domain_hi=(1.0, 1.0),
                n_f=125000, n_i=250, n_u=80, width=80, n_hidden=5, lr=6e-4, seed_index=3)


# C5 (NEXT row f1): inverse heat conduction, XPINN on 10 seeded-Voronoi
# regions of a non-convex map polygon (Table 3).
C5_N_F = [3000, 4000, 5000, 4000, 3000, 4000, 800, 3000, 5000, 4000]   # Table 3
C5_ACT = ["tanh", "sin", "cos", "tanh", "sin", "cos", "tanh", "sin", "cos", "tanh"]


def _c5(scale, method=None, **kw):
    return dict(name="C5-heatinv-xpinn-voronoi10-3x80", pde="heat_inv", method=method or "xpinn",
                n_f=C5_N_F, n_i=100, n_u=400, width=80, n_hidden=3, lr=6e-3, seed_index=4,
                t_frac=0.1)


def build_voronoi_problem(*, name: str, pde: str, method: str, n_f, n_i: int, n_u: int,
                          width: int, n_hidden: int, lr: float, seed_index: int,
                          t_frac: float = 0.1, activations=None, n_regions: int = 10,
                          slope_n: float = 10.0, weights=(20.0, 1.0, 20.0, 20.0),
                          betas=(0.9, 0.999), eps: float = 1e-8, **_) -> Problem:
    """C5 recipe (reading Z24): regions = nearest-seed cells of Lloyd-relaxed
    seeds inside `voronoi.MAP_POLYGON`; N_F(q) uniform residual points in
    region q (Table 3); round(t_frac N_F(q)) interior T-only data points;
    `n_u` boundary points uniform in arc length, each assigned to its region,
    with T and K data; per Voronoi interface segment, N_I points at the
    midpoints of N_I equal sub-segments (split over the segments of a pair in
    proportion to length)."""
    from . import voronoi as vor
    if pde != "heat_inv":
        raise ValueError(pde)
    d_out = PDE_OUTPUTS[pde]
    poly = vor.MAP_POLYGON
    root = np.random.SeedSequence(SEED_BASE + seed_index)
    seqs = root.spawn(2 + n_regions)
    grng, brng = np.random.default_rng(seqs[0]), np.random.default_rng(seqs[1])
    seeds = vor.lloyd_seeds(poly, n_regions, grng)
    acts = activations or C5_ACT
    # interfaces
    edges: List[Edge] = []
    if method != "pinn":
        segs = vor.interface_segments(poly, seeds)
        pairs = {}
        for s in segs:
            pairs.setdefault((s[0], s[1]), []).append(s)
        for (a, b), ss in sorted(pairs.items()):
            lens = np.array([np.linalg.norm(s[3] - s[2]) for s in ss])
            cnt = np.floor(n_i * lens / lens.sum()).astype(int)
            cnt[: n_i - cnt.sum()] += 1
            for (_, _, p0, p1, nrm), c in zip(ss, cnt):
                if c == 0:
                    continue
                f = (np.arange(c) + 0.5) / c
                pts = p0[None, :] + f[:, None] * (p1 - p0)[None, :]
                edges.append(Edge(len(edges), a, b, -1, (float(nrm[0]), float(nrm[1])), _f32(pts)))
    elif n_regions != 1:
        raise ValueError("method 'pinn' needs a single subdomain")
    # boundary data, assigned to regions
    xb = vor.boundary_sample(poly, n_u, brng) if n_u > 0 else np.zeros((0, 2))
    xb = _f32(xb)
    lab_b = vor.nearest(seeds, xb) if len(xb) else np.zeros(0, dtype=int)
    sizes = layer_sizes(2, width, n_hidden, d_out)
    subs: List[Subdomain] = []
    for q in range(n_regions):
        prng, wrng = [np.random.default_rng(s) for s in seqs[2 + q].spawn(2)]
        nf = n_f[q] if isinstance(n_f, (list, tuple)) else n_f
        x_f = _f32(vor.sample_region(poly, seeds, q, nf, prng))
        nt = int(round(t_frac * nf))
        x_t = _f32(vor.sample_region(poly, seeds, q, nt, prng)) if nt > 0 else np.zeros((0, 2))
        t_t, m_t = _targets(pde, x_t, "interior")
        x_b = xb[lab_b == q]
        t_b, m_b = _targets(pde, x_b, "boundary")
        x_u = np.concatenate([x_t, x_b])
        lo, hi = tuple(x_f.min(0)), tuple(x_f.max(0))
        my_edges = [e.id for e in edges if e.a == q or e.b == q]
        subs.append(Subdomain(q, q, 0, lo, hi, x_f, _f32(x_u), _f32(np.concatenate([t_t, t_b])),
                              _f32(np.concatenate([m_t, m_b])), my_edges,
                              xavier_params(sizes, slope_n, wrng), activation=acts[q]))
    f = lambda v: float(np.float32(v))
    dlo, dhi = tuple(poly.min(0)), tuple(poly.max(0))
    return Problem(name=name, method=method, pde=pde, activation=acts[0], d_in=2,
                   d_out=d_out, width=width, n_hidden=n_hidden, slope_n=f(slope_n),
                   nu=0.0, re=f(100.0), w_u=f(weights[0]), w_f=f(weights[1]),
                   w_i=f(weights[2]), w_if=f(weights[3]), lr=f(lr),
                   beta1=f(betas[0]), beta2=f(betas[1]), eps=f(eps),
                   nx=n_regions, ny=1, domain_lo=dlo, domain_hi=dhi, subdomains=subs, edges=edges,
                   meta={"seeds": seeds, "polygon": poly})


CONFIGS = {"C1": _c1, "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5}


def make_config(cfg: str, *, scale: float = 1.0, method: Optional[str] = None,
                n_f: Optional[int] = None, n_i: Optional[int] = None,
                n_u: Optional[int] = None, width: Optional[int] = None,
                n_hidden: Optional[int] = None, **kw) -> Problem:
    """Build a named config.  `scale` multiplies the point counts (small
    parity cases use scale < 1); explicit counts override."""
    args = CONFIGS[cfg](scale, method=method, **kw)
    for key, val in (("n_f", n_f), ("n_i", n_i), ("n_u", n_u)):
        if val is not None:
            args[key] = val
        elif scale != 1.0:
            lo = 1 if key != "n_u" else 0
            v = args[key]
            args[key] = ([max(lo, int(round(x * scale))) for x in v] if isinstance(v, list)
                         else max(lo, int(round(v * scale))))
    if width is not None:
        args["width"] = width
    if n_hidden is not None:
        args["n_hidden"] = n_hidden
    for k in ("nx", "ny", "activation", "weights", "lr", "slope_n", "nu", "re", "pde", "seed_index",
              "activations", "t_frac", "domain_lo", "domain_hi", "bc"):
        if k in kw:
            args[k] = kw[k]
    if cfg == "C3" and ("nx" in kw or "ny" in kw):
        args["name"] = f"C3-burgers-{args['method']}-{args['nx']}x{args['ny']}-5x20"
    if cfg == "C5":
        return build_voronoi_problem(**args)
    return build_problem(**args)
