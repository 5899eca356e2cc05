"""Input generator (pre-processing stage)."""

import numpy as np
import pytest

from pinn_inputs import make_config, build_problem


def test_grid_edges_and_neighbours():
    # SPEC.md:487-489 / PAPER Fig. 3: a 4x3 grid has 17 interior edges; corner
    # subdomains have 2 live edges, interior ones 4.
    p = build_problem(name="t", pde="poisson", method="xpinn", nx=4, ny=3,
                      domain_lo=(0, 0), domain_hi=(1, 1), n_f=4, n_i=3, n_u=4,
                      width=3, n_hidden=1, lr=1e-3, seed_index=9)
    assert len(p.edges) == 17
    deg = [len(s.edges) for s in p.subdomains]
    assert deg[0] == 2 and deg[3] == 2 and deg[8] == 2 and deg[11] == 2
    assert deg[5] == 4 and deg[6] == 4
    for e in p.edges:
        assert e in [] or (e.id in p.subdomains[e.a].edges and e.id in p.subdomains[e.b].edges)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_points_inside_cells_and_counts(cfg):
    p = make_config(cfg, scale=0.05)
    for s in p.subdomains:
        assert np.all(s.x_f[:, 0] >= s.lo[0]) and np.all(s.x_f[:, 0] <= s.hi[0])
        assert np.all(s.x_f[:, 1] >= s.lo[1]) and np.all(s.x_f[:, 1] <= s.hi[1])
        assert s.u_target.shape == s.u_mask.shape == (len(s.x_u), p.d_out)
    for e in p.edges:
        sa, sb = p.subdomains[e.a], p.subdomains[e.b]
        # shared interface points lie on the common boundary of both cells
        ax = e.axis
        assert np.all(e.pts[:, ax] == np.float32(sa.hi[ax]))
        assert np.all(e.pts[:, ax] == np.float32(sb.lo[ax]))


def test_full_size_counts():
    p = make_config("C2")
    assert p.n_sub == 16 and len(p.edges) == 24
    assert all(len(s.x_f) == 15000 for s in p.subdomains)
    assert all(len(p.edges[e].pts) == 250 for s in p.subdomains for e in s.edges)
    # boundary subdomains carry 80 data points, the 4 interior ones none
    nu = sorted(len(s.x_u) for s in p.subdomains)
    assert nu == [0] * 4 + [80] * 12


def test_determinism_and_float32_exact():
    a = make_config("C1", scale=0.1)
    b = make_config("C1", scale=0.1)
    for sa, sb in zip(a.subdomains, b.subdomains):
        assert np.array_equal(sa.x_f, sb.x_f) and np.array_equal(sa.params, sb.params)
        assert np.array_equal(sa.x_f.astype(np.float32).astype(np.float64), sa.x_f)
        assert np.array_equal(sa.params.astype(np.float32).astype(np.float64), sa.params)


def test_init_slopes():
    # PAPER.md:95 n a^k = 1 at init (SPEC.md:121 every a^k = 0.1 for n = 10)
    from pinn_inputs import param_layout
    p = make_config("C3", scale=0.01)
    for ent in param_layout(p.sizes):
        if "a" in ent:
            assert all(np.float32(s.params[ent["a"][0]]) == np.float32(0.1) for s in p.subdomains)


def _segments_cross(p, q, r, s):
    d = lambda a, b, c: (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
    return (d(p, q, r) * d(p, q, s) < 0) and (d(r, s, p) * d(r, s, q) < 0)


def test_c5_voronoi_geometry():
    """C5 recipe (reading Z24): simple non-convex polygon; residual points in
    their own region; interface points on the bisector of their two seeds
    with no third seed nearer; boundary data on the polygon boundary."""
    from pinn_inputs import voronoi as vor
    from pinn_inputs.workloads import C5_ACT, C5_N_F
    P = vor.MAP_POLYGON
    n = len(P)
    for i in range(n):
        for j in range(i + 2, n):
            if (j + 1) % n == i:
                continue
            assert not _segments_cross(P[i], P[(i + 1) % n], P[j], P[(j + 1) % n])
    e = np.roll(P, -1, 0) - P
    cr = e[:, 0] * np.roll(e, -1, 0)[:, 1] - e[:, 1] * np.roll(e, -1, 0)[:, 0]
    assert (cr > 0).any() and (cr < 0).any()          # non-convex
    p = make_config("C5", scale=0.1)
    seeds = p.meta["seeds"]
    assert [s.activation for s in p.subdomains] == C5_ACT
    assert [len(s.x_f) for s in p.subdomains] == [round(0.1 * v) for v in C5_N_F]
    for s in p.subdomains:
        assert vor.inside(P, s.x_f).all()
        assert (vor.nearest(seeds, s.x_f) == s.id).all()
    assert len(p.edges) >= 9                           # a connected 10-region partition
    for ed in p.edges:
        x = ed.pts
        da = np.linalg.norm(x - seeds[ed.a], axis=1)
        db = np.linalg.norm(x - seeds[ed.b], axis=1)
        np.testing.assert_allclose(da, db, rtol=0, atol=2e-6)
        dmin = np.min(np.linalg.norm(x[:, None, :] - seeds[None], axis=2), axis=1)
        assert np.all(dmin >= da - 2e-6)
        assert vor.inside(P, x).all()
        nrm = np.array(ed.normal)
        assert abs(np.linalg.norm(nrm) - 1.0) < 1e-6
        np.testing.assert_allclose(np.abs((x[1:] - x[:-1]) @ nrm), 0.0, atol=2e-6)
    # boundary data carry K; interior data do not
    nb = 0
    for s in p.subdomains:
        kb = s.u_mask[:, 1] == 1.0
        nb += kb.sum()
        xb = s.x_u[kb]
        if len(xb):
            a, b = P[None, :, :], np.roll(P, -1, 0)[None, :, :]
            t = np.clip((((xb[:, None] - a) * (b - a)).sum(-1)) / ((b - a) ** 2).sum(-1), 0, 1)
            dist = np.linalg.norm(xb[:, None] - (a + t[..., None] * (b - a)), axis=2).min(1)
            assert dist.max() < 1e-5
    assert nb == round(0.1 * 400)
