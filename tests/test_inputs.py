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
