"""Pins for oracle/loss.py: SPEC worked loss examples, structural invariants of
Eq. (3)/(5)/(6), finite-difference gradients, closed-form Adam, Eq. (4)."""

import dataclasses
import math

import numpy as np
import pytest
import torch

from oracle import loss as OL
from pinn_inputs import make_config, n_params, param_layout, perturb_params

DT = torch.float64


def _const_params(prob, c):
    """Parameters of a net whose output is the constant vector c."""
    th = np.zeros(n_params(prob.sizes))
    lay = param_layout(prob.sizes)
    for ent in lay:
        if "a" in ent:
            th[ent["a"][0]] = 0.1
    o, n = lay[-1]["b"]
    th[o:o + n] = c
    return th


def _with_params(prob, params):
    subs = [dataclasses.replace(s, params=np.asarray(p, dtype=np.float64))
            for s, p in zip(prob.subdomains, params)]
    return dataclasses.replace(prob, subdomains=subs)


def _small(cfg, **kw):
    base = dict(n_f=24, n_i=6, n_u=8, width=5, n_hidden=2)
    base.update(kw)
    return make_config(cfg, **base)


def test_mse_examples():
    # SPEC.md:390 predictions (0,0), targets (1,3) -> 5 ; empty -> 0
    r = torch.tensor([[1.0], [3.0]], dtype=DT)
    assert float(OL._mse_sum(r)) == 5.0
    assert float(OL._mse_sum(torch.zeros((0, 1), dtype=DT))) == 0.0


def test_uavg_and_flux_examples_through_subdomain_loss():
    """SPEC.md:402 local 1, neighbour 3 -> |1-2|^2 = 1 ; SPEC.md:411 flux 1.5 vs
    0.5 -> 1.  Constant nets u = 1 and u = sqrt(3): Burgers flux u^2/2 = 0.5 / 1.5."""
    p = _small("C1")
    p = _with_params(p, [_const_params(p, 1.0), _const_params(p, 3.0)])
    th = [torch.tensor(s.params) for s in p.subdomains]
    _, (mu, mf, ma, mi) = OL.subdomain_loss(p, 0, th)
    assert float(ma) == pytest.approx(1.0, abs=1e-15)
    p = _with_params(p, [_const_params(p, 1.0), _const_params(p, math.sqrt(3.0))])
    th = [torch.tensor(s.params) for s in p.subdomains]
    _, (mu, mf, ma, mi) = OL.subdomain_loss(p, 0, th)
    assert float(mi) == pytest.approx(1.0, abs=1e-14)
    assert float(mf) == 0.0        # constant field solves Burgers


def test_residual_jump_and_two_edges_examples():
    """SPEC.md:418 residual 2 vs 0 -> 4 ; SPEC.md:403 two live edges each
    contributing 1 -> 2 (2x2 XPINN, corner subdomain has two edges)."""
    p = _small("C3", gpus=4)            # 2x2 Burgers XPINN
    p = _with_params(p, [_const_params(p, c) for c in (1.0, 3.0, 3.0, 5.0)])
    th = [torch.tensor(s.params) for s in p.subdomains]
    _, (mu, mf, ma, mi) = OL.subdomain_loss(p, 0, th)
    assert len(p.subdomains[0].edges) == 2
    assert float(ma) == pytest.approx(2.0, abs=1e-15)
    # inject neighbour residual payloads = 2 on every edge of subdomain 0
    pay = {}
    for e in p.subdomains[0].edges:
        nb = p.edge_neighbor(0, e)
        n_i = len(p.edges[e].pts)
        pay[(nb, e)] = (torch.full((n_i, 1), 3.0, dtype=DT), torch.full((n_i, 1), 2.0, dtype=DT))
    _, (mu, mf, ma, mi) = OL.subdomain_loss(p, 0, th, pay)
    assert float(mi) == pytest.approx(8.0, abs=1e-14)   # 4 per edge, two edges


def test_total_weighting_example():
    # SPEC.md:428 weights (1,1,20,20) on (0.1, 0.2, 0.01, 0.02) -> 0.9
    w = (1.0, 1.0, 20.0, 20.0)
    parts = (0.1, 0.2, 0.01, 0.02)
    assert sum(a * b for a, b in zip(w, parts)) == pytest.approx(0.9, abs=1e-15)
    p = _small("C1")
    p = dataclasses.replace(p, w_u=1.0, w_f=1.0, w_i=20.0, w_if=20.0)
    th = [torch.tensor(s.params) for s in p.subdomains]
    J, (mu, mf, ma, mi) = OL.subdomain_loss(p, 0, th)
    assert float(J) == pytest.approx(float(mu + mf + 20 * ma + 20 * mi), rel=1e-15)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_single_subdomain_degenerates_to_pinn(cfg):
    """N_sd = 1: cPINN (Eq. 5) = XPINN (Eq. 6) = PINN (Eq. 3) bitwise (PAPER.md:113 vs 151)."""
    Js = []
    for m in ("pinn", "cpinn", "xpinn"):
        p = _small(cfg, method=m, nx=1, ny=1)
        th = [torch.tensor(s.params) for s in p.subdomains]
        J, (mu, mf, ma, mi) = OL.subdomain_loss(p, 0, th)
        assert float(ma) == 0.0 and float(mi) == 0.0
        assert float(J) == float(p.w_u * mu + p.w_f * mf)
        Js.append(float(J))
    assert Js[0] == Js[1] == Js[2]


@pytest.mark.parametrize("cfg,method", [("C1", "cpinn"), ("C2", "cpinn"), ("C2", "xpinn"),
                                        ("C3", "xpinn"), ("C4", "xpinn"), ("C4", "cpinn"),
                                        ("C5", "xpinn"), ("C5", "cpinn")])
def test_identical_neighbours_have_zero_interface_loss(cfg, method):
    """{{u}} = (u_q + u_q+)/2: identical nets give MSE_uavg = MSE_flux = MSE_R = 0 exactly
    (C5: with one activation everywhere -- identical parameters are identical nets)."""
    kw = dict(activations=["sin"] * 10) if cfg == "C5" else {}
    p = _small(cfg, method=method, **kw)
    p = _with_params(p, [p.subdomains[0].params] * p.n_sub)
    th = [torch.tensor(s.params) for s in p.subdomains]
    for q in range(p.n_sub):
        _, (mu, mf, ma, mi) = OL.subdomain_loss(p, q, th)
        assert float(ma) == 0.0 and float(mi) == 0.0


def test_symmetric_mismatch():
    """q's interface mismatch on an edge equals q+'s."""
    p = _small("C1")
    th = [torch.tensor(s.params) for s in p.subdomains]
    _, a = OL.subdomain_loss(p, 0, th)
    _, b = OL.subdomain_loss(p, 1, th)
    assert float(a[2]) == pytest.approx(float(b[2]), rel=1e-14)
    assert float(a[3]) == pytest.approx(float(b[3]), rel=1e-14)


def test_cpinn_rejects_time_interfaces():
    p = _small("C3", method="cpinn", gpus=4)
    th = [torch.tensor(s.params) for s in p.subdomains]
    with pytest.raises(ValueError):
        OL.subdomain_loss(p, 0, th)


@pytest.mark.parametrize("cfg,method", [("C1", "cpinn"), ("C2", "cpinn"), ("C2", "xpinn"),
                                        ("C3", "xpinn"), ("C3", "hybrid"), ("C4", "xpinn"), ("C4", "cpinn"),
                                        ("C5", "xpinn"), ("C5-sin", "xpinn"), ("C5-cos", "xpinn")])
def test_gradient_matches_central_differences(cfg, method):
    """dJ_q/dTheta_q vs central differences of the literal loss (h = 1e-6),
    neighbours fixed.  This also pins reading Z1: the
    u_q inside {{u}} is differentiated.  C5 variants put a tanh / sin / cos
    region last (its neighbours keep Table 3's mixed activations)."""
    kw = dict(n_f=10, n_i=4, n_u=5, width=4, n_hidden=2)
    if cfg == "C3":
        kw["gpus"] = 4
    if cfg.startswith("C5"):
        last = cfg[3:] or "tanh"
        kw["activations"] = ["tanh", "sin", "cos", "tanh", "sin", "cos", "tanh", "sin", "cos", last]
        cfg = "C5"
    p = perturb_params(make_config(cfg, method=method, **kw), scale=0.2)
    th = [torch.tensor(s.params) for s in p.subdomains]
    q = p.n_sub - 1
    _, g = OL.loss_and_grad(p, q, th)
    h = 1e-5 if p.pde == "heat_inv" else 1e-6   # C5: J ~ 1e4 (T, K ~ 20), so rounding needs a larger h
    fd = np.zeros(len(g))
    for i in range(len(g)):
        tp = [t.clone() for t in th]; tm = [t.clone() for t in th]
        tp[q][i] += h; tm[q][i] -= h
        Jp, _ = OL.subdomain_loss(p, q, tp)
        Jm, _ = OL.subdomain_loss(p, q, tm)
        fd[i] = (float(Jp) - float(Jm)) / (2 * h)
    err = np.max(np.abs(g.numpy() - fd) / np.maximum(1.0, np.abs(fd)))
    assert err < 1e-6, err


@pytest.mark.parametrize("cfg,method", [("C1", "cpinn"), ("C2", "xpinn"), ("C4", "cpinn"), ("C5", "xpinn")])
def test_slope_gradient_homogeneity_identity(cfg, method):
    """J depends on (a^k, W^k, b^k) only through (n a^k W^k, n a^k b^k) (Eq. 2 with
    the slope inside Phi), hence a^k dJ/da^k = <W^k, dJ/dW^k> + <b^k, dJ/db^k>
    exactly, for every hidden layer k."""
    from pinn_inputs import param_layout
    kw = dict(n_f=30, n_i=6, n_u=8, width=6, n_hidden=3)
    p = perturb_params(make_config(cfg, method=method, **kw), scale=0.3)
    th = [torch.tensor(s.params) for s in p.subdomains]
    q = p.n_sub - 1
    _, g = OL.loss_and_grad(p, q, th)
    t = th[q].numpy(); g = g.numpy()
    for ent in param_layout(p.sizes):
        if "a" not in ent:
            continue
        (ow, nw), (ob, nb), (oa, _) = ent["W"], ent["b"], ent["a"]
        lhs = t[oa] * g[oa]
        rhs = t[ow:ow + nw] @ g[ow:ow + nw] + t[ob:ob + nb] @ g[ob:ob + nb]
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(rhs)), (lhs, rhs)


def test_gradient_linearity():
    """grad(a L1 + b L2) = a grad L1 + b grad L2 (weights enter linearly)."""
    p = _small("C2", method="xpinn")
    th = [torch.tensor(s.params) for s in p.subdomains]
    g = {}
    for tag, w in (("u", (1, 0, 0, 0)), ("f", (0, 1, 0, 0)), ("all", (2.0, 3.0, 0, 0))):
        pp = dataclasses.replace(p, w_u=w[0], w_f=w[1], w_i=w[2], w_if=w[3])
        _, g[tag] = OL.loss_and_grad(pp, 5, th)
    np.testing.assert_allclose(g["all"].numpy(), (2 * g["u"] + 3 * g["f"]).numpy(), rtol=1e-12, atol=1e-12)


def test_adam_closed_forms():
    th = torch.tensor([0.5, -1.0, 2.0], dtype=DT)
    st = OL.adam_init(th)
    # SPEC.md:571 zero gradient -> unchanged
    th1, st1 = OL.adam_step(th, torch.zeros(3, dtype=DT), st, 1e-3)
    assert torch.equal(th1, th) and st1.t == 1
    # SPEC.md:572 first step -> -lr g / (|g| + eps)
    g = torch.tensor([0.3, -2.0, 1e-9], dtype=DT)
    th1, _ = OL.adam_step(th, g, st, 1e-3)
    np.testing.assert_allclose((th1 - th).numpy(), (-1e-3 * g / (g.abs() + 1e-8)).numpy(), rtol=1e-12)
    # SPEC.md:573 f(w) = w^2, lr 0.1: |w| decreases after burn-in
    w = torch.tensor([1.0], dtype=DT)
    st = OL.adam_init(w)
    hist = []
    for _ in range(100):
        w, st = OL.adam_step(w, 2 * w, st, 0.1)
        hist.append(abs(float(w)))
    assert hist[-1] < 0.05 * hist[0] + 1e-3


def test_stitch_partition_of_unity_and_examples():
    # interface S=2 average of 1 and 3 -> 2; 4-way corner (1,2,3,4) -> 2.5
    p = _small("C3", gpus=4)     # 2x2 on [-1,1]x[0,1]
    p = _with_params(p, [_const_params(p, c) for c in (1.0, 2.0, 3.0, 4.0)])
    th = [torch.tensor(s.params) for s in p.subdomains]
    X = np.array([[0.0, 0.5], [-0.5, 0.25], [0.0, 0.25], [-0.5, 0.5], [0.5, 0.75]])
    u = OL.stitch(p, th, X)[:, 0].numpy()
    np.testing.assert_allclose(u, [2.5, 1.0, 1.5, 2.0, 4.0], rtol=1e-15)
    # partition of unity: constant 1 everywhere -> stitched 1 on a probe grid incl. edges
    p1 = _with_params(p, [_const_params(p, 1.0)] * 4)
    th = [torch.tensor(s.params) for s in p1.subdomains]
    g = np.stack(np.meshgrid(np.linspace(-1, 1, 9), np.linspace(0, 1, 5)), -1).reshape(-1, 2)
    np.testing.assert_allclose(OL.stitch(p1, th, g)[:, 0].numpy(), 1.0, rtol=1e-15)


def test_train_step_decreases_loss_on_average():
    """Soft trend: 30 synchronous steps on small C1 lower the total loss."""
    p = _small("C1", n_f=40)
    p = dataclasses.replace(p, lr=5e-3)
    st = OL.init_state(p)
    st, bd0 = OL.train_step(p, st)
    for _ in range(29):
        st, bd = OL.train_step(p, st)
    assert sum(b.total for b in bd) < sum(b.total for b in bd0)


@pytest.mark.parametrize("cfg,method", [("C2", "cpinn"), ("C4", "xpinn")])
def test_chunked_loss_terms_match_graph_loss(cfg, method):
    """The chunked, no-grad evaluation used for full-size checks equals the
    graph-building Eq. (5)/(6) evaluation."""
    p = perturb_params(_small(cfg, method=method, n_f=50), scale=0.2)
    th = [torch.tensor(s.params) for s in p.subdomains]
    for q in (0, p.n_sub - 1):
        J, parts = OL.subdomain_loss(p, q, th)
        bd = OL.subdomain_loss_terms(p, q, th, chunk=7)
        ref = [float(x) for x in parts] + [float(J)]
        np.testing.assert_allclose(bd.as_list(), ref, rtol=1e-12, atol=1e-15)


def test_hybrid_is_flux_in_space_residual_in_time():
    """hybrid = cPINN flux continuity on x-normal edges + XPINN
    residual continuity on t-normal edges; per-edge terms add up."""
    p = perturb_params(_small("C3", method="hybrid", gpus=4), scale=0.2)
    th = [torch.tensor(s.params) for s in p.subdomains]
    pc = dataclasses.replace(p, method="cpinn")
    px = dataclasses.replace(p, method="xpinn")
    for q in range(4):
        _, (mu, mf, ma, mi) = OL.subdomain_loss(p, q, th)
        want = 0.0
        for e in p.subdomains[q].edges:
            ed = p.edges[e]
            nb = p.edge_neighbor(q, e)
            X = torch.tensor(ed.pts)
            pp = pc if ed.axis == 0 else px
            _, sq = OL.interface_payload(pp, th[q], X, ed.normal, create_graph=False)
            _, sn = OL.interface_payload(pp, th[nb], X, ed.normal, create_graph=False)
            want += float(((sq - sn) ** 2).sum()) / len(X)
        assert float(mi) == pytest.approx(want, rel=1e-12)


# --------------------------------------------------------------------------
# Systems (D_o > 1): the output mask of MSE_u and the sum over fields (Z4),
# pinned with constant networks and hand-computed values.
# --------------------------------------------------------------------------

def test_mse_u_output_mask_and_field_sum_ns():
    """NS cavity data (Z16): targets (u, v) = (1, 0) on the lid y = 1, (0, 0)
    on the other walls, p unconstrained (mask 0).  A constant net (1, 2, 3)
    gives per point (t_u - 1)^2 + (0 - 2)^2 (+ 0 for p, whatever the net's
    p), so MSE_u = mean over data points of (t_u - 1)^2 + 4 (P:159 summed
    over fields, reading Z4; the mask drops p)."""
    p = make_config("C4", method="xpinn", n_f=5, n_i=4, n_u=16, width=5, n_hidden=2)
    base = [_const_params(p, [1.0, 2.0, 3.0]) for _ in range(p.n_sub)]
    alt = [_const_params(p, [1.0, 2.0, -50.0]) for _ in range(p.n_sub)]
    for q in range(p.n_sub):
        s = p.subdomains[q]
        tu = s.u_target[:, 0]
        assert np.all(s.u_mask[:, 2] == 0) and np.all(s.u_mask[:, :2] == 1)
        want = float(np.mean((tu - 1.0) ** 2 + 4.0)) if len(tu) else 0.0
        for params in (base, alt):                          # p never enters MSE_u
            pp = _with_params(p, params)
            th = [torch.tensor(s2.params) for s2 in pp.subdomains]
            _, (mu, mf, ma, mi) = OL.subdomain_loss(pp, q, th)
            assert float(mu) == pytest.approx(want, rel=1e-14, abs=1e-300)
        lid = np.sum(s.x_u[:, 1] == 1.0)
        if s.iy == 1 and len(tu):
            assert lid > 0 and want == pytest.approx(4.0 + (len(tu) - lid) / len(tu), rel=1e-14)


def test_interface_terms_sum_over_fields_ns():
    """Z4 for the interface terms with constant nets q = (1, 2, 3),
    neighbour = (3, 4, 7), all derivatives 0:
      u_avg : per point sum_o ((u_q - u_n)/2)^2 = 1 + 1 + 4 = 6 -> 6 per edge;
      XPINN residual jump: F = (0, 0, 0) on both sides -> 0;
      cPINN flux jump, Table 1 with n = (1, 0): q (u^2 + p, uv, u) = (4, 2, 1),
        neighbour (9 + 7, 12, 3) = (16, 12, 3) -> 144 + 100 + 4 = 248 per point;
        with n = (0, 1): q (uv, v^2 + p, v) = (2, 7, 2), neighbour (12, 23, 4)
        -> 100 + 256 + 4 = 360 per point."""
    for method in ("xpinn", "cpinn"):
        p = make_config("C4", method=method, n_f=5, n_i=4, n_u=8, width=5, n_hidden=2)
        params = []
        for q in range(p.n_sub):
            params.append(_const_params(p, [1.0, 2.0, 3.0] if q == 0 else [3.0, 4.0, 7.0]))
        pp = _with_params(p, params)
        th = [torch.tensor(s.params) for s in pp.subdomains]
        _, (mu, mf, ma, mi) = OL.subdomain_loss(pp, 0, th)
        edges = pp.subdomains[0].edges
        assert len(edges) == 2                              # corner subdomain of the 4x2 grid
        assert float(ma) == pytest.approx(6.0 * len(edges), rel=1e-14)
        assert float(mf) == 0.0
        if method == "xpinn":
            assert float(mi) == 0.0
        else:
            axes = sorted(pp.edges[e].axis for e in edges)
            assert axes == [0, 1]
            assert float(mi) == pytest.approx(248.0 + 360.0, rel=1e-14)
