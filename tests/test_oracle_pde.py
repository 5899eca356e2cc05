"""Pins for oracle/pde.py: exact PDE solutions give residual 0, Table 1 columns,
SPEC worked flux examples, and a network that IS an exact Burgers solution."""

import math

import numpy as np
import pytest
import torch

from oracle import net as onet
from oracle import pde as opde
from pinn_inputs import make_config, n_params, param_layout

DT = torch.float64


def _pts(n=1000, lo=(-1, 0), hi=(1, 1), seed=0):
    rng = np.random.default_rng(seed)
    return torch.tensor(np.stack([rng.uniform(lo[0], hi[0], n), rng.uniform(lo[1], hi[1], n)], 1), dtype=DT)


def _autograd_fields(fn_list, X):
    """Fields of closed-form functions by autograd (independent of oracle.net)."""
    X = X.clone().requires_grad_(True)
    out = []
    for fn in fn_list:
        u = fn(X)
        g = torch.autograd.grad(u.sum(), X, create_graph=True)[0]
        g11 = torch.autograd.grad(g[:, 0].sum(), X, create_graph=True)[0][:, 0]
        g22 = torch.autograd.grad(g[:, 1].sum(), X, create_graph=True)[0][:, 1]
        out.append({"u": u, "d1": g[:, 0], "d2": g[:, 1], "d11": g11, "d22": g22})
    return out, X


class _P:  # minimal problem stand-in for the dispatchers
    def __init__(self, pde, nu=0.01 / math.pi, re=100.0):
        self.pde, self.nu, self.re = pde, nu, re


NU = 0.01 / math.pi


def test_burgers_trivial_examples():
    X = _pts(10)
    c = torch.full((10,), 2.5, dtype=DT)
    z = torch.zeros(10, dtype=DT)
    # SPEC.md:291 u == c -> 0
    F = opde.burgers_residual([{"u": c, "d1": z, "d2": z, "d11": z}], X, NU)
    assert torch.all(F == 0)
    # SPEC.md:292 u = x -> F = x
    F = opde.burgers_residual([{"u": X[:, 0], "d1": z + 1, "d2": z, "d11": z}], X, NU)
    assert torch.allclose(F[:, 0], X[:, 0], rtol=0, atol=0)
    # SPEC.md:299-300 flux: u==0 -> 0 ; u==2, u_x=0 -> 2 (n = (1, 0))
    assert torch.all(opde.burgers_flux_n([{"u": z, "d1": z}], X, (1.0, 0.0), NU) == 0)
    assert torch.all(opde.burgers_flux_n([{"u": z + 2, "d1": z}], X, (1.0, 0.0), NU) == 2)


def test_burgers_exact_solutions_vanish():
    X = _pts(1000)
    # u = x/(t+1): u_t = -x/(t+1)^2, u u_x = x/(t+1)^2, u_xx = 0
    x, t = X[:, 0], X[:, 1]
    z = torch.zeros_like(x)
    fl = [{"u": x / (t + 1), "d1": 1 / (t + 1), "d2": -x / (t + 1) ** 2, "d11": z}]
    assert opde.burgers_residual(fl, X, NU).abs().max() < 1e-14
    # viscous travelling wave u = c - a tanh(a (x - c t)/(2 nu)), derivatives by hand
    a, c = 0.8, 0.3
    T = torch.tanh(a * (x - c * t) / (2 * NU))
    S = 1 - T * T
    fl = [{"u": c - a * T, "d1": -a * a * S / (2 * NU), "d2": a * a * c * S / (2 * NU),
           "d11": 2 * a ** 3 * T * S / (4 * NU * NU)}]
    F = opde.burgers_residual(fl, X, NU)
    assert F.abs().max() < 1e-9 * (a ** 3 / NU)


def test_network_that_is_an_exact_burgers_solution():
    """Closed-form network fixture: one tanh unit reproduces the travelling wave
    exactly, so the oracle's full pipeline (net -> AD -> F) must give F = 0."""
    a, c = 0.8, 0.3
    sizes = [2, 3, 1]                      # extra units have zero output weight
    lay = param_layout(sizes)
    th = torch.zeros(n_params(sizes), dtype=DT)
    o = lay[0]["W"][0]
    th[o:o + 2] = torch.tensor([a / (2 * NU), -a * c / (2 * NU)], dtype=DT)
    th[o + 2:o + 6] = torch.tensor([0.3, -0.7, 1.1, 0.2], dtype=DT)
    th[lay[0]["a"][0]] = 0.1               # s = n a = 1
    th[lay[1]["W"][0]] = -a
    th[lay[1]["b"][0]] = c
    X = _pts(500, seed=3)
    fl, Xg = onet.fields(th, sizes, X, "tanh", 10.0, second=(True, False))
    F = opde.burgers_residual(fl, Xg, NU)
    assert F.abs().max() < 1e-9 * (a ** 3 / NU)


def test_poisson_exact_solution():
    X = _pts(1000, (0, 0), (1, 1))
    pi = math.pi
    fl, Xg = _autograd_fields([lambda X: torch.sin(pi * X[:, 0]) * torch.sin(pi * X[:, 1])], X)
    assert opde.poisson_residual(fl, Xg).abs().max() < 1e-12
    # flux along n = (1, 0) is u_x, along (0, 1) is u_y
    f1 = opde.poisson_flux_n(fl, Xg, (1.0, 0.0))[:, 0]
    assert torch.allclose(f1, pi * torch.cos(pi * X[:, 0]) * torch.sin(pi * X[:, 1]), atol=1e-13)


def test_heat_paper_fields():
    # PAPER.md:828-829 T = 20 exp(-0.1 y), K = 20 + exp(0.1 y) sin(0.5 x) -> F = 0
    X = _pts(1000, (0, 0), (6, 6))
    fl, Xg = _autograd_fields([lambda X: 20.0 * torch.exp(-0.1 * X[:, 1])], X)
    assert opde.heat_residual(fl, Xg).abs().max() < 1e-12
    # SPEC.md:335-337 K(0,0) = 20 ; K(pi, 0) = 21 ; T(., 0) = 20
    K, _, _ = opde.heat_K(torch.tensor([[0.0, 0.0], [math.pi, 0.0]], dtype=DT))
    assert K[0] == 20.0 and abs(float(K[1]) - 21.0) < 1e-14


def test_heat_expanded_form_is_divergence_of_flux():
    """For a field with T_x != 0 the expanded residual equals d_x(K T_x) +
    d_y(K T_y) - f computed by autograd (pins K_x and K_y)."""
    X = _pts(300, (0, 0), (3, 3), seed=5).requires_grad_(True)
    T = X[:, 0] ** 2 * X[:, 1] + torch.sin(X[:, 0]) * torch.cos(0.7 * X[:, 1])
    K = 20.0 + torch.exp(0.1 * X[:, 1]) * torch.sin(0.5 * X[:, 0])
    g = torch.autograd.grad(T.sum(), X, create_graph=True)[0]
    div = torch.autograd.grad((K * g[:, 0]).sum(), X, create_graph=True)[0][:, 0] + \
        torch.autograd.grad((K * g[:, 1]).sum(), X, create_graph=True)[0][:, 1]
    ref = div - 4.0 * torch.exp(-0.1 * X[:, 1])
    fl, Xg = _autograd_fields([lambda X: X[:, 0] ** 2 * X[:, 1] + torch.sin(X[:, 0]) * torch.cos(0.7 * X[:, 1])],
                              X.detach())
    F = opde.heat_residual(fl, Xg)[:, 0]
    assert torch.allclose(F, ref.detach(), rtol=1e-12, atol=1e-11)


def test_ns_uniform_flow_and_kovasznay():
    X = _pts(1000, (0, 0), (1, 1))
    z = torch.zeros(1000, dtype=DT)
    one = {"u": z + 1, "d1": z, "d2": z, "d11": z, "d22": z}
    zero = {"u": z, "d1": z, "d2": z, "d11": z, "d22": z}
    assert torch.all(opde.ns_residual([one, zero, zero], X, 100.0) == 0)
    # SPEC.md:318-319 u=1, v=0, p=0, n=(1,0) -> x-mom 1, y-mom 0, mass 1
    fx = opde.ns_flux_n([one, zero, zero], X, (1.0, 0.0), 100.0)
    assert torch.all(fx[:, 0] == 1) and torch.all(fx[:, 1] == 0) and torch.all(fx[:, 2] == 1)
    # Kovasznay flow (exact steady NS solution)
    Re = 40.0
    lam = Re / 2 - math.sqrt(Re * Re / 4 + 4 * math.pi ** 2)
    pi = math.pi
    fns = [lambda X: 1 - torch.exp(lam * X[:, 0]) * torch.cos(2 * pi * X[:, 1]),
           lambda X: lam / (2 * pi) * torch.exp(lam * X[:, 0]) * torch.sin(2 * pi * X[:, 1]),
           lambda X: 0.5 * (1 - torch.exp(2 * lam * X[:, 0]))]
    fl, Xg = _autograd_fields(fns, X)
    assert opde.ns_residual(fl, Xg, Re).abs().max() < 1e-11


def test_ns_table1_worked_example():
    """Table 1 evaluated at u=1, v=2, p=3, u_x=4, u_y=5,
    v_x=6, v_y=7, Re=10, by hand:
      x-dir: x-mom u^2+p-u_x/Re = 1+3-0.4 = 3.6 ; y-mom uv-v_x/Re = 2-0.6 = 1.4 ; mass u = 1
      y-dir: x-mom uv-u_y/Re = 2-0.5 = 1.5 ; y-mom v^2+p-v_y/Re = 4+3-0.7 = 6.3 ; mass v = 2"""
    one = torch.ones(1, dtype=DT)
    u = {"u": 1 * one, "d1": 4 * one, "d2": 5 * one}
    v = {"u": 2 * one, "d1": 6 * one, "d2": 7 * one}
    p = {"u": 3 * one, "d1": 0 * one, "d2": 0 * one}
    fx = opde.ns_flux_n([u, v, p], None, (1.0, 0.0), 10.0)[0]
    fy = opde.ns_flux_n([u, v, p], None, (0.0, 1.0), 10.0)[0]
    np.testing.assert_allclose(fx.numpy(), [3.6, 1.4, 1.0], rtol=1e-15)
    np.testing.assert_allclose(fy.numpy(), [1.5, 6.3, 2.0], rtol=1e-15)


def test_inputs_targets_match_paper_conditions():
    # Burgers IC u(0, x) = -sin(pi x)
    p = make_config("C1")
    for s in p.subdomains:
        ic = s.x_u[:, 1] == 0.0
        assert ic.sum() == 50
        np.testing.assert_allclose(s.u_target[ic, 0], -np.sin(np.pi * s.x_u[ic, 0]), atol=1e-7)
        assert np.all(s.u_target[~ic, 0] == 0) and np.all(np.abs(s.x_u[~ic, 0]) == 1.0)


# --------------------------------------------------------------------------
# inverse heat (C5): one net with outputs (T, K) (reading Z17')
# --------------------------------------------------------------------------

def _tk(X):
    return (lambda X: 20.0 * torch.exp(-0.1 * X[:, 1]),
            lambda X: 20.0 + torch.exp(0.1 * X[:, 1]) * torch.sin(0.5 * X[:, 0]))


def test_heat_inv_paper_pair_vanishes():
    # the exact (T, K) pair satisfies d_x(K T_x) + d_y(K T_y) = f
    X = _pts(1000, (0, 0), (10, 6), seed=3)
    fl, Xg = _autograd_fields(list(_tk(X)), X)
    assert opde.heat_inv_residual(fl, Xg).abs().max() < 1e-12
    # T_x = 0, so K = 20 + C e^{0.1 y} solves it too (reading Z22, identifiability):
    # K = 20 gives 0; K = 25 gives F = 25 * 0.2 e^{-0.1 y} - 4 e^{-0.1 y} = e^{-0.1 y}
    for c, want in ((20.0, 0.0), (25.0, 1.0)):
        fl2, Xg2 = _autograd_fields([_tk(X)[0], lambda X, c=c: c + 0.0 * X[:, 0] * X[:, 1]], X)
        F = opde.heat_inv_residual(fl2, Xg2)[:, 0]
        assert torch.allclose(F, want * torch.exp(-0.1 * X[:, 1]), rtol=1e-12, atol=1e-12)


def test_heat_inv_is_divergence_of_flux_and_reduces_to_heat():
    """For arbitrary smooth T and K: the expanded residual equals
    div(K grad T) - f by autograd (pins which output is T and which is K and
    the K_x T_x + K_y T_y cross terms); the flux with n = e1, e2 is K T_x,
    K T_y; with K = the known heat_K it equals the forward heat residual."""
    X = _pts(300, (0, 0), (4, 3), seed=9)
    Tf = lambda X: X[:, 0] ** 2 * X[:, 1] + torch.sin(X[:, 0]) * torch.cos(0.7 * X[:, 1])
    Kf = lambda X: 3.0 + X[:, 0] * X[:, 1] ** 2 + torch.cos(0.3 * X[:, 0])
    Xr = X.clone().requires_grad_(True)
    T, K = Tf(Xr), Kf(Xr)
    g = torch.autograd.grad(T.sum(), Xr, create_graph=True)[0]
    div = torch.autograd.grad((K * g[:, 0]).sum(), Xr, create_graph=True)[0][:, 0] + \
        torch.autograd.grad((K * g[:, 1]).sum(), Xr, create_graph=True)[0][:, 1]
    ref = (div - 4.0 * torch.exp(-0.1 * Xr[:, 1])).detach()
    fl, Xg = _autograd_fields([Tf, Kf], X)
    assert torch.allclose(opde.heat_inv_residual(fl, Xg)[:, 0], ref, rtol=1e-12, atol=1e-11)
    fx = opde.heat_inv_flux_n(fl, Xg, (1.0, 0.0))[:, 0]
    fy = opde.heat_inv_flux_n(fl, Xg, (0.0, 1.0))[:, 0]
    assert torch.allclose(fx, (K * g[:, 0]).detach(), rtol=1e-13)
    assert torch.allclose(fy, (K * g[:, 1]).detach(), rtol=1e-13)
    fl3, Xg3 = _autograd_fields([Tf, _tk(X)[1]], X)
    flh, Xgh = _autograd_fields([Tf], X)
    assert torch.allclose(opde.heat_inv_residual(fl3, Xg3), opde.heat_residual(flh, Xgh), rtol=1e-12, atol=1e-11)


def test_heat_inv_c5_targets_are_the_paper_fields():
    p = make_config("C5", scale=0.05)
    for s in p.subdomains:
        x = s.x_u
        np.testing.assert_allclose(s.u_target[:, 0], 20.0 * np.exp(-0.1 * x[:, 1]), rtol=1e-6)
        np.testing.assert_allclose(s.u_target[:, 1], 20.0 + np.exp(0.1 * x[:, 1]) * np.sin(0.5 * x[:, 0]),
                                   rtol=1e-6)
        assert np.all(s.u_mask[:, 0] == 1.0)           # T data everywhere (interior + boundary)


# --------------------------------------------------------------------------
# Flux / residual consistency: for every operator in conservation form the
# divergence of the interface flux f(u) (the quantity cPINN matches across an
# edge, Table 1) equals the residual F plus the forcing.
# Each flux is evaluated with n = e1 and n = e2 as a field of X and
# differentiated by autograd, so every term of f (including the viscous
# -nu u_x of Burgers and K of the heat flux) is pinned against the residual
# written independently in oracle/pde.py.
# --------------------------------------------------------------------------

def _div_flux(flux_fn, fl, Xg):
    fx = flux_fn(fl, Xg, (1.0, 0.0))
    fy = flux_fn(fl, Xg, (0.0, 1.0))
    cols = []
    for e in range(fx.shape[1]):
        gx = torch.autograd.grad(fx[:, e].sum(), Xg, create_graph=True)[0][:, 0]
        gy = torch.autograd.grad(fy[:, e].sum(), Xg, create_graph=True)[0][:, 1]
        cols.append(gx + gy)
    return torch.stack(cols, dim=1)


def test_burgers_flux_divergence_is_residual():
    """d_x (u^2/2 - nu u_x) + d_t u = u_t + u u_x - nu u_xx = F (SPEC.md:342,
    reading Z13) for a field with u_x, u_xx != 0: pins the viscous term."""
    X = _pts(400, seed=11)
    fl, Xg = _autograd_fields([lambda X: torch.sin(2.0 * X[:, 0]) * torch.cos(X[:, 1]) + X[:, 0] ** 2 * X[:, 1]], X)
    F = opde.burgers_residual(fl, Xg, NU)
    D = _div_flux(lambda f, x, n: opde.burgers_flux_n(f, x, n, NU), fl, Xg)
    assert torch.allclose(D, F, rtol=1e-12, atol=1e-12)
    # and the viscous term is really there: dropping nu changes the divergence by nu u_xx
    D0 = _div_flux(lambda f, x, n: opde.burgers_flux_n(f, x, n, 0.0), fl, Xg)
    assert torch.allclose(D - D0, -NU * fl[0]["d11"][:, None], rtol=1e-10, atol=1e-14)
    assert float((D - D0).abs().max()) > 1e-4


def test_poisson_and_heat_flux_divergence_is_residual_plus_forcing():
    """div(grad u) = F + f (Poisson) and div(K grad u) = F + f (heat, Eq. 15
    P:824) with K(x, y) of P:829: pins heat_flux_n (K times the normal
    derivative)."""
    X = _pts(400, (0, 0), (3, 2), seed=12)
    fn = lambda X: X[:, 0] ** 2 * X[:, 1] + torch.sin(X[:, 0]) * torch.cos(0.7 * X[:, 1])
    fl, Xg = _autograd_fields([fn], X)
    Dp = _div_flux(opde.poisson_flux_n, fl, Xg)
    assert torch.allclose(Dp[:, 0], opde.poisson_residual(fl, Xg)[:, 0] + opde.poisson_forcing(Xg),
                          rtol=1e-12, atol=1e-11)
    Dh = _div_flux(opde.heat_flux_n, fl, Xg)
    assert torch.allclose(Dh[:, 0], opde.heat_residual(fl, Xg)[:, 0] + opde.heat_forcing(Xg),
                          rtol=1e-12, atol=1e-10)
    # heat flux at a hand-checked point: x = pi, y = 0 -> K = 21; u = x^2 y + sin x cos 0.7y
    # u_x = 2 x y + cos x cos 0.7 y = -1 ; u_y = x^2 - 0.7 sin x sin 0.7 y = pi^2
    P = torch.tensor([[math.pi, 0.0]], dtype=DT)
    flp, Xp = _autograd_fields([fn], P)
    fx = float(opde.heat_flux_n(flp, Xp, (1.0, 0.0))[0, 0])
    fy = float(opde.heat_flux_n(flp, Xp, (0.0, 1.0))[0, 0])
    assert fx == pytest.approx(-21.0, rel=1e-13)
    assert fy == pytest.approx(21.0 * math.pi ** 2, rel=1e-13)


def test_ns_table1_flux_divergence():
    """Table 1 is the conservative momentum / mass flux of Eq. (11)
    (P:415-417): div of the x-/y-momentum rows = F_x + u div(u) and
    F_y + v div(u); div of the mass row = F_mass, for a field that is NOT
    divergence free (pins every Table 1 entry, signs of the viscous terms
    included)."""
    X = _pts(300, (0, 0), (1, 1), seed=13)
    fns = [lambda X: torch.sin(X[:, 0]) * X[:, 1] + X[:, 0] ** 2,
           lambda X: torch.cos(X[:, 1]) * X[:, 0] - X[:, 1] ** 3,
           lambda X: X[:, 0] * X[:, 1] + torch.sin(X[:, 0] + X[:, 1])]
    fl, Xg = _autograd_fields(fns, X)
    re = 7.0
    F = opde.ns_residual(fl, Xg, re)
    D = _div_flux(lambda f, x, n: opde.ns_flux_n(f, x, n, re), fl, Xg)
    div = fl[0]["d1"] + fl[1]["d2"]
    assert torch.allclose(D[:, 0], F[:, 0] + fl[0]["u"] * div, rtol=1e-12, atol=1e-12)
    assert torch.allclose(D[:, 1], F[:, 1] + fl[1]["u"] * div, rtol=1e-12, atol=1e-12)
    assert torch.allclose(D[:, 2], F[:, 2], rtol=1e-12, atol=1e-12)
