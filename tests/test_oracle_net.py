"""Pins for oracle/net.py (Eq. 2 network, AD input derivatives).

Each pin is something the oracle's own code cannot fake: SPEC worked examples,
closed-form derivatives of a 1-hidden-layer net, complex-step derivatives of
the forward pass, and finite differences of the AD first derivatives.
"""

import math

import numpy as np
import pytest
import torch

from oracle import net as onet
from pinn_inputs import layer_sizes, n_params, param_layout

DT = torch.float64


def _rand_theta(sizes, seed=0, scale=0.7, slope_n=10.0):
    rng = np.random.default_rng(seed)
    th = rng.standard_normal(n_params(sizes)) * scale
    for ent in param_layout(sizes):
        if "a" in ent:
            th[ent["a"][0]] = (1.0 + 0.3 * rng.standard_normal()) / slope_n
    return torch.tensor(th, dtype=DT)


@pytest.mark.parametrize("sizes,expected", [
    (layer_sizes(2, 20, 3, 1), 924),       # C1
    (layer_sizes(2, 20, 5, 1), 1766),      # C3
    (layer_sizes(2, 40, 6, 1), 8367),      # C2
    (layer_sizes(2, 80, 5, 3), 26408),     # C4: 26403 weights+biases + 5 slopes
])
def test_param_count(sizes, expected):
    assert n_params(sizes) == expected


def test_zero_net_is_zero():
    # SPEC.md:130 "all-zero weights and biases -> output zero"
    sizes = layer_sizes(2, 7, 3, 2)
    th = torch.zeros(n_params(sizes), dtype=DT)
    X = torch.rand(5, 2, dtype=DT)
    assert torch.all(onet.forward(th, sizes, X) == 0)


def test_one_unit_tanh_example():
    # W1=[1], b1=0, W2=[1], b2=0, n a = 1, input 0.5 -> tanh(0.5)
    sizes = [1, 1, 1]
    lay = param_layout(sizes)
    th = torch.zeros(n_params(sizes), dtype=DT)
    th[lay[0]["W"][0]] = 1.0
    th[lay[0]["a"][0]] = 0.1
    th[lay[1]["W"][0]] = 1.0
    u = onet.forward(th, sizes, torch.tensor([[0.5]], dtype=DT), slope_n=10.0)
    assert float(u) == pytest.approx(math.tanh(0.5), abs=1e-15)


def test_slope_neutral_at_init():
    # PAPER.md:95 n a^k = 1 at init -> the plain tanh network (textbook MLP)
    sizes = layer_sizes(2, 9, 3, 2)
    rng = np.random.default_rng(3)
    th = rng.standard_normal(n_params(sizes))
    lay = param_layout(sizes)
    for ent in lay:
        if "a" in ent:
            th[ent["a"][0]] = 0.1
    X = rng.uniform(-1, 1, (11, 2))
    h = X
    for k, ent in enumerate(lay, start=1):
        o, n = ent["W"]
        W = th[o:o + n].reshape(sizes[k], sizes[k - 1])
        o, n = ent["b"]
        h = h @ W.T + th[o:o + n]
        if k < len(lay):
            h = np.tanh(h)
    u = onet.forward(torch.tensor(th), sizes, torch.tensor(X)).numpy()
    np.testing.assert_allclose(u, h, rtol=0, atol=1e-14)


@pytest.mark.parametrize("act", ["tanh", "sin", "cos"])
def test_one_hidden_layer_closed_form_derivatives(act):
    """u = sum_j w2_j s(s_a (w1_j . x + b1_j)) + b2 has closed-form u_x, u_xx."""
    width, slope_n = 6, 10.0
    sizes = [2, width, 1]
    th = _rand_theta(sizes, seed=11)
    lay = param_layout(sizes)
    W1 = th[lay[0]["W"][0]:lay[0]["W"][0] + 2 * width].reshape(width, 2).numpy()
    b1 = th[lay[0]["b"][0]:lay[0]["b"][0] + width].numpy()
    s = slope_n * float(th[lay[0]["a"][0]])
    w2 = th[lay[1]["W"][0]:lay[1]["W"][0] + width].numpy()
    X = np.random.default_rng(5).uniform(-1, 1, (17, 2))
    z = s * (X @ W1.T + b1)
    if act == "tanh":
        t = np.tanh(z); d1 = 1 - t * t; d2 = -2 * t * d1
    elif act == "sin":
        d1 = np.cos(z); d2 = -np.sin(z)
    else:
        d1 = -np.sin(z); d2 = -np.cos(z)
    ux = (d1 * s * W1[:, 0]) @ w2
    uy = (d1 * s * W1[:, 1]) @ w2
    uxx = (d2 * (s * W1[:, 0]) ** 2) @ w2
    uyy = (d2 * (s * W1[:, 1]) ** 2) @ w2
    fl, _ = onet.fields(th, sizes, torch.tensor(X), act, slope_n, create_graph=False)
    for key, ref in (("d1", ux), ("d2", uy), ("d11", uxx), ("d22", uyy)):
        np.testing.assert_allclose(fl[0][key].numpy(), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("act", ["tanh", "sin", "cos"])
def test_first_derivatives_complex_step(act):
    """du/dx_i = Im u(x + i h e_i)/h (h = 1e-30) -- exact to rounding."""
    sizes = layer_sizes(2, 12, 4, 3)
    th = _rand_theta(sizes, seed=2).to(torch.complex128)
    X = torch.tensor(np.random.default_rng(9).uniform(-1, 1, (23, 2)), dtype=DT)
    fl, _ = onet.fields(th.real.clone(), sizes, X, act, 10.0, create_graph=False)
    h = 1e-30
    for i, key in ((0, "d1"), (1, "d2")):
        Xc = X.to(torch.complex128)
        Xc[:, i] += 1j * h
        uc = onet.forward(th, sizes, Xc, act, 10.0)
        cs = uc.imag / h
        for o in range(3):
            np.testing.assert_allclose(fl[o][key].numpy(), cs[:, o].numpy(), rtol=1e-12, atol=1e-13)


def test_second_derivatives_finite_difference():
    """d11/d22 against central differences of the (complex-step-pinned) first
    derivatives and against second differences of the forward value."""
    sizes = layer_sizes(2, 10, 4, 2)
    th = _rand_theta(sizes, seed=4)
    X = torch.tensor(np.random.default_rng(1).uniform(-1, 1, (15, 2)), dtype=DT)
    fl, _ = onet.fields(th, sizes, X, "tanh", 10.0, create_graph=False)
    h = 1e-5
    for i, k1, k2 in ((0, "d1", "d11"), (1, "d2", "d22")):
        e = torch.zeros(2, dtype=DT); e[i] = h
        fp, _ = onet.fields(th, sizes, X + e, "tanh", 10.0, create_graph=False)
        fm, _ = onet.fields(th, sizes, X - e, "tanh", 10.0, create_graph=False)
        for o in range(2):
            fd = (fp[o][k1] - fm[o][k1]) / (2 * h)
            np.testing.assert_allclose(fl[o][k2].numpy(), fd.numpy(), rtol=1e-6, atol=1e-7)
        H = 1e-4
        e = torch.zeros(2, dtype=DT); e[i] = H
        up = onet.forward(th, sizes, X + e); u0 = onet.forward(th, sizes, X); um = onet.forward(th, sizes, X - e)
        fd2 = (up - 2 * u0 + um) / H ** 2
        for o in range(2):
            np.testing.assert_allclose(fl[o][k2].numpy(), fd2[:, o].numpy(), rtol=1e-4, atol=1e-5)


def test_linear_jet_example():
    # SPEC.md:138 "linear network u = 2x + 3t -> u_x = 2, u_xx = 0": a net whose
    # hidden unit works in its linear regime is not linear, so use sin with a
    # zero-weight hidden layer and the output bias path: u = W^L h + b with
    # h = const -> all derivatives 0 (SPEC.md:53 constant case).
    sizes = [2, 3, 1]
    th = torch.zeros(n_params(sizes), dtype=DT)
    lay = param_layout(sizes)
    th[lay[0]["b"][0]:lay[0]["b"][0] + 3] = torch.tensor([0.1, 0.2, 0.3], dtype=DT)
    th[lay[0]["a"][0]] = 0.1
    th[lay[1]["W"][0]:lay[1]["W"][0] + 3] = 1.0
    fl, _ = onet.fields(th, sizes, torch.rand(4, 2, dtype=DT), "tanh", 10.0, create_graph=False)
    for key in ("d1", "d2", "d11", "d22"):
        assert torch.all(fl[0][key] == 0)
    np.testing.assert_allclose(fl[0]["u"].numpy(), np.tanh([0.1, 0.2, 0.3]).sum(), rtol=1e-15)
