"""Eq. (2) feed-forward network with layer-wise adaptive slopes (FP64, CPU).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:93-100: N^1(z) = W^1 z + b^1 and, for 2 <= k <= L,
N^k(z) = W^k Phi(n a^{k-1} N^{k-1}(z)) + b^k, identity activation on the last
layer, W^k in R^{N_k x N_{k-1}}.  Eq. (2) as printed omits the scale n; the text
 says the slope is n*a^k with n = 10 -- reading Z6.
"""

from __future__ import annotations

from typing import List

import torch

from pinn_inputs import param_layout

DT = torch.float64

ACTS = {
    "tanh": torch.tanh,
    "sin": torch.sin,
    "cos": torch.cos,
}


def unpack(theta: torch.Tensor, sizes: List[int]):
    """Split a flat layer-major parameter vector into [(W^k, b^k, a^k or None)]."""
    out = []
    for k, ent in enumerate(param_layout(sizes), start=1):
        o, n = ent["W"]
        W = theta[o:o + n].reshape(sizes[k], sizes[k - 1])
        o, n = ent["b"]
        b = theta[o:o + n]
        a = theta[ent["a"][0]] if "a" in ent else None
        out.append((W, b, a))
    return out


def forward(theta: torch.Tensor, sizes: List[int], X: torch.Tensor,
            activation: str = "tanh", slope_n: float = 10.0) -> torch.Tensor:
    """u_Theta(X) = N^L(X; Theta) for a batch X [n, d_in] -> [n, d_out]."""
    phi = ACTS[activation]
    layers = unpack(theta, sizes)
    h = X
    L = len(layers)
    for k, (W, b, a) in enumerate(layers, start=1):
        z = h @ W.T + b                      # N^k = W^k (.) + b^k
        if k < L:
            h = phi(slope_n * a * z)         # Phi(n a^k N^k), input of layer k+1
        else:
            h = z                            # last layer: identity activation
    return h


def fields(theta: torch.Tensor, sizes: List[int], X: torch.Tensor,
           activation: str = "tanh", slope_n: float = 10.0,
           second=(True, True), create_graph: bool = True):
    """u and its input derivatives by reverse-mode AD.

    Returns a list over outputs o of dicts with keys
    "u", "d1", "d2" (first derivatives wrt x1, x2) and "d11", "d22" (pure
    second derivatives, only those requested in `second`).  Each point's
    output depends only on that point, so the gradient of the batch sum is the
    per-point gradient."""
    X = X.detach().clone().requires_grad_(True)
    u = forward(theta, sizes, X, activation, slope_n)
    out = []
    for o in range(u.shape[1]):
        uo = u[:, o]
        g = torch.autograd.grad(uo.sum(), X, create_graph=True)[0]
        f = {"u": uo, "d1": g[:, 0], "d2": g[:, 1]}
        if second[0]:
            f["d11"] = torch.autograd.grad(g[:, 0].sum(), X, create_graph=True)[0][:, 0]
        if second[1]:
            f["d22"] = torch.autograd.grad(g[:, 1].sum(), X, create_graph=True)[0][:, 1]
        if not create_graph:
            f = {k: v.detach() for k, v in f.items()}
        out.append(f)
    return out, X
