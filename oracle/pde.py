"""PDE residuals F := L_x(u; lambda) - f and interface fluxes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

All functions are pointwise in the field values: they take the list of per-output
dicts produced by `oracle.net.fields` (or closed-form fields built by a test)
plus the coordinates X [n, 2], and return a tensor [n, n_eq].

Coordinates: x1 = x, x2 = t for Burgers ("time t as one of the
components of x"), x2 = y otherwise.
"""

from __future__ import annotations

import math

import torch

# which pure second derivatives each operator needs (d11, d22)
SECOND = {
    "burgers": (True, False),
    "poisson": (True, True),
    "heat": (True, True),
    "ns": (True, True),
    "heat_inv": (True, True),
}

N_EQ = {"burgers": 1, "poisson": 1, "heat": 1, "ns": 3, "heat_inv": 1}


# --------------------------------------------------------------------------
# Burgers, Eq. (10)/(14): u_t + u u_x - nu u_xx = 0
# --------------------------------------------------------------------------

def burgers_residual(fl, X, nu):
    u = fl[0]
    return (u["d2"] + u["u"] * u["d1"] - nu * u["d11"])[:, None]


def burgers_flux_n(fl, X, n, nu):
    """Conservative space-time flux of Eq. (10), (u^2/2 - nu u_x, u), dotted with n.

    The paper never prints the Burgers flux; u^2/2 - nu u_x is the x-flux of
    the conservation form u_t + (u^2/2 - nu u_x)_x = 0 (reading Z13).  cPINN is
    only used with x-normal interfaces, where this is
    (u^2/2 - nu u_x) n_x."""
    u = fl[0]
    fx = 0.5 * u["u"] * u["u"] - nu * u["d1"]
    ft = u["u"]
    return (fx * n[0] + ft * n[1])[:, None]


# --------------------------------------------------------------------------
# Poisson / heat, Eq. (15): d_x(K T_x) + d_y(K T_y) = f
# --------------------------------------------------------------------------

def poisson_forcing(X):
    """f for the manufactured solution u* = sin(pi x) sin(pi y) (reading Z15)."""
    return -2.0 * math.pi ** 2 * torch.sin(math.pi * X[:, 0]) * torch.sin(math.pi * X[:, 1])


def heat_K(X):
    """K(x, y) = 20 + exp(0.1 y) sin(0.5 x) and its gradient."""
    x, y = X[:, 0], X[:, 1]
    e = torch.exp(0.1 * y)
    return 20.0 + e * torch.sin(0.5 * x), 0.5 * e * torch.cos(0.5 * x), 0.1 * e * torch.sin(0.5 * x)


def heat_forcing(X):
    """f = div(K grad T*) for T* = 20 exp(-0.1 y): f = 4 exp(-0.1 y)."""
    return 4.0 * torch.exp(-0.1 * X[:, 1])


def poisson_residual(fl, X):
    u = fl[0]
    return (u["d11"] + u["d22"] - poisson_forcing(X))[:, None]


def poisson_flux_n(fl, X, n):
    u = fl[0]
    return (u["d1"] * n[0] + u["d2"] * n[1])[:, None]


def heat_residual(fl, X):
    """d_x(K u_x) + d_y(K u_y) - f expanded by the product rule."""
    u = fl[0]
    K, Kx, Ky = heat_K(X)
    return (K * (u["d11"] + u["d22"]) + Kx * u["d1"] + Ky * u["d2"] - heat_forcing(X))[:, None]


def heat_flux_n(fl, X, n):
    u = fl[0]
    K, _, _ = heat_K(X)
    return (K * (u["d1"] * n[0] + u["d2"] * n[1]))[:, None]


# --------------------------------------------------------------------------
# Inverse heat conduction, Eq. (15) with K unknown: one net
# per region with outputs (T, K) (reading Z17'), F = d_x(K T_x) + d_y(K T_y) - f
# with both T and K from the net, f = 4 exp(-0.1 y) of the exact pair
# T* = 20 exp(-0.1 y), K* = 20 + exp(0.1 y) sin(0.5 x).
# --------------------------------------------------------------------------

def heat_inv_residual(fl, X):
    T, K = fl
    return (K["u"] * (T["d11"] + T["d22"]) + K["d1"] * T["d1"] + K["d2"] * T["d2"]
            - heat_forcing(X))[:, None]


def heat_inv_flux_n(fl, X, n):
    T, K = fl
    return (K["u"] * (T["d1"] * n[0] + T["d2"] * n[1]))[:, None]


# --------------------------------------------------------------------------
# Steady incompressible NS, Eq. (11) and Table 1 fluxes
# --------------------------------------------------------------------------

def ns_residual(fl, X, re):
    u, v, p = fl
    lap_u = u["d11"] + u["d22"]
    lap_v = v["d11"] + v["d22"]
    fx = u["u"] * u["d1"] + v["u"] * u["d2"] + p["d1"] - lap_u / re
    fy = u["u"] * v["d1"] + v["u"] * v["d2"] + p["d2"] - lap_v / re
    div = u["d1"] + v["d2"]
    return torch.stack([fx, fy, div], dim=1)


def ns_flux_n(fl, X, n, re):
    """Table 1 dotted with the canonical edge normal."""
    u, v, p = fl
    U, V, P = u["u"], v["u"], p["u"]
    xm = (U * U + P - u["d1"] / re) * n[0] + (U * V - u["d2"] / re) * n[1]
    ym = (U * V - v["d1"] / re) * n[0] + (V * V + P - v["d2"] / re) * n[1]
    ms = U * n[0] + V * n[1]
    return torch.stack([xm, ym, ms], dim=1)


# --------------------------------------------------------------------------
# dispatch
# --------------------------------------------------------------------------

def residual(prob, fl, X):
    if prob.pde == "burgers":
        return burgers_residual(fl, X, prob.nu)
    if prob.pde == "poisson":
        return poisson_residual(fl, X)
    if prob.pde == "heat":
        return heat_residual(fl, X)
    if prob.pde == "ns":
        return ns_residual(fl, X, prob.re)
    if prob.pde == "heat_inv":
        return heat_inv_residual(fl, X)
    raise ValueError(prob.pde)


def flux_n(prob, fl, X, n):
    if prob.pde == "burgers":
        return burgers_flux_n(fl, X, n, prob.nu)
    if prob.pde == "poisson":
        return poisson_flux_n(fl, X, n)
    if prob.pde == "heat":
        return heat_flux_n(fl, X, n)
    if prob.pde == "ns":
        return ns_flux_n(fl, X, n, prob.re)
    if prob.pde == "heat_inv":
        return heat_inv_flux_n(fl, X, n)
    raise ValueError(prob.pde)
