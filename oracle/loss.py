"""Subdomain losses Eq. (3)/(5)/(6), gradients, Adam, Algorithm 1 step, Eq. (4).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings:
* Z1  -- {{u}} = (u_q + u_{q+})/2 is written out literally; u_q inside the
         average is differentiated, u_{q+} is a constant.
* Z2  -- the 1/N_{I_q} is a per-edge mean, summed over live edges q+
         (PAPER.md:158-159, 175-176).
* Z3  -- one canonical normal per edge, used on both sides.
* Z4  -- systems: per-field squared errors are summed.
* Z11 -- Adam in the Kingma-Ba form, beta = (0.9, 0.999), eps = 1e-8
         (SPEC.md:565-568).
* Z12 -- one Adam step per exchange; neighbour payloads come from the
         parameters at the start of the iteration.
* Z14 -- interface points enter only the interface terms; MSE_u = 0 when a
         subdomain has no training points.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import net as onet
from . import pde as opde

DT = torch.float64


def _t(a) -> torch.Tensor:
    return torch.as_tensor(np.asarray(a), dtype=DT)


def _mse_sum(r: torch.Tensor) -> torch.Tensor:
    """(1/N) sum_i sum_fields |r_i|^2 ; 0 for an empty set."""
    if r.shape[0] == 0:
        return torch.zeros((), dtype=DT)
    return (r * r).sum() / r.shape[0]


def _act(prob, q):
    """Activation of subdomain q (per region in C5, Table 3)."""
    return prob.act(q) if q is not None else prob.activation


def eval_fields(prob, theta, X, create_graph=True, q=None):
    fl, Xg = onet.fields(theta, prob.sizes, X, _act(prob, q), prob.slope_n,
                         second=opde.SECOND[prob.pde], create_graph=create_graph)
    return fl, Xg


def uses_flux(prob, normal) -> bool:
    """Interface condition of an edge: cPINN -> normal-flux continuity
    (Eq. 5); XPINN -> residual continuity (Eq. 6); hybrid (PAPER.md:948,
    "cPINN in space + XPINN in time") -> flux on x1-normal edges, residual on
    x2-normal (time) edges."""
    if prob.method == "cpinn":
        return True
    if prob.method == "hybrid":
        return normal[1] == 0.0
    return False


def interface_payload(prob, theta, X, normal, create_graph=True, q=None):
    """What subdomain q sends for one edge (Algorithm 1):
    u(x_I) [n, d_out] and f(x_I).n (cPINN) or F(x_I) (XPINN) [n, n_eq]."""
    fl, Xg = eval_fields(prob, theta, X, create_graph, q)
    u = torch.stack([f["u"] for f in fl], dim=1)
    if uses_flux(prob, normal):
        s = opde.flux_n(prob, fl, Xg, normal)
    else:
        s = opde.residual(prob, fl, Xg)
    if not create_graph:
        u, s = u.detach(), s.detach()
    return u, s


@dataclass
class Breakdown:
    mse_u: float
    mse_f: float
    mse_uavg: float
    mse_if: float        # MSE_flux (cPINN) or MSE_R (XPINN)
    total: float

    def as_list(self):
        return [self.mse_u, self.mse_f, self.mse_uavg, self.mse_if, self.total]


def subdomain_loss(prob, q: int, thetas: Sequence[torch.Tensor],
                   payloads: Optional[Dict] = None):
    """J(Theta_q) of Eq. (5) (cPINN) or Eq. (6) (XPINN); Eq. (3) if q has no
    live interface.  `thetas[q]` may require grad; every neighbour quantity is
    computed from the neighbour's parameters and detached."""
    if prob.method == "cpinn":
        for e in prob.subdomains[q].edges:
            if prob.edges[e].axis == 1 and prob.pde == "burgers":
                raise ValueError("cPINN with a time-axis interface (PAPER.md:816; SPEC.md:689)")
    s = prob.subdomains[q]
    th = thetas[q]
    # MSE_F : residual points
    X_f = _t(s.x_f)
    if len(X_f):
        fl, Xg = eval_fields(prob, th, X_f, q=q)
        mse_f = _mse_sum(opde.residual(prob, fl, Xg))
    else:
        mse_f = torch.zeros((), dtype=DT)
    # MSE_u : training points, masked outputs
    if len(s.x_u):
        u = onet.forward(th, prob.sizes, _t(s.x_u), _act(prob, q), prob.slope_n)
        mse_u = _mse_sum(_t(s.u_mask) * (_t(s.u_target) - u))
    else:
        mse_u = torch.zeros((), dtype=DT)
    # interface terms, per edge mean, summed over q+ (Z2)
    mse_uavg = torch.zeros((), dtype=DT)
    mse_if = torch.zeros((), dtype=DT)
    for e in s.edges:
        ed = prob.edges[e]
        nb = prob.edge_neighbor(q, e)
        X_i = _t(ed.pts)
        u_q, s_q = interface_payload(prob, th, X_i, ed.normal, q=q)
        if payloads is not None:
            u_n, s_n = payloads[(nb, e)]
        else:
            u_n, s_n = interface_payload(prob, thetas[nb].detach(), X_i, ed.normal,
                                         create_graph=False, q=nb)
        uavg = 0.5 * (u_q + u_n)                      # {{u}}
        mse_uavg = mse_uavg + _mse_sum(u_q - uavg)
        mse_if = mse_if + _mse_sum(s_q - s_n)
    total = prob.w_u * mse_u + prob.w_f * mse_f + prob.w_i * mse_uavg + prob.w_if * mse_if
    return total, (mse_u, mse_f, mse_uavg, mse_if)


def subdomain_loss_terms(prob, q: int, thetas: Sequence[torch.Tensor], chunk: int = 8192):
    """The four MSE terms and J of subdomain q (same definitions as
    `subdomain_loss`), evaluated in point chunks without a parameter graph, for
    full-size problems.  Sums of squares are accumulated in float64."""
    s = prob.subdomains[q]
    th = thetas[q].detach()
    sq = torch.zeros((), dtype=DT)
    X_f = _t(s.x_f)
    for i in range(0, len(X_f), chunk):
        fl, Xg = eval_fields(prob, th, X_f[i:i + chunk], create_graph=False, q=q)
        r = opde.residual(prob, fl, Xg).detach()
        sq = sq + (r * r).sum()
    mse_f = sq / len(X_f) if len(X_f) else torch.zeros((), dtype=DT)
    with torch.no_grad():
        if len(s.x_u):
            u = onet.forward(th, prob.sizes, _t(s.x_u), _act(prob, q), prob.slope_n)
            mse_u = _mse_sum(_t(s.u_mask) * (_t(s.u_target) - u))
        else:
            mse_u = torch.zeros((), dtype=DT)
    mse_uavg = torch.zeros((), dtype=DT)
    mse_if = torch.zeros((), dtype=DT)
    for e in s.edges:
        ed = prob.edges[e]
        nb = prob.edge_neighbor(q, e)
        X_i = _t(ed.pts)
        u_q, s_q = interface_payload(prob, th, X_i, ed.normal, create_graph=False, q=q)
        u_n, s_n = interface_payload(prob, thetas[nb].detach(), X_i, ed.normal, create_graph=False,
                                     q=nb)
        mse_uavg = mse_uavg + _mse_sum(u_q - 0.5 * (u_q + u_n))
        mse_if = mse_if + _mse_sum(s_q - s_n)
    total = prob.w_u * mse_u + prob.w_f * mse_f + prob.w_i * mse_uavg + prob.w_if * mse_if
    return Breakdown(float(mse_u), float(mse_f), float(mse_uavg), float(mse_if), float(total))


def loss_and_grad(prob, q: int, thetas: Sequence[torch.Tensor], payloads=None):
    th = thetas[q].detach().clone().requires_grad_(True)
    ths = list(thetas)
    ths[q] = th
    J, parts = subdomain_loss(prob, q, ths, payloads)
    (g,) = torch.autograd.grad(J, th)
    bd = Breakdown(*[float(p.detach()) for p in parts], float(J.detach()))
    return bd, g.detach()


def all_payloads(prob, thetas):
    """Every (subdomain, edge) payload from the current parameters (Z12)."""
    pay = {}
    for e, ed in enumerate(prob.edges):
        for q in (ed.a, ed.b):
            pay[(q, e)] = interface_payload(prob, thetas[q].detach(), _t(ed.pts), ed.normal,
                                            create_graph=False, q=q)
    return pay


def loss_grad_all(prob, thetas):
    """Per-subdomain (Breakdown, gradient) for the whole decomposition."""
    pay = all_payloads(prob, thetas)
    return [loss_and_grad(prob, q, thetas, pay) for q in range(prob.n_sub)]


# --------------------------------------------------------------------------
# Adam (Kingma & Ba)
# --------------------------------------------------------------------------

@dataclass
class AdamState:
    m: torch.Tensor
    v: torch.Tensor
    t: int


def adam_init(theta: torch.Tensor) -> AdamState:
    return AdamState(torch.zeros_like(theta), torch.zeros_like(theta), 0)


def adam_step(theta, g, st: AdamState, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    t = st.t + 1
    m = beta1 * st.m + (1.0 - beta1) * g
    v = beta2 * st.v + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** t)
    v_hat = v / (1.0 - beta2 ** t)
    theta = theta - lr * m_hat / (torch.sqrt(v_hat) + eps)
    return theta, AdamState(m, v, t)


@dataclass
class TrainState:
    thetas: List[torch.Tensor]
    adam: List[AdamState]


def init_state(prob) -> TrainState:
    th = [_t(s.params) for s in prob.subdomains]
    return TrainState(th, [adam_init(t) for t in th])


def train_step(prob, st: TrainState):
    """Algorithm 1, one epoch: payloads from the current
    parameters, J_q and its gradient per subdomain, one Adam step each."""
    res = loss_grad_all(prob, st.thetas)
    new_th, new_ad = [], []
    for q, (bd, g) in enumerate(res):
        th, ad = adam_step(st.thetas[q], g, st.adam[q], prob.lr, prob.beta1, prob.beta2, prob.eps)
        new_th.append(th)
        new_ad.append(ad)
    return TrainState(new_th, new_ad), [bd for bd, _ in res]


# --------------------------------------------------------------------------
# Eq. (4) stitched solution
# --------------------------------------------------------------------------

def owners(prob, X: np.ndarray) -> List[List[int]]:
    """Subdomains whose closed cell contains each point."""
    out = []
    for x in np.asarray(X):
        o = [s.id for s in prob.subdomains
             if s.lo[0] <= x[0] <= s.hi[0] and s.lo[1] <= x[1] <= s.hi[1]]
        out.append(o)
    return out


def stitch(prob, thetas, X: np.ndarray) -> torch.Tensor:
    """u(z) = sum_q u_q(z) 1_{Omega_q}(z), indicator 1 inside, 1/S on an
    interface shared by S subdomains, 0 outside."""
    Xt = _t(X)
    own = owners(prob, X)
    u = torch.zeros((len(X), prob.d_out), dtype=DT)
    for q in range(prob.n_sub):
        w = torch.tensor([1.0 / len(o) if q in o else 0.0 for o in own], dtype=DT)
        if float(w.abs().sum()) == 0.0:
            continue
        uq = onet.forward(thetas[q].detach(), prob.sizes, Xt, _act(prob, q), prob.slope_n)
        u = u + w[:, None] * uq
    return u
