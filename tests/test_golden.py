"""Golden fixtures: the oracle against worked examples printed in SPEC.md and
PAPER.md Table 1 (tests/golden/spec_worked_examples.json, each entry cited).

Every expected value in the fixture is the printed one (or the printed
arithmetic carried out); none comes from oracle/ or the CUDA path."""

import json
import math
import os
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import loss as oloss
from oracle import net as onet
from oracle import pde as opde
from pinn_inputs import n_params, param_layout
from pinn_inputs.workloads import xavier_params

DT = torch.float64
_HERE = os.path.dirname(__file__)
with open(os.path.join(_HERE, "golden", "spec_worked_examples.json")) as _f:
    EXAMPLES = json.load(_f)["examples"]


def _x(ex):
    x = np.array([[0.0 if v is None else v for v in r] for r in ex["x"]], dtype=np.float64)
    return torch.tensor(x, dtype=DT)


def _theta(ex):
    sizes = ex["sizes"]
    lay = param_layout(sizes)
    th = torch.zeros(n_params(sizes), dtype=DT)
    for k, ent in enumerate(lay):
        if "a" in ent:
            th[ent["a"][0]] = ex["a"][k]
        if not ex.get("zero"):
            o, n = ent["W"]
            th[o:o + n] = torch.tensor(ex["W"][k], dtype=DT).reshape(-1)
            o, n = ent["b"]
            th[o:o + n] = torch.tensor(ex["b"][k], dtype=DT)
    return th


def _field(spec, X):
    """Closed-form field dict: numbers are constants, strings name x-expressions."""
    x = X[:, 0]
    expr = {"x": x, "x2": x * x, "2x": 2 * x}
    return {k: (expr[v] if isinstance(v, str) else torch.full_like(x, float(v)))
            for k, v in spec.items()}


def _fields(ex, X):
    f = ex["fields"]
    return [_field(s, X) for s in (f if isinstance(f, list) else [f])]


def _stitch_problem(ex):
    nx, ny = ex["grid"]
    lo, hi = ex["lo"], ex["hi"]
    dx, dy = (hi[0] - lo[0]) / nx, (hi[1] - lo[1]) / ny
    subs = []
    for j in range(ny):
        for i in range(nx):
            q = j * nx + i
            subs.append(SimpleNamespace(id=q, lo=(lo[0] + i * dx, lo[1] + j * dy),
                                        hi=(lo[0] + (i + 1) * dx, lo[1] + (j + 1) * dy),
                                        activation=None))
    prob = SimpleNamespace(subdomains=subs, n_sub=len(subs), d_out=1, sizes=[2, 3, 1],
                           slope_n=10.0, activation="tanh")
    prob.act = lambda q: "tanh"
    # constant networks u_q = values[q]: random hidden layer, W^L = 0, b^L = c
    lay = param_layout(prob.sizes)
    thetas = []
    rng = np.random.default_rng(0)
    for c in ex["values"]:
        th = torch.tensor(xavier_params(prob.sizes, 10.0, rng), dtype=DT)
        o, n = lay[-1]["W"]
        th[o:o + n] = 0.0
        th[lay[-1]["b"][0]] = c
        thetas.append(th)
    return prob, thetas


@pytest.mark.parametrize("ex", EXAMPLES, ids=[e["id"] for e in EXAMPLES])
def test_golden_example(ex):
    op = ex["op"]
    if op == "forward":
        u = onet.forward(_theta(ex), ex["sizes"], _x(ex)[:, :ex["sizes"][0]],
                         "tanh", ex["slope_n"])
        assert torch.allclose(u[:, 0], torch.tensor(ex["expected"], dtype=DT), rtol=1e-15, atol=0)
    elif op == "fields":
        fl, _ = onet.fields(_theta(ex), ex["sizes"], _x(ex), "tanh", ex["slope_n"],
                            create_graph=False)
        for k, v in ex["expected"].items():
            assert torch.all(fl[0][k] == v), k
    elif op == "param_count":
        sizes = ex["sizes"]
        lay = param_layout(sizes)
        n_slopes = sum("a" in e for e in lay)
        assert n_slopes == ex["expected_slopes"]
        assert n_params(sizes) - n_slopes == ex["expected_wb"]
        # the oracle's unpack consumes exactly that vector
        parts = onet.unpack(torch.zeros(n_params(sizes), dtype=DT), sizes)
        assert sum(W.numel() + b.numel() for W, b, _ in parts) == ex["expected_wb"]
        assert sum(a is not None for _, _, a in parts) == ex["expected_slopes"]
    elif op == "init_slope":
        th = xavier_params(ex["sizes"], ex["slope_n"], np.random.default_rng(1))
        parts = onet.unpack(torch.tensor(th, dtype=DT), ex["sizes"])
        for _, _, a in parts[:-1]:
            assert float(a) == pytest.approx(ex["expected"], rel=2 ** -24)   # stored as FP32
    elif op == "burgers_residual":
        X = _x(ex)
        F = opde.burgers_residual(_fields(ex, X), X, ex["nu"])
        assert torch.allclose(F[:, 0], torch.tensor(ex["expected"], dtype=DT), rtol=0, atol=1e-15)
    elif op == "burgers_flux":
        X = _x(ex)
        f = opde.burgers_flux_n(_fields(ex, X), X, tuple(ex["n"]), ex["nu"])
        assert torch.all(f[:, 0] == torch.tensor(ex["expected"], dtype=DT))
    elif op == "ns_residual":
        X = _x(ex)
        F = opde.ns_residual(_fields(ex, X), X, ex["re"])
        assert torch.all(F == torch.tensor([ex["expected"]], dtype=DT))
    elif op == "ns_flux":
        X = _x(ex)
        f = opde.ns_flux_n(_fields(ex, X), X, tuple(ex["n"]), ex["re"])
        if "expected" in ex:
            assert torch.all(f == torch.tensor([ex["expected"]], dtype=DT))
        else:
            assert float(f[0, ex["expected_index"]]) == ex["expected_component"]
    elif op == "heat_K":
        K, _, _ = opde.heat_K(_x(ex))
        assert torch.allclose(K, torch.tensor(ex["expected"], dtype=DT), rtol=1e-15, atol=0)
    elif op == "heat_inv_residual":
        X = _x(ex)
        F = opde.heat_inv_residual(_fields(ex, X), X)
        f = 4.0 * torch.exp(-0.1 * X[:, 1])          # PAPER.md:828-829 forcing of the exact pair
        assert torch.allclose(F[:, 0], ex["expected_minus_forcing"] - f, rtol=1e-15, atol=1e-15)
    elif op == "mse":
        r = torch.tensor(ex["residuals"], dtype=DT).reshape(-1, 1)
        assert float(oloss._mse_sum(r)) == ex["expected"]
    elif op == "stitch":
        prob, thetas = _stitch_problem(ex)
        u = oloss.stitch(prob, thetas, np.array(ex["x"], dtype=np.float64))
        assert torch.allclose(u[:, 0], torch.tensor(ex["expected"], dtype=DT), rtol=1e-14, atol=0)
    else:
        raise AssertionError(f"unknown golden op {op}")


def test_every_golden_example_is_cited():
    for ex in EXAMPLES:
        assert "SPEC.md:" in ex["cite"] or "PAPER.md:" in ex["cite"], ex["id"]
