"""Diagnostic: per-tensor gradient errors of the CUDA path vs the FP64 oracle,
including the slope gradients a^k, for the parity cases (and optionally at a
trained state).  Prints one JSON line per (case, subdomain) with the worst
W/b error, each a^k relative error and its cancellation ratio
R = (sum|W dJ/dW| + sum|b dJ/db|) / |a dJ/da|."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import loss as OL  # noqa: E402
from pinn_inputs import make_config, param_layout, perturb_params  # noqa: E402

CASES = [
    ("C1", dict()), ("C1", dict(n_f=333, n_i=17, n_u=29)),
    ("C2", dict(method="cpinn", n_f=300, n_i=25, n_u=20)),
    ("C2", dict(method="xpinn", n_f=300, n_i=25, n_u=20)),
    ("C2", dict(method="cpinn", pde="heat", n_f=200, n_i=20, n_u=20)),
    ("C3", dict(method="xpinn", gpus=8, n_f=400, n_i=30, n_u=40)),
    ("C4", dict(method="xpinn", n_f=150, n_i=20, n_u=16)),
    ("C4", dict(method="cpinn", n_f=150, n_i=20, n_u=16)),
    ("C5", dict(scale=0.02, n_i=24, n_u=40)),
    ("C5", dict(scale=0.02, n_i=24, n_u=40, activations=["cos"] * 10)),
]


def report(tag, prob, grad, th, ref):
    lay = param_layout(prob.sizes)
    out = []
    for q, (_, g) in enumerate(ref):
        gg = grad[q].double().cpu().numpy()
        gr = g.numpy()
        t = th[q].numpy()
        wb = 0.0
        arel, R = [], []
        for ent in lay:
            for key in ("W", "b"):
                o, n = ent[key]
                den = np.max(np.abs(gr[o:o + n]))
                if den > 1e-30:
                    wb = max(wb, np.max(np.abs(gg[o:o + n] - gr[o:o + n])) / den)
            if "a" in ent:
                (ow, nw), (ob, nb), (oa, _) = ent["W"], ent["b"], ent["a"]
                arel.append(abs(gg[oa] - gr[oa]) / max(abs(gr[oa]), 1e-300))
                gross = np.abs(t[ow:ow + nw] * gr[ow:ow + nw]).sum() + np.abs(t[ob:ob + nb] * gr[ob:ob + nb]).sum()
                R.append(gross / max(abs(t[oa] * gr[oa]), 1e-300))
        out.append(dict(case=tag, q=q, wb=wb, a_rel=arel, R=R))
    return out


def main():
    import __graft_entry__ as ge
    ge.build()
    from paper_2104_10013_b200.binding import PinnDD
    res = []
    for cfg, kw in CASES:
        for pert in (0.0, 0.2):
            prob = make_config(cfg, **kw)
            if pert:
                prob = perturb_params(prob, scale=pert)
            m = PinnDD(prob, device="cuda:0")
            m.interface_payload()
            loss, grad = m.loss_grad()
            torch.cuda.synchronize()
            th = OL.init_state(prob).thetas
            ref = OL.loss_grad_all(prob, th)
            for r in report(f"{cfg}{kw} p{pert}", prob, grad, th, ref):
                print(json.dumps(r), flush=True)
                res.append(r)
            m.close()
    worst = max(max(r["a_rel"]) for r in res)
    print("WORST a_rel", worst, "WORST wb", max(r["wb"] for r in res))


if __name__ == "__main__":
    main()
