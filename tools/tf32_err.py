"""TF32 tensor-core mode (PINN_DD_FLAG_TF32) vs the FP64 oracle and vs the FP32
kernel: relative errors of every loss term and per-tensor gradient errors."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import loss as OL
from pinn_inputs import make_config, param_layout, perturb_params
import __graft_entry__ as ge
ge.build()
from paper_2104_10013_b200.binding import PinnDD, FLAG_GRAPH, FLAG_TF32

CASES = [("C4", dict(method="xpinn", n_f=150, n_i=20, n_u=16)), ("C4", dict(method="cpinn", n_f=150, n_i=20, n_u=16)),
         ("C4", dict(method="xpinn", n_f=2000, n_i=64, n_u=40)), ("C5", dict(scale=0.1, n_i=24, n_u=40)),
         ("C5", dict(scale=0.05, n_i=24, n_u=40, activations=["cos"] * 10))]
for cfg, kw in CASES:
    for pert in (0.0, 0.2):
        prob = make_config(cfg, **kw)
        if pert:
            prob = perturb_params(prob, scale=pert)
        th = OL.init_state(prob).thetas
        ref = OL.loss_grad_all(prob, th)
        out = {}
        for name, fl in (("fp32", FLAG_GRAPH), ("tf32", FLAG_GRAPH | FLAG_TF32)):
            m = PinnDD(prob, device="cuda:0", flags=fl)
            m.interface_payload()
            loss, grad = m.loss_grad()
            torch.cuda.synchronize()
            out[name] = (loss.cpu().numpy(), grad.double().cpu().numpy())
            m.close()
        lay = param_layout(prob.sizes)
        for name, (l, g) in out.items():
            lrel = [max(abs(l[q, i] - bd.as_list()[i]) / max(abs(bd.as_list()[i]), 1e-300) for q, (bd, _) in enumerate(ref))
                    for i in range(5)]
            grel = 0.0
            arel = 0.0
            for q, (_, gr) in enumerate(ref):
                gr = gr.numpy()
                for ent in lay:
                    for key in ("W", "b"):
                        o, n = ent[key]
                        den = np.abs(gr[o:o + n]).max()
                        if den > 0:
                            grel = max(grel, np.abs(g[q, o:o + n] - gr[o:o + n]).max() / den)
                    if "a" in ent:
                        oa = ent["a"][0]
                        arel = max(arel, abs(g[q, oa] - gr[oa]) / abs(gr[oa]))
            print(json.dumps(dict(case=f"{cfg}{kw}", pert=pert, mode=name, loss_rel=[float(x) for x in lrel],
                                  grad_rel=float(grel), slope_rel=float(arel))), flush=True)
