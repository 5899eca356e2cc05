"""Debug: one-step Adam parity along a GPU trajectory (test_train_steps_track_oracle), worst entries."""
import dataclasses, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import loss as OL
from pinn_inputs import make_config, param_layout
import __graft_entry__ as ge
ge.build()
from paper_2104_10013_b200.binding import PinnDD
prob = make_config("C5", scale=0.05, n_i=30, n_u=40)
m = PinnDD(prob, device="cuda:0")
lay = param_layout(prob.sizes)
names = []
for k, ent in enumerate(lay, 1):
    for key in ("W", "b", "a"):
        if key in ent:
            o, n = ent[key]; names += [f"{key}{k}[{i}]" for i in range(n)]
for t in range(10):
    th = [m.get(q, 0).double().cpu() for q in range(prob.n_sub)]
    mm = [m.get(q, 1).double().cpu() for q in range(prob.n_sub)]
    vv = [m.get(q, 2).double().cpu() for q in range(prob.n_sub)]
    cur = dataclasses.replace(prob, subdomains=[dataclasses.replace(sd, params=p.numpy()) for sd, p in zip(prob.subdomains, th)])
    res = OL.loss_grad_all(cur, th)
    m.step(1)
    torch.cuda.synchronize()
    for q in (0, 3):
        bd, g = res[q]
        gg = m.get(q, 3).double().cpu().numpy()
        want, st = OL.adam_step(th[q], g, OL.AdamState(mm[q], vv[q], t), prob.lr, prob.beta1, prob.beta2, prob.eps)
        got = m.get(q, 0).double().cpu().numpy()
        d = np.abs(got - want.numpy())
        i = int(np.argmax(d))
        print(t, q, names[i], "d", d[i], "th", th[q][i].item(), "got", got[i], "want", want[i].item(), "g_or", g[i].item(),
              "g_gpu", gg[i], "m", mm[q][i].item(), "v", vv[q][i].item(), "J", bd.total)
