"""f4 calibration: train closed-form-solution problems with graph-replayed
pinn_dd_step and log the Eq. (4) stitched relative L2 error (library
classification) against the exact solution.
usage: python tools/train_accuracy.py [name ...]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from pinn_inputs import make_config  # noqa: E402
from pinn_inputs.workloads import kovasznay, burgers_wave  # noqa: E402

CASES = {
    "kovasznay_xpinn": (dict(cfg="C4", method="xpinn", nx=2, ny=2, re=40.0, bc="kovasznay", domain_lo=(-0.5, -0.5),
                             domain_hi=(1.0, 1.5), n_f=2000, n_i=80, n_u=200, lr=1e-3), 6000),
    "kovasznay_cpinn": (dict(cfg="C4", method="cpinn", nx=2, ny=2, re=40.0, bc="kovasznay", domain_lo=(-0.5, -0.5),
                             domain_hi=(1.0, 1.5), n_f=2000, n_i=80, n_u=200, lr=1e-3), 6000),
    "burgers_wave_xpinn": (dict(cfg="C3", method="xpinn", gpus=8, nu=0.05, bc="wave", n_f=2000, n_i=60, n_u=100,
                                lr=2e-3), 6000),
    "burgers_wave_hybrid": (dict(cfg="C3", method="hybrid", gpus=8, nu=0.05, bc="wave", n_f=2000, n_i=60, n_u=100,
                                 lr=2e-3), 6000),
    "burgers_wave_cpinn": (dict(cfg="C1", nu=0.05, bc="wave", n_f=2000, n_i=60, n_u=150, lr=2e-3), 6000),
}


def exact(prob, X):
    if prob.pde == "ns":
        return kovasznay(X, prob.re)[:, :2]
    return burgers_wave(X, prob.nu)[:, None]


def main():
    import __graft_entry__ as ge
    ge.build()
    from paper_2104_10013_b200.binding import PinnDD
    names = sys.argv[1:] or list(CASES)
    for name in names:
        kw, iters = CASES[name]
        kw = dict(kw)
        prob = make_config(kw.pop("cfg"), **kw)
        m = PinnDD(prob, device="cuda:0")
        lo, hi = np.array(prob.domain_lo), np.array(prob.domain_hi)
        g1 = np.linspace(lo[0], hi[0], 61)
        g2 = np.linspace(lo[1], hi[1], 61)
        X = np.stack(np.meshgrid(g1, g2, indexing="ij"), -1).reshape(-1, 2).astype(np.float32)
        ref = exact(prob, X.astype(np.float64))
        pts = torch.tensor(X.T.copy(), device="cuda:0")
        t0 = time.time()
        done = 0
        for stop in (500, 1000, 2000, 3000, 4000, 6000, 8000, 10000):
            if stop > iters:
                break
            out = m.step(stop - done)
            done = stop
            u = m.predict(pts).cpu().numpy().T[:, :ref.shape[1]]
            err = [float(np.linalg.norm(u[:, o] - ref[:, o]) / np.linalg.norm(ref[:, o])) for o in range(ref.shape[1])]
            print(f"{name} it {stop} rel_l2 {['%.4f' % e for e in err]} J {out[:, 4].sum():.3e} "
                  f"t {time.time() - t0:.1f}s", flush=True)
        m.close()


if __name__ == "__main__":
    main()
