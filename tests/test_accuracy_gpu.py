"""f4: training to accuracy against closed-form solutions, with
the Eq. (4) stitched prediction classified by the library.

* Kovasznay flow (exact steady NS solution, Re = 40) on [-0.5, 1] x [-0.5, 1.5]
  with Dirichlet data of (u, v, p), 2 x 2 subdomains, C4's 5 x 80 network,
  XPINN and cPINN (PAPER.md:413-434 solve NS this way; the cavity of C4 has no
  closed form).
* The viscous Burgers travelling wave u = c - a tanh(a (x - c t) / (2 nu))
  (nu = 0.05, a = 0.5, c = 0.2) on [-1, 1] x [0, 1] with its initial and
  boundary data: C3's 4 x 2 x-t XPINN and hybrid (cPINN in x, XPINN in t,
  P:948) with 5 x 20 networks, and C1's 2 x 1 cPINN with 3 x 20 networks
  (PAPER.md:313-316, 778-816).

Calibration (tools/train_accuracy.py, profiles/r02_train_accuracy.log): after
6000 graph-replayed iterations the relative L2 errors are u 1.2 % / v 7.1 %
(Kovasznay XPINN), 1.3 % / 5.3 % (cPINN), 1.5 % (Burgers XPINN), 0.12 %
(hybrid), 0.09 % (cPINN); the thresholds leave ~2x margin."""

import numpy as np
import pytest
import torch

from pinn_inputs import make_config
from pinn_inputs.workloads import burgers_wave, kovasznay

pytestmark = pytest.mark.gpu

KOV = dict(re=40.0, bc="kovasznay", domain_lo=(-0.5, -0.5), domain_hi=(1.0, 1.5), nx=2, ny=2, n_f=2000,
           n_i=80, n_u=200, lr=1e-3)
WAVE = dict(nu=0.05, bc="wave", n_f=2000, n_i=60, lr=2e-3)

CASES = [
    ("C4", dict(method="xpinn", **KOV), (0.03, 0.15)),
    ("C4", dict(method="cpinn", **KOV), (0.03, 0.12)),
    ("C3", dict(method="xpinn", gpus=8, n_u=100, **WAVE), (0.04,)),
    ("C3", dict(method="hybrid", gpus=8, n_u=100, **WAVE), (0.02,)),
    ("C1", dict(n_u=150, **WAVE), (0.02,)),
]


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()


@pytest.mark.parametrize("cfg,kw,thresholds", CASES)
def test_train_to_closed_form(cfg, kw, thresholds):
    from paper_2104_10013_b200.binding import PinnDD
    prob = make_config(cfg, **kw)
    m = PinnDD(prob, device="cuda:0")
    lo, hi = np.array(prob.domain_lo), np.array(prob.domain_hi)
    g = [np.linspace(lo[i], hi[i], 61) for i in range(2)]
    X = np.stack(np.meshgrid(*g, indexing="ij"), -1).reshape(-1, 2).astype(np.float32)
    Xd = X.astype(np.float64)
    ref = kovasznay(Xd, prob.re)[:, :2] if prob.pde == "ns" else burgers_wave(Xd, prob.nu)[:, None]
    pts = torch.tensor(X.T.copy(), device="cuda:0")

    def errs():
        u = m.predict(pts).cpu().numpy().T
        return [np.linalg.norm(u[:, o] - ref[:, o]) / np.linalg.norm(ref[:, o]) for o in range(ref.shape[1])]

    e0 = errs()
    m.step(6000, want_loss=False)
    e = errs()
    assert m.adam_t(0) == 6000
    for o, (a, b, t) in enumerate(zip(e0, e, thresholds)):
        assert b < t and b < 0.2 * a, (cfg, kw["method"] if "method" in kw else "cpinn", o, a, b)
    m.close()
