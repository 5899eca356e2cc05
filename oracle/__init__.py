"""FP64 CPU ORACLE for the parallel cPINN / XPINN training step (arXiv 2104.10013).

*** TEST INFRASTRUCTURE ONLY. ***  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import or execute
anything in this package.  The product path (`paper_2104_10013_b200/`) never
imports it, and it never imports the product path; the two share only the
seeded input generator `pinn_inputs` (which holds none of the method's
arithmetic).

What it computes is the plain definition of the paper's quantities, in float64,
with plain PyTorch CPU ops:

* `net`    -- Eq. (2) feed-forward net with layer-wise adaptive slope n*a^k
              (PAPER.md:93-103).
* `pde`    -- residuals F := L_x(u) - f of Burgers
              (Eq. 10/14), Poisson / heat (Eq. 15,
              PAPER.md:823-829) and 2-D steady NS (Eq. 11);
              normal fluxes of Table 1.
* `loss`   -- Eq. (3) PINN, Eq. (5) cPINN and Eq. (6) XPINN subdomain losses
              (PAPER.md:110-119, 149-177), their gradients, Adam,
              Algorithm 1's synchronous step and the Eq. (4)
              stitched solution.

Input derivatives u_x, u_xx, ... are obtained the way the paper obtains them:
reverse-mode automatic differentiation through the computational graph
 -- `torch.autograd.grad` with `create_graph=True`.  The
CUDA path instead propagates forward Taylor jets, so the two agree only if
both are right.  Parameter gradients are reverse-mode AD of J_q with every
neighbour quantity held constant.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): closed-form 1-hidden-layer
derivatives, complex-step and finite differences, exact PDE solutions
(Cole-Hopf travelling wave, u = x/(t+1), sin*sin Poisson, the paper's heat
fields, Kovasznay flow), Table 1 columns, the SPEC worked loss examples,
structural invariants (N_sd = 1 degeneracy, identical neighbours, symmetric
mismatch), finite-difference gradients and closed-form Adam steps.  No
function here is "parity unpinned".
"""

from . import net, pde, loss  # noqa: F401
