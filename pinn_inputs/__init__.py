"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no network evaluation, no
derivative, no residual, no loss, no optimiser).  It only produces the
*inputs* of the paper's pre-processing stage (Algorithm 1, blue block,
PAPER.md:225-232 / Sec. 5.1):

* the Cartesian decomposition of the domain into non-overlapping subdomains,
* the residual, training (boundary/initial) and interface point sets of every
  subdomain, with the boundary/initial target values the paper prescribes,
* the seeded initial network parameters (Xavier-uniform W, zero b, a = 1/n;
  PAPER.md:95, 103).

Both `oracle/` and `paper_2104_10013_b200/` import it; neither imports the
other.  Every float it emits is exactly representable in float32 so that the
FP64 oracle and the FP32 GPU path see bit-identical inputs.
"""

from .workloads import (  # noqa: F401
    Edge,
    Problem,
    Subdomain,
    CONFIGS,
    build_problem,
    make_config,
    layer_sizes,
    param_layout,
    n_params,
    perturb_params,
)
