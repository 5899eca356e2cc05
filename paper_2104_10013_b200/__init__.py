"""B200-native parallel cPINN / XPINN training step (arXiv 2104.10013).

The compute path lives in `libpinn_dd.so` (sm_100a CUDA kernels behind the C ABI
of include/pinn_dd.h); `binding` is its thin ctypes wrapper.  Importing this
package does not load the library; `PinnDD(...)` does, and fails loudly when it
is missing.
"""

__all__ = ["binding", "LIB_PATH"]

import os as _os

LIB_PATH = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "libpinn_dd.so")
