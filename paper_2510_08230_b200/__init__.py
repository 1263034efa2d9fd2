"""B200-native SpMV + Krylov hot path of pyGinkgo (arXiv 2510.08230).

Subpackages mirror the reference's two layers:

* ``paper_2510_08230_b200.sparseops``   -- device core (formats, SpMV, BLAS-1, Jacobi,
  CG / CGS / BiCGSTAB / GMRES, config solve), the reference ``sparseops`` API;
* ``paper_2510_08230_b200.pysparseops`` -- the frontend (``device``, ``read``,
  ``as_tensor``, ``solve``, ``solver.*``, ``preconditioner.*``, typed ``bindings``).

All compute runs in ``libsparseb200.so`` (hand-written sm_100a CUDA behind the C ABI
in include/sparseb200.h); there is no CPU fallback.
"""

from . import pysparseops, sparseops
from ._lib import LIB_PATH, LibraryUnavailableError

__version__ = "0.1.0"
__all__ = ["pysparseops", "sparseops", "LIB_PATH", "LibraryUnavailableError"]
