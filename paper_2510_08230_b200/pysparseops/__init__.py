"""pysparseops (B200): the reference frontend's API on the device backend.

Same entry points as the reference's pysparseops (pkg/frontend/src/pysparseops/
__init__.py): ``device``, ``read``, ``as_tensor``, ``solve``, ``spmv``/``dot``/
``norm2``/``axpy``/``scal``, the ``solver`` and ``preconditioner`` factories and the
raw ``bindings`` -- with ``device("cuda")`` as the execution device, ELL / SELL-P /
Hybrid formats, ``solver.bicgstab`` and ``matrix(...)`` constructors from NumPy,
SciPy and torch.  Usage::

    import paper_2510_08230_b200.pysparseops as pg
    dev = pg.device("cuda")
    A = pg.matrix(dev, scipy_csr)                  # or pg.read(dev, "A.mtx")
    b = pg.as_tensor(np.ones(A.rows), device=dev)
    x = pg.as_tensor(dim=A.rows, fill=0.0, device=dev)
    logger, x = pg.solver.cg(dev, A, pg.preconditioner.Jacobi(dev, A),
                             max_iters=1000, reduction_factor=1e-8).apply(b, x)
"""

from ..sparseops import ConvergenceLog
from . import bindings, preconditioner, solver
from .api import axpy, device, dot, matrix, norm2, read, scal, solve, spmv
from .eigen import rayleigh_ritz
from .errors import (BindingError, CopyRequiredError, InstantiationMismatchError,
                     NoMatchingInstantiationError, OrthonormalityError)
from .tensor import Tensor, as_tensor

__version__ = "0.1.0"

__all__ = ["ConvergenceLog", "Tensor", "as_tensor", "axpy", "bindings", "device", "dot",
           "matrix", "norm2", "preconditioner", "rayleigh_ritz", "read", "scal", "solve", "solver",
           "spmv",
           "BindingError", "CopyRequiredError", "InstantiationMismatchError",
           "NoMatchingInstantiationError", "OrthonormalityError"]
