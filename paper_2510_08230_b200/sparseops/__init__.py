"""sparseops (B200): device-resident mirror of the reference's core package.

Same public names as the reference ``sparseops`` (pkg/src/sparseops/__init__.py)
for the hot path -- devices, dense storage, BLAS-1, CSR/COO storage and conversion,
LinOp, Jacobi, ILU(0)/IC(0) and triangular solves, CG/CGS/GMRES solvers, criteria,
config solve -- plus ELL, SELL-P, Hybrid and BiCGSTAB.  All compute runs in libsparseb200 on the GPU.
"""

from . import errors
from .config import (PreconditionerConfig, SolverConfig, build_solver, config_solve,
                     load_config, parse_config)
from .core import (DenseMatrix, Device, DeviceKind, IndexWidth, Precision, axpy, copy_into,
                   create_device, dense_create, dense_from_array, dot, norm2, scal)
from .formats import (CooMatrix, CsrMatrix, EllMatrix, HybridMatrix, SellpMatrix,
                      coo_from_arrays, coo_from_csr, coo_from_triplets, csr_from_coo,
                      csr_from_dense, ell_from_csr, from_scipy, from_torch, hybrid_ell_width,
                      hybrid_from_csr, sellp_from_csr, validate)
from .linop import LinOp, apply_advanced, solve_lower_tri, solve_upper_tri
from .mmio import (DuplicateEntryWarning, MatrixMarketHeader, read_matrix_market,
                   write_matrix_market)
from .precond import (IcFactor, IluFactors, JacobiPreconditioner, ic0_factorize, ic_apply,
                      ilu0_factorize, ilu_apply, jacobi_create)
from .solvers import (Bicgstab, Cg, Cgs, ConvergenceLog, Gmres, GmresTraceEvent, Iteration, ResidualNorm,
                      SolverParams, bicgstab_solve, cg_solve, cgs_solve, check_criteria,
                      gmres_solve, givens_rotation, validate_criteria)


def spmv_csr(a, b, x):
    """x = A*b for CSR storage (linop.spmv_csr contract)."""
    if not isinstance(a, CsrMatrix):
        raise errors.InvalidArgumentError(f"expected CsrMatrix, got {type(a).__name__}")
    return a.apply(b, x)


def spmv_coo(a, b, x):
    """x = A*b for COO storage (linop.spmv_coo contract)."""
    if not isinstance(a, CooMatrix):
        raise errors.InvalidArgumentError(f"expected CooMatrix, got {type(a).__name__}")
    return a.apply(b, x)


__version__ = "0.1.0"
