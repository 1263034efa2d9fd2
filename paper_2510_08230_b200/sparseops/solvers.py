"""Krylov solvers whose whole iteration runs on the device: CG, CGS, BiCGSTAB, GMRES(m).

Host-side API mirrors the reference (solvers.py:1-488): OR-composed stopping
criteria with a mandatory Iteration entry, ``solve(b, x) -> ConvergenceLog``,
solver-as-LinOp ``apply``, the ``*_solve`` helpers and ``SolverParams``.  One call
enqueues the setup kernels and one CUDA-graph WHILE loop over fused iteration
kernels (libsparseb200 ``sb_<solver>_solve_<value>_<index>``); the host waits once
for the final control block and residual history.  BiCGSTAB is new (the reference
lacks it); its exact recurrence is documented in oracle/sbref.cpp.

Fused device loops take a sparse operator with Jacobi, ILU(0), IC(0) or no
preconditioner.  Any other LinOp operator or preconditioner (a solver used as a
preconditioner, a dense matrix, a user operator) and GMRES ``trace=`` run the
reference's loop composed from device BLAS-1 kernels and ``LinOp.apply`` (composed.py).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _lib
from .core import DenseMatrix, dense_create
from .errors import (BreakdownError, DimensionMismatchError, InvalidArgumentError,
                     NumericFailureError, PrecisionMismatchError, UnsupportedFeatureError)
from .formats import _SparseBase, _stream
from .linop import LinOp
from .precond import IcFactor, IluFactors, JacobiPreconditioner
from .linop import tri_workspace
from . import composed
from .composed import GmresTraceEvent

__all__ = ["Iteration", "ResidualNorm", "ConvergenceLog", "SolverParams", "check_criteria",
           "validate_criteria", "givens_rotation", "Cg", "Cgs", "Gmres", "Bicgstab",
           "cg_solve", "cgs_solve", "gmres_solve", "bicgstab_solve", "BREAKDOWN_RTOL",
           "GmresTraceEvent"]

BREAKDOWN_RTOL = 1e-30
STOP_RESIDUAL = "residual"
STOP_MAX_ITERS = "max_iters"
_HISTORY_CAP = 1 << 22


@dataclass(frozen=True)
class Iteration:
    """Stop once the iteration count reaches ``max_iters``."""

    max_iters: int

    def __post_init__(self):
        if self.max_iters < 1:
            raise InvalidArgumentError("max_iters must be positive")


@dataclass(frozen=True)
class ResidualNorm:
    """Stop once ||r|| <= reduction_factor * ||b|| (absolute if ||b|| == 0)."""

    reduction_factor: float
    baseline: str = "rhs_norm"

    def __post_init__(self):
        if self.reduction_factor <= 0:
            raise InvalidArgumentError("reduction_factor must be positive")
        if self.baseline != "rhs_norm":
            raise UnsupportedFeatureError(
                f"unsupported residual baseline {self.baseline!r}; only 'rhs_norm'")


@dataclass
class ConvergenceLog:
    """Iterations executed, one residual per criteria check, and the stop reason."""

    iterations: int
    residual_history: list = field(default_factory=list)
    converged: bool = False
    stop_reason: str = STOP_MAX_ITERS


@dataclass
class SolverParams:
    """Direct-construction bundle; ``reduction_factor=None`` means fixed iterations."""

    max_iters: int
    reduction_factor: float | None = None
    krylov_dim: int = 30
    preconditioner: LinOp | None = None

    def criteria(self) -> list:
        crit: list = [Iteration(self.max_iters)]
        if self.reduction_factor is not None:
            crit.append(ResidualNorm(self.reduction_factor))
        return crit


def validate_criteria(criteria) -> list:
    if not criteria:
        raise InvalidArgumentError("criteria list must be non-empty")
    if not any(isinstance(c, Iteration) for c in criteria):
        raise InvalidArgumentError("criteria must contain an Iteration entry")
    for c in criteria:
        if not isinstance(c, (Iteration, ResidualNorm)):
            raise InvalidArgumentError(f"unknown criterion {c!r}")
    return list(criteria)


def check_criteria(criteria, iterations: int, residual: float, rhs_norm: float):
    """Host statement of the stop rule the device evaluates (solvers.py:121-135)."""
    for c in criteria:
        if isinstance(c, ResidualNorm):
            thr = c.reduction_factor * rhs_norm if rhs_norm > 0 else c.reduction_factor
            if residual <= thr:
                return STOP_RESIDUAL
    for c in criteria:
        if isinstance(c, Iteration) and iterations >= c.max_iters:
            return STOP_MAX_ITERS
    return None


def givens_rotation(a: float, b: float) -> tuple[float, float, float]:
    """(c, s, r) with c*a + s*b = r and -s*a + c*b = 0; (0, 0) -> (1, 0, 0)."""
    if a == 0.0 and b == 0.0:
        return 1.0, 0.0, 0.0
    r = math.hypot(a, b)
    return a / r, b / r, r


def _criteria_struct(criteria) -> _lib.SbCriteria:
    # OR semantics: the earliest Iteration and the loosest ResidualNorm decide
    max_iters = min(c.max_iters for c in criteria if isinstance(c, Iteration))
    rfs = [c.reduction_factor for c in criteria if isinstance(c, ResidualNorm)]
    return _lib.SbCriteria(max_iters, 1 if rfs else 0, 0, float(max(rfs)) if rfs else 0.0)


_KINDS = {"cg": _lib.SOLVER_CG, "cgs": _lib.SOLVER_CGS, "gmres": _lib.SOLVER_GMRES,
          "bicgstab": _lib.SOLVER_BICGSTAB}


class _SolverBase(LinOp):
    _kind = None

    def __init__(self, a, criteria=None, preconditioner=None, params: SolverParams | None = None):
        rows, cols = a.shape
        if rows != cols:
            raise DimensionMismatchError(f"solver needs a square operator, got {rows}x{cols}")
        if params is not None:
            if criteria is not None:
                raise InvalidArgumentError("pass either criteria or params, not both")
            criteria = params.criteria()
            if preconditioner is None:
                preconditioner = params.preconditioner
        self.a = a
        self.criteria = validate_criteria(criteria)
        self.preconditioner = preconditioner
        self._ws = None
        self.krylov_dim = getattr(self, "krylov_dim", 0)

    @property
    def shape(self):
        return self.a.shape

    @property
    def device(self):
        return self.a.device

    def apply(self, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
        self.solve(b, x)
        return x

    # -- device solve -------------------------------------------------------------
    def _workspace(self, n: int, vbytes: int, cap: int) -> torch.Tensor:
        need = int(_lib.fn("sb_solver_workspace_bytes")(_KINDS[self._kind], vbytes, n,
                                                         self.krylov_dim, cap))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device.torch)
        return self._ws

    def _composed(self, b, x, trace=None) -> ConvergenceLog:
        """The reference loop composed from device BLAS-1 + LinOp.apply (composed.py)."""
        chk = lambda *args: check_criteria(*args)  # noqa: E731  (late-bound, patchable)
        m = self.preconditioner
        if self._kind == "gmres":
            return composed.run_gmres(self.a, b, x, self.criteria, m, self.krylov_dim, chk,
                                      ConvergenceLog, trace)
        run = {"cg": composed.run_cg, "cgs": composed.run_cgs,
               "bicgstab": composed.run_bicgstab}[self._kind]
        return run(self.a, b, x, self.criteria, m, chk, ConvergenceLog)

    def _fused_operands(self) -> bool:
        m = self.preconditioner
        return isinstance(self.a, _SparseBase) and (
            m is None or isinstance(m, (JacobiPreconditioner, IluFactors, IcFactor)))

    def solve(self, b: DenseMatrix, x: DenseMatrix) -> ConvergenceLog:
        a = self.a
        if not self._fused_operands():
            return self._composed(b, x)
        n = a.rows
        if b.shape != (n, 1) or x.shape != (n, 1):
            raise DimensionMismatchError(
                f"expected {n}x1 vectors, got b {b.shape} and x {x.shape}")
        if not (a.values.dtype == b.values.dtype == x.values.dtype):
            raise PrecisionMismatchError("matrix, b and x must share one precision")
        m = self.preconditioner
        tri = None
        if m is None:
            inv = None
        elif isinstance(m, JacobiPreconditioner):
            if m.inv_diag.numel() != n or m.inv_diag.dtype != a.values.dtype:
                raise DimensionMismatchError("preconditioner does not match the operator")
            inv = m.inv_diag
        elif isinstance(m, (IluFactors, IcFactor)):
            l, l_unit, u = m.tri_factors()
            if l.rows != n or u.rows != n or l.values.dtype != a.values.dtype or \
                    u.values.dtype != a.values.dtype or l.index_width != a.index_width or \
                    u.index_width != a.index_width:
                raise DimensionMismatchError("preconditioner factors do not match the operator")
            inv = None
            ls, us = l.struct(), u.struct()
            tws = tri_workspace(a.device, n)
            tri = (_lib.SbTriPrecond(ctypes.pointer(ls), int(l_unit), 0, ctypes.pointer(us),
                                     tws.data_ptr()), ls, us, tws)
        else:  # unreachable: _fused_operands() routed it to the composed loop
            raise UnsupportedFeatureError(f"{type(m).__name__} preconditioner")
        # contiguous, 16-byte aligned vectors for the fused kernels (a padded stride or an
        # offset view is copied around)
        bb = b if _packed(b) else _contiguous_copy(b)
        xx = x if _packed(x) else _contiguous_copy(x)
        crit = _criteria_struct(self.criteria)
        cap = int(min(crit.max_iters, _HISTORY_CAP))
        hist = np.zeros(max(cap, 1), np.float64)
        log = _lib.SbLog(0, 0, 0, 0, hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap)
        ws = self._workspace(n, a.precision.itemsize, cap)
        mat = a.matrix_struct()
        bs, xs = bb.struct(), xx.struct()
        name = f"sb_{self._kind}_solve_{a._suffix()}"
        inv_p = ctypes.c_void_p(inv.data_ptr() if inv is not None else 0)
        def _log():
            hl = min(int(log.history_len), cap)
            return ConvergenceLog(int(log.iterations), hist[:hl].tolist(), bool(log.converged),
                                  STOP_RESIDUAL if log.stop_reason == 0 else STOP_MAX_ITERS)

        try:
            if tri is not None:
                tname = f"sb_{self._kind}_solve_tri_{a._suffix()}"
                extra = (int(self.krylov_dim),) if self._kind == "gmres" else ()
                _lib.call(tname, ctypes.byref(mat), ctypes.byref(tri[0]), ctypes.byref(bs),
                          ctypes.byref(xs), ctypes.byref(crit), *extra,
                          ctypes.c_void_p(ws.data_ptr()), ctypes.byref(log), _stream(a.device))
            elif self._kind == "gmres":
                _lib.call(name, ctypes.byref(mat), inv_p, ctypes.byref(bs), ctypes.byref(xs),
                          ctypes.byref(crit), int(self.krylov_dim), ctypes.c_void_p(ws.data_ptr()),
                          ctypes.byref(log), _stream(a.device))
            else:
                _lib.call(name, ctypes.byref(mat), inv_p, ctypes.byref(bs), ctypes.byref(xs),
                          ctypes.byref(crit), ctypes.c_void_p(ws.data_ptr()), ctypes.byref(log),
                          _stream(a.device))
        except (BreakdownError, NumericFailureError) as exc:
            exc.log = _log()  # residual history up to the failure (diagnostics)
            raise
        finally:
            if xx is not x:
                x.array.copy_(xx.array)
        return _log()


def _packed(v: DenseMatrix) -> bool:
    return v.stride == 1 and v.values.data_ptr() % 16 == 0


def _contiguous_copy(v: DenseMatrix) -> DenseMatrix:
    out = dense_create(v.device, v.rows, v.cols, v.precision, 0.0)
    out.array.copy_(v.array)
    return out


class Cg(_SolverBase):
    """Preconditioned conjugate gradient (SPD operators), solvers.py:188-224."""

    _kind = "cg"


class Cgs(_SolverBase):
    """Conjugate gradient squared, solvers.py:231-284."""

    _kind = "cgs"


class Bicgstab(_SolverBase):
    """Right-preconditioned BiCGSTAB (van der Vorst); two SpMVs per iteration."""

    _kind = "bicgstab"


class Gmres(_SolverBase):
    """Restarted GMRES(krylov_dim) with right preconditioning, single-pass MGS, Givens
    rotations and the residual estimate checked every inner iteration (solvers.py:322-399)."""

    _kind = "gmres"

    def __init__(self, a, criteria=None, preconditioner=None, params: SolverParams | None = None,
                 krylov_dim: int | None = None):
        if krylov_dim is None:
            krylov_dim = params.krylov_dim if params is not None else 30
        if krylov_dim < 1:
            raise InvalidArgumentError("krylov_dim must be positive")
        self.krylov_dim = int(krylov_dim)
        super().__init__(a, criteria, preconditioner, params)

    def solve(self, b, x, trace=None):
        if trace is not None:  # host snapshots every inner iteration: the composed loop
            return self._composed(b, x, trace)
        return super().solve(b, x)


def cg_solve(a, b, x, params: SolverParams):
    """Solve A x = b with CG; x is overwritten, b untouched."""
    return Cg(a, params=params).solve(b, x), x


def cgs_solve(a, b, x, params: SolverParams):
    return Cgs(a, params=params).solve(b, x), x


def bicgstab_solve(a, b, x, params: SolverParams):
    return Bicgstab(a, params=params).solve(b, x), x


def gmres_solve(a, b, x, params: SolverParams, trace=None):
    return Gmres(a, params=params).solve(b, x, trace=trace), x
