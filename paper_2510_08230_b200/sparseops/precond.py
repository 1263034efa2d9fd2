"""Preconditioners on the device (precond.py of the reference).

``jacobi_create`` extracts the stored diagonal by a per-row binary search and
inverts it in fp64 before casting (bit-exact with the reference); a zero or missing
diagonal raises SingularDiagonalError naming the first such row.

``ilu0_factorize`` / ``ic0_factorize`` (precond.py:155-256) run as sync-free device
sweeps (csrc/trisolve.cu): one thread per row, rows claimed in order, each row waiting
on the ready flags of the rows it reads -- the reference's row loops in the reference's
order, so the factors are bit-exact; errors name the reference's row (ZeroPivotError,
IndefinitePivotError).  ``IluFactors`` / ``IcFactor`` apply by two device triangular
solves (linop.solve_lower_tri / solve_upper_tri) and plug into the device CG and GMRES.
"""

from __future__ import annotations

import ctypes

import torch

from .. import _lib
from .core import DenseMatrix, Device, reduce_workspace
from .core import dense_create
from .errors import DimensionMismatchError, InvalidArgumentError, UnsupportedFeatureError
from .formats import CooMatrix, CsrMatrix, _ptr, _stream, coo_from_arrays, csr_from_coo
from .linop import LinOp, solve_lower_tri, solve_upper_tri, tri_workspace

__all__ = ["JacobiPreconditioner", "jacobi_create", "ilu0_factorize", "ic0_factorize",
           "IluFactors", "IcFactor", "ilu_apply", "ic_apply"]


class JacobiPreconditioner(LinOp):
    """Pointwise Jacobi: ``apply`` multiplies elementwise by the inverted diagonal."""

    def __init__(self, device: Device, inv_diag: torch.Tensor, max_block_size: int = 1):
        self._device = device
        self.inv_diag = inv_diag
        self.max_block_size = max_block_size

    @property
    def shape(self):
        n = self.inv_diag.numel()
        return (n, n)

    @property
    def device(self):
        return self._device

    def apply(self, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
        if b.rows != self.inv_diag.numel():
            raise DimensionMismatchError(
                f"expected vectors of length {self.inv_diag.numel()}, got {b.rows}")
        bs, xs = b.struct(), x.struct()
        _lib.call(f"sb_jacobi_apply_{b.precision.suffix}", _ptr(self.inv_diag), ctypes.byref(bs),
                  ctypes.byref(xs), _stream(self._device))
        return x


def _as_csr(a) -> CsrMatrix:
    if isinstance(a, CsrMatrix):
        return a
    if isinstance(a, CooMatrix):
        return csr_from_coo(a)
    raise InvalidArgumentError(f"preconditioners need CSR or COO storage, got {type(a).__name__}")


def jacobi_create(a, max_block_size: int = 1) -> JacobiPreconditioner:
    """Jacobi preconditioner from the matrix diagonal; only scalar blocks are supported."""
    if max_block_size != 1:
        raise UnsupportedFeatureError(
            f"block Jacobi (max_block_size={max_block_size}) is not supported; use 1")
    a = _as_csr(a)
    if a.rows != a.cols:
        raise DimensionMismatchError(f"expected a square matrix, got {a.rows}x{a.cols}")
    inv = torch.empty(a.rows, dtype=a.values.dtype, device=a.device.torch)
    ws = reduce_workspace(a.device)
    st = a.struct()
    _lib.call(f"sb_jacobi_create_{a._suffix()}", ctypes.byref(st), _ptr(inv), _ptr(ws),
              _stream(a.device))
    return JacobiPreconditioner(a.device, inv, max_block_size)


class IluFactors(LinOp):
    """ILU(0) factors (precond.py:98-120): L unit lower triangular with the unit diagonal
    implicit, U upper triangular including the diagonal; apply is x = U^{-1}(L^{-1} b)."""

    def __init__(self, l: CsrMatrix, u: CsrMatrix):
        self.l = _as_csr(l)
        self.u = _as_csr(u)

    @property
    def shape(self):
        return self.l.shape

    @property
    def device(self):
        return self.l.device

    def apply(self, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
        y = dense_create(self.device, b.rows, b.cols, b.precision, 0.0)
        solve_lower_tri(self.l, b, y, unit_diag=True)
        solve_upper_tri(self.u, y, x)
        return x

    def tri_factors(self):
        """(L, L has unit diagonal, U) for the device solvers' preconditioned loops."""
        return self.l, True, self.u


class IcFactor(LinOp):
    """IC(0) factor (precond.py:123-144): L lower triangular with a positive diagonal;
    apply is x = L^{-T}(L^{-1} b)."""

    def __init__(self, l: CsrMatrix):
        self.l = _as_csr(l)
        self._lt = _csr_transpose(self.l)

    @property
    def shape(self):
        return self.l.shape

    @property
    def device(self):
        return self.l.device

    def apply(self, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
        y = dense_create(self.device, b.rows, b.cols, b.precision, 0.0)
        solve_lower_tri(self.l, b, y, unit_diag=False)
        solve_upper_tri(self._lt, y, x)
        return x

    def tri_factors(self):
        return self.l, False, self._lt


def _csr_transpose(m: CsrMatrix) -> CsrMatrix:
    """precond._csr_transpose: (col, row, value) triplets canonicalised on the device."""
    counts = m.row_ptrs[1:] - m.row_ptrs[:-1]
    rows = torch.repeat_interleave(torch.arange(m.rows, device=m.device.torch), counts.long())
    coo = coo_from_arrays(m.device, m.cols, m.rows, m.col_idxs.long(), rows, m.values,
                          m.precision, m.index_width)
    return csr_from_coo(coo)


def _require_square(a: CsrMatrix):
    if a.rows != a.cols:
        raise DimensionMismatchError(f"factorization needs a square matrix, got {a.rows}x{a.cols}")


def _split(a: CsrMatrix, values: torch.Tensor, incl_diag: bool):
    """_split_lu (precond.py:190-202) on the device: entries with col < row (col <= row)
    and the rest, each as (row_ptrs, col_idxs, values) in stored order."""
    n, dev, it = a.rows, a.device.torch, a.col_idxs.dtype
    counts = torch.zeros(n, dtype=torch.int64, device=dev)
    _lib.call(f"sb_csr_split_count_{a.index_width.suffix}", n, _ptr(a.row_ptrs), _ptr(a.col_idxs),
              int(incl_diag), _ptr(counts), _stream(a.device))
    lp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=lp[1:])
    up = a.row_ptrs.long() - lp
    lp, up = lp.to(it), up.to(it)
    nl, nu = int(lp[-1]), int(up[-1])
    lc = torch.empty(nl, dtype=it, device=dev)
    lv = torch.empty(nl, dtype=values.dtype, device=dev)
    uc = torch.empty(nu, dtype=it, device=dev)
    uv = torch.empty(nu, dtype=values.dtype, device=dev)
    _lib.call(f"sb_csr_split_scatter_{a._suffix()}", n, _ptr(a.row_ptrs), _ptr(a.col_idxs),
              _ptr(values), _ptr(lp), _ptr(up), _ptr(lc), _ptr(lv), _ptr(uc), _ptr(uv),
              _stream(a.device))
    return (lp, lc, lv), (up, uc, uv)


def ilu0_factorize(a) -> IluFactors:
    """Incomplete LU with zero fill-in (precond.py:155-187): IKJ elimination restricted to
    the stored pattern, no pivoting; a zero pivot raises ZeroPivotError naming the row."""
    a = _as_csr(a)
    _require_square(a)
    n, dev = a.rows, a.device.torch
    vals = torch.empty_like(a.values)
    ws = tri_workspace(a.device, n)
    dpos = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    st = a.struct()
    _lib.call(f"sb_ilu0_{a._suffix()}", ctypes.byref(st), _ptr(vals), _ptr(ws), _ptr(dpos),
              _stream(a.device))
    (lp, lc, lv), (up, uc, uv) = _split(a, vals, incl_diag=False)
    return IluFactors(CsrMatrix(a.device, n, n, lp, lc, lv), CsrMatrix(a.device, n, n, up, uc, uv))


def ic0_factorize(a) -> IcFactor:
    """Incomplete Cholesky with zero fill-in on the lower triangle of A (precond.py:205-256),
    in fp64 like the reference's Python floats; a non-positive pivot raises
    IndefinitePivotError naming the row."""
    a = _as_csr(a)
    _require_square(a)
    n, dev = a.rows, a.device.torch
    (lp, lc, la), _ = _split(a, a.values, incl_diag=True)
    out = torch.empty_like(la)
    scratch = torch.empty(max(la.numel(), 1), dtype=torch.float64, device=dev)
    ws = tri_workspace(a.device, n)
    _lib.call(f"sb_ic0_{a._suffix()}", n, _ptr(lp), _ptr(lc), _ptr(la), _ptr(out), _ptr(ws),
              _ptr(scratch), _stream(a.device))
    return IcFactor(CsrMatrix(a.device, n, n, lp, lc, out))


def ilu_apply(factors: IluFactors, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
    """x = U^{-1}(L^{-1} b)."""
    return factors.apply(b, x)


def ic_apply(factor: IcFactor, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
    """x = L^{-T}(L^{-1} b)."""
    return factor.apply(b, x)
