"""Jacobi preconditioning on the device (precond.py:40-84 of the reference).

``jacobi_create`` extracts the stored diagonal by a per-row binary search and
inverts it in fp64 before casting (bit-exact with the reference); a zero or missing
diagonal raises SingularDiagonalError naming the first such row.  The incomplete
factorisations (ILU(0)/IC(0)) are outside this build's hot path:
their constructors exist for API compatibility and raise UnsupportedFeatureError.
"""

from __future__ import annotations

import ctypes

import torch

from .. import _lib
from .core import DenseMatrix, Device, reduce_workspace
from .errors import DimensionMismatchError, InvalidArgumentError, UnsupportedFeatureError
from .formats import CooMatrix, CsrMatrix, _ptr, _stream, csr_from_coo
from .linop import LinOp

__all__ = ["JacobiPreconditioner", "jacobi_create", "ilu0_factorize", "ic0_factorize"]


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


def ilu0_factorize(a):
    raise UnsupportedFeatureError(
        "ILU(0) is not part of the B200 hot path (SURVEY.md §8f f4); use Jacobi")


def ic0_factorize(a):
    raise UnsupportedFeatureError(
        "IC(0) is not part of the B200 hot path (SURVEY.md §8f f4); use Jacobi")
