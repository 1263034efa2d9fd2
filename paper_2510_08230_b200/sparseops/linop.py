"""The linear-operator contract (linop.py:44-99 of the reference).

Anything with ``shape``, ``device`` and ``apply(b, x)`` is a LinOp: every storage
format, solver and preconditioner shares it.  ``apply_advanced`` computes
``x := alpha*Op(b) + beta*x`` with the reference's rounding (temporary, then
copy+scal for beta == 0, else scal(beta)+axpy(alpha)); sparse formats do it in one
fused device pass (sb_apply_advanced_*).
"""

from __future__ import annotations

import abc
import ctypes

from .. import _lib
from .core import DenseMatrix, Device, _check_apply_shapes, axpy, copy_into, dense_create, scal
from .errors import DimensionMismatchError, InvalidArgumentError

__all__ = ["LinOp", "apply_advanced", "solve_lower_tri", "solve_upper_tri"]


class LinOp(abc.ABC):
    """Abstract linear operator."""

    @property
    @abc.abstractmethod
    def shape(self) -> tuple[int, int]:
        """(rows, cols) of the operator."""

    @property
    def size(self) -> tuple[int, int]:
        return self.shape

    @property
    @abc.abstractmethod
    def device(self) -> Device:
        """Device the operator executes on."""

    @abc.abstractmethod
    def apply(self, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
        """Write x = Op(b) and return x."""

    def apply_advanced(self, alpha: float, b: DenseMatrix, beta: float,
                       x: DenseMatrix) -> DenseMatrix:
        """Write x := alpha*Op(b) + beta*x and return x."""
        return apply_advanced(self, alpha, b, beta, x)


LinOp.register(DenseMatrix)


def apply_advanced(op, alpha: float, b: DenseMatrix, beta: float, x: DenseMatrix) -> DenseMatrix:
    """Generic x := alpha*op(b) + beta*x; beta == 0 overwrites x (stale NaN/Inf in x
    cannot leak), exactly as linop.py:81-99."""
    _check_apply_shapes(op.shape, b, x)
    fused = getattr(op, "_apply_advanced_device", None)
    if fused is not None:
        return fused(alpha, b, beta, x)
    t = dense_create(x.device, x.rows, x.cols, x.precision, 0.0)
    op.apply(b, t)
    if beta == 0:
        copy_into(t, x)
        scal(alpha, x)
    else:
        scal(beta, x)
        axpy(alpha, t, x)
    return x


# ------------------------------------------------------------------ triangular solves
_TRI_WS = {}


def tri_workspace(device: Device, n: int):
    """Per-device scratch of the sync-free triangular sweeps (ready flags, counters)."""
    import torch

    need = int(_lib.fn("sb_tri_workspace_bytes")(n))
    key = device.id
    ws = _TRI_WS.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=device.torch)
        _TRI_WS[key] = ws
    return ws


def _trisolve(t, b: DenseMatrix, x: DenseMatrix, lower: bool, unit: bool) -> DenseMatrix:
    from .formats import CsrMatrix, _ptr, _stream

    if not isinstance(t, CsrMatrix):
        raise InvalidArgumentError(f"triangular solves need CSR storage, got {type(t).__name__}")
    if t.rows != t.cols:
        raise DimensionMismatchError(f"triangular solve needs a square matrix, got {t.shape}")
    _check_apply_shapes(t.shape, b, x)
    ws = tri_workspace(t.device, t.rows)
    st, bs, xs = t.struct(), b.struct(), x.struct()
    _lib.call(f"sb_csr_trisolve_{t._suffix()}", ctypes.byref(st), int(lower), int(unit),
              ctypes.byref(bs), ctypes.byref(xs), _ptr(ws), _stream(t.device))
    return x


def solve_lower_tri(l, b: DenseMatrix, x: DenseMatrix, unit_diag: bool = False) -> DenseMatrix:
    """Solve L*x = b by forward substitution (linop.py:169-189); the device sweep keeps the
    reference's per-row order (bit-exact).  With ``unit_diag`` the diagonal is implicitly
    1 and stored diagonal entries are ignored as values; entries above the diagonal raise
    NotTriangularError, a missing / zero diagonal SingularTriangleError (first row)."""
    return _trisolve(l, b, x, True, unit_diag)


def solve_upper_tri(u, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
    """Solve U*x = b by backward substitution (linop.py:192-198)."""
    return _trisolve(u, b, x, False, False)
