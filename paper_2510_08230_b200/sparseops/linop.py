"""The linear-operator contract (linop.py:44-99 of the reference).

Anything with ``shape``, ``device`` and ``apply(b, x)`` is a LinOp: every storage
format, solver and preconditioner shares it.  ``apply_advanced`` computes
``x := alpha*Op(b) + beta*x`` with the reference's rounding (temporary, then
copy+scal for beta == 0, else scal(beta)+axpy(alpha)); sparse formats do it in one
fused device pass (sb_apply_advanced_*).
"""

from __future__ import annotations

import abc

from .core import DenseMatrix, Device, _check_apply_shapes, axpy, copy_into, dense_create, scal

__all__ = ["LinOp", "apply_advanced"]


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
