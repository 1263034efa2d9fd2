"""Preconditioner factories (the reference's preconditioner.py:1-31)."""

from __future__ import annotations

from .. import sparseops as core

__all__ = ["Ilu", "Ic", "Jacobi"]


def Jacobi(device, a, max_block_size=1):
    """Pointwise Jacobi preconditioner (block size 1), built on the device."""
    return core.jacobi_create(a, max_block_size)


def Ilu(device, a):
    return core.ilu0_factorize(a)


def Ic(device, a):
    return core.ic0_factorize(a)
