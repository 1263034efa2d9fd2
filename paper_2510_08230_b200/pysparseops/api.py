"""High-level entry points (the reference's api.py:1-45): device, read, solve and the
dispatched vector ops, plus ``matrix`` constructors from NumPy / SciPy / torch."""

from __future__ import annotations

from .. import sparseops as core
from . import dispatch
from .dispatch import axpy, dot, norm2, scal, spmv

__all__ = ["device", "read", "solve", "matrix", "dot", "norm2", "axpy", "scal", "spmv"]

_INDEX = {"i32": core.IndexWidth.i32, "int32": core.IndexWidth.i32,
          "i64": core.IndexWidth.i64, "int64": core.IndexWidth.i64}
_FORMATS = ("csr", "coo", "ell", "sellp", "hybrid")


def device(name: str = "cuda", id: int = 0, threads: int | None = None) -> core.Device:
    """Create an execution device ("cuda" in this build)."""
    return core.create_device(name, id, threads)


def _index(index):
    key = str(index).lower()
    if key not in _INDEX:
        raise core.errors.UnsupportedFeatureError(
            f"unknown index width {index!r}; expected 'i32' or 'i64'")
    return _INDEX[key]


def _convert(m, fmt):
    if fmt in ("csr", "coo"):
        return m
    csr = m if isinstance(m, core.CsrMatrix) else core.csr_from_coo(m)
    return {"ell": core.ell_from_csr, "sellp": core.sellp_from_csr,
            "hybrid": core.hybrid_from_csr}[fmt](csr)


def read(device, path, dtype="double", format="Csr", index="i32"):
    """Read a Matrix Market file onto the device in the requested format."""
    vdt = dispatch.value_dtype(dtype)
    fmt = str(format).lower()
    if fmt not in _FORMATS:
        raise core.errors.MatrixMarketError(
            f"unknown format {format!r}; expected one of Csr, Coo, Ell, Sellp, Hybrid")
    iw = _index(index)
    base = "coo" if fmt == "coo" else "csr"
    m = dispatch.resolve(f"read_{base}", vdt, iw.dtype)(device, path)
    return _convert(m, fmt)


def matrix(device, source, dtype=None, format="Csr", index="i32"):
    """Sparse matrix on the device from a scipy.sparse matrix, a torch sparse / dense
    tensor, a dense NumPy array or (row, col, value) triplet arrays."""
    fmt = str(format).lower()
    if fmt not in _FORMATS:
        raise core.errors.InvalidArgumentError(f"unknown format {format!r}")
    iw = _index(index)
    prec = None if dtype is None else core.Precision.from_dtype(dispatch.value_dtype(dtype))
    import numpy as np
    import torch

    if hasattr(source, "tocoo"):
        m = core.from_scipy(device, source, prec, iw, "coo" if fmt == "coo" else "csr")
    elif isinstance(source, torch.Tensor):
        m = core.from_torch(device, source if prec is None else source.to(prec.torch_dtype), iw,
                            "coo" if fmt == "coo" else "csr")
    elif isinstance(source, tuple) and len(source) == 4:
        shape, ri, ci, vals = source
        coo = core.coo_from_arrays(device, shape[0], shape[1], ri, ci, vals,
                                   prec or core.Precision.double, iw)
        m = coo if fmt == "coo" else core.csr_from_coo(coo)
    else:
        m = core.csr_from_dense(device, np.asarray(source), prec or core.Precision.double, iw)
        if fmt == "coo":
            m = core.coo_from_csr(m)
    return _convert(m, fmt)


def solve(args, a, b, x):
    """Config-driven solve (Listing 2): returns (logger, result); result aliases x."""
    logger, _ = core.config_solve(args, a.device, a, b, x)
    return logger, x
