"""Helpers shared by the GPU parity tests."""

import numpy as np
import torch

from paper_2510_08230_b200 import sparseops as sp

TOL = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}


def csr(dev, row_ptrs, col_idxs, values, cols=None, kernel="auto"):
    rows = len(row_ptrs) - 1
    return sp.CsrMatrix(dev, rows, rows if cols is None else cols, row_ptrs, col_idxs, values,
                        kernel=kernel)


def vec(dev, v, dtype=None):
    v = np.asarray(v, dtype=dtype)
    return sp.dense_from_array(dev, v.copy())


def out(dev, n, dtype, fill=np.nan, cols=1):
    return sp.dense_create(dev, n, cols, sp.Precision.from_dtype(dtype), fill)


def host(x):
    torch.cuda.synchronize()
    return x.numpy()[:, 0] if x.cols == 1 else x.numpy()


def scale(row_ptrs, values, b):
    """max_i sum_j |a_ij| * max|b| (test_acceptance.py:80-87 scale)."""
    rp = np.asarray(row_ptrs, np.int64)
    absv = np.abs(np.asarray(values, np.float64))
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    rs = np.bincount(rows, weights=absv, minlength=len(rp) - 1)
    mx = rs.max(initial=0.0)
    return max(mx * max(np.abs(np.asarray(b, np.float64)).max(initial=0.0), 1e-30), 1e-30)


def assert_close(x, ref, row_ptrs, values, b):
    tol = TOL[np.dtype(np.asarray(ref).dtype)]
    err = np.abs(np.asarray(x, np.float64) - np.asarray(ref, np.float64)).max(initial=0.0)
    assert err <= tol * scale(row_ptrs, values, b), f"error {err:.3e} > {tol} * scale"
