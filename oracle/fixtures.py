"""Synthetic test-matrix generators (NumPy), restating the reference's fixtures.

TEST INFRASTRUCTURE ONLY (see oracle/sbref.py).  These are the generators of
SURVEY.md §10 (themselves the vectorised form of the reference's
``tests/helpers.py:26-54``) returning raw triplets; ``canonical_csr`` turns them
into canonical CSR through the oracle's ``coo_from_arrays`` restatement.
"""

from __future__ import annotations

import numpy as np

from . import sbref


def poisson2d_triplets(p: int):
    """5-point Laplacian on a p x p grid (helpers.py:26-42): i = gy*p + gx, diag 4, -1 off."""
    n = p * p
    idx = np.arange(n, dtype=np.int64)
    gx, gy = idx % p, idx // p
    rows, cols, vals = [idx], [idx], [np.full(n, 4.0)]
    for m, off in ((gx > 0, -1), (gx < p - 1, 1), (gy > 0, -p), (gy < p - 1, p)):
        rows.append(idx[m])
        cols.append(idx[m] + off)
        vals.append(np.full(int(m.sum()), -1.0))
    return n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def stencil3d_triplets(p: int, c: float = 0.0):
    """7-point 3D stencil: c = 0 is Poisson, c = 0.5 the convection-diffusion
    operator of config #4 (lower neighbours -1-c/2, upper -1+c/2, diag 6)."""
    n = p ** 3
    idx = np.arange(n, dtype=np.int64)
    gx, gy, gz = idx % p, (idx // p) % p, idx // (p * p)
    rows, cols, vals = [idx], [idx], [np.full(n, 6.0)]
    for m, off, v in ((gx > 0, -1, -1 - c / 2), (gx < p - 1, 1, -1 + c / 2),
                      (gy > 0, -p, -1 - c / 2), (gy < p - 1, p, -1 + c / 2),
                      (gz > 0, -p * p, -1 - c / 2), (gz < p - 1, p * p, -1 + c / 2)):
        rows.append(idx[m])
        cols.append(idx[m] + off)
        vals.append(np.full(int(m.sum()), v))
    return n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def powerlaw_triplets(n=4_000_000, mean=16, alpha=2.0, seed=20251008):
    """Config #3 pin: pareto row lengths, uniform columns, normal values."""
    rng = np.random.default_rng(seed)
    raw = rng.pareto(alpha, n) + 1.0
    lens = np.maximum(1, np.round(raw * (mean / raw.mean()))).astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size)
    return n, rows, cols, vals


def random_sparse_triplets(rng, rows, cols, density):
    """helpers.random_sparse (helpers.py:45-54): unique positions, values in [-1, 1)."""
    nnz = max(0, int(round(density * rows * cols)))
    nnz = min(nnz, rows * cols)
    flat = rng.choice(rows * cols, size=nnz, replace=False) if nnz else np.empty(0, np.int64)
    vals = rng.uniform(-1.0, 1.0, size=nnz)
    flat = np.asarray(flat, dtype=np.int64)
    return flat // cols, flat % cols, vals


def oracle_suite(count=200, seed=2024):
    """The acceptance suite's 200 random matrices (test_acceptance.py:58-72), as
    (rows, cols, row_idxs, col_idxs, values, b) raw triplets in the same RNG order."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        rows = int(rng.integers(1, 201))
        cols = int(rng.integers(1, 201))
        density = float(rng.uniform(0.005, 0.10))
        ri, ci, v = random_sparse_triplets(rng, rows, cols, density)
        bv = rng.standard_normal(cols)
        out.append((rows, cols, ri, ci, v, bv))
    return out


def canonical_csr(rows, row_idxs, col_idxs, values, dtype=np.float64, index=np.int32):
    """coo_from_arrays + csr_from_coo via the oracle restatement."""
    r, c, v = sbref.coo_canonicalize(row_idxs, col_idxs, values, dtype)
    return sbref.csr_row_ptrs(r, rows, index), c.astype(index), v


def stencil_csr(p, dim=3, c=0.0, dtype=np.float64, index=np.int32):
    """Canonical CSR of a stencil matrix without the generic sort (the stencil rows are
    generated per row in column order, so this equals coo_from_arrays + csr_from_coo)."""
    if dim == 2:
        n, r, cc, v = poisson2d_triplets(p)
    else:
        n, r, cc, v = stencil3d_triplets(p, c)
    order = np.lexsort((cc, r))
    r, cc, v = r[order], cc[order], v[order]
    return sbref.csr_row_ptrs(r, n, index), cc.astype(index), v.astype(dtype)
