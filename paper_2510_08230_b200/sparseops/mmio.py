"""Matrix Market ingest feeding device construction.

Host text parsing (NumPy) of ``coordinate`` / ``array`` bodies with ``real``,
``integer`` or ``pattern`` fields and ``general`` / ``symmetric`` /
``skew-symmetric`` symmetry (mirrored entries added), then canonicalisation on the
device through coo_from_arrays.  Errors use the reference's mmio kinds.
"""

from __future__ import annotations

import numpy as np

from .core import IndexWidth, Precision
from .errors import (EntryCountError, MalformedBannerError, MalformedSizeError,
                     UnsupportedFieldError)
from .formats import coo_from_arrays, csr_from_coo

__all__ = ["read_matrix_market", "write_matrix_market"]


def _parse(path):
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines or not lines[0].lower().startswith("%%matrixmarket"):
        raise MalformedBannerError(f"{path}: missing %%MatrixMarket banner")
    parts = lines[0].lower().split()
    if len(parts) != 5 or parts[1] != "matrix":
        raise MalformedBannerError(f"{path}: malformed banner {lines[0]!r}")
    layout, field, symmetry = parts[2], parts[3], parts[4]
    if layout not in ("coordinate", "array"):
        raise MalformedBannerError(f"{path}: unknown layout {layout!r}")
    if field not in ("real", "integer", "pattern", "double"):
        raise UnsupportedFieldError(f"{path}: unsupported field {field!r}")
    if symmetry not in ("general", "symmetric", "skew-symmetric"):
        raise UnsupportedFieldError(f"{path}: unsupported symmetry {symmetry!r}")
    body = [ln for ln in lines[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        raise MalformedSizeError(f"{path}: missing size line")
    try:
        size = [int(t) for t in body[0].split()]
    except ValueError:
        raise MalformedSizeError(f"{path}: malformed size line {body[0]!r}") from None
    return layout, field, symmetry, size, body[1:]


def read_matrix_market(device, path, precision: Precision = Precision.double, format="Csr",
                       index_width: IndexWidth = IndexWidth.i32):
    layout, field, symmetry, size, entries = _parse(path)
    if layout == "coordinate":
        if len(size) != 3:
            raise MalformedSizeError(f"{path}: expected 'rows cols nnz'")
        rows, cols, count = size
        if len(entries) != count:
            raise EntryCountError(f"{path}: expected {count} entries, found {len(entries)}")
        if count:
            tab = np.array([ln.split() for ln in entries], dtype=object)
            ri = tab[:, 0].astype(np.int64) - 1
            ci = tab[:, 1].astype(np.int64) - 1
            vals = np.ones(count) if field == "pattern" else tab[:, 2].astype(np.float64)
        else:
            ri = ci = np.zeros(0, np.int64)
            vals = np.zeros(0)
    else:
        if len(size) != 2:
            raise MalformedSizeError(f"{path}: expected 'rows cols'")
        rows, cols = size
        data = np.array([float(ln.split()[0]) for ln in entries])
        if symmetry == "general":
            if data.size != rows * cols:
                raise EntryCountError(f"{path}: expected {rows * cols} values, found {data.size}")
            ci, ri = np.divmod(np.arange(rows * cols, dtype=np.int64), rows)  # column-major
        else:
            ri_l, ci_l = [], []
            for j in range(cols):
                for i in range(j if symmetry == "symmetric" else j + 1, rows):
                    ri_l.append(i)
                    ci_l.append(j)
            if data.size != len(ri_l):
                raise EntryCountError(f"{path}: expected {len(ri_l)} values, found {data.size}")
            ri, ci = np.asarray(ri_l, np.int64), np.asarray(ci_l, np.int64)
        vals = data
        keep = vals != 0.0
        ri, ci, vals = ri[keep], ci[keep], vals[keep]
    if symmetry != "general":
        off = ri != ci
        sign = -1.0 if symmetry == "skew-symmetric" else 1.0
        ri, ci, vals = (np.concatenate([ri, ci[off]]), np.concatenate([ci, ri[off]]),
                        np.concatenate([vals, sign * vals[off]]))
    coo = coo_from_arrays(device, rows, cols, ri, ci, vals, precision, index_width)
    return coo if str(format).lower() == "coo" else csr_from_coo(coo)


def write_matrix_market(path, m):
    """Write any sparse matrix as 'coordinate real general' (%.17g round-trips fp64)."""
    r, c, v = m._entries_host()
    order = np.lexsort((c, r))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{m.rows} {m.cols} {len(v)}\n")
        for k in order:
            fh.write(f"{int(r[k]) + 1} {int(c[k]) + 1} {float(v[k]):.17g}\n")
