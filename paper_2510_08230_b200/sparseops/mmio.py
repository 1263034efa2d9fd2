"""Matrix Market ingest feeding device construction.

The text layer is host work by nature (a file is parsed once); what it produces is a
raw triplet stream that ``coo_from_arrays`` canonicalises ON THE DEVICE (CUB radix
sort + ordered duplicate sums, csrc/convert.cu).  The triplet stream must therefore be
exactly the reference's, entry for entry and in the same order, or the canonical
arrays (nnz, row_ptrs, col_idxs, the summed values) differ.  Semantics follow
reference ``pkg/src/sparseops/mmio.py``:

* banner  (``_parse_banner`` :51-70): 5 tokens, case-insensitive; ``complex`` ->
  UnsupportedFieldError, every other unknown object/format/field/symmetry and
  ``array`` + ``pattern`` -> MalformedBannerError;
* size line (``_parse_size`` :80-91): first non-blank, non-``%`` line; 3 (coordinate)
  or 2 (array) non-negative integers else MalformedSizeError; non-general symmetry on
  a non-square shape -> MalformedSizeError (:214-218, :222-226);
* coordinate bodies (:94-125): one numeric table, ``%`` comments allowed anywhere;
  ragged / unparsable -> MatrixMarketError; entry count -> EntryCountError;
  non-integral indices -> MatrixMarketError; first out-of-range entry ->
  IndexBoundsError; ``pattern`` values are 1.0;
* array bodies (:128-166): every token of every data line, column-major, **explicit
  zeros kept**; symmetric stores the lower triangle with its diagonal, skew the
  strict lower triangle;
* symmetry expansion (:169-177) appends the mirrored off-diagonal entries after the
  stored ones (skew negated); duplicates warn once (:180-191) and are summed by the
  canonicalisation;
* writer (:235-244): ``write_matrix_market(m, path)``, coordinate/real/general,
  1-based, ``%.17g`` (bit-exact fp64 round trip).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from .core import IndexWidth, Precision
from .errors import (EntryCountError, IndexBoundsError, MalformedBannerError,
                     MalformedSizeError, MatrixMarketError, UnsupportedFieldError)
from .formats import coo_from_arrays, csr_from_coo

__all__ = ["MatrixMarketHeader", "DuplicateEntryWarning", "read_matrix_market",
           "write_matrix_market", "read_entries"]


class DuplicateEntryWarning(UserWarning):
    """A coordinate position occurs more than once; the values are summed (mmio.py:40-41)."""


@dataclass(frozen=True)
class MatrixMarketHeader:
    """The parsed banner (mmio.py:44-49)."""

    object: str
    format: str
    field: str
    symmetry: str


_VALID = {
    "format": ("coordinate", "array"),
    "field": ("real", "integer", "pattern"),
    "symmetry": ("general", "symmetric", "skew-symmetric"),
}


def parse_banner(line: str) -> MatrixMarketHeader:
    words = line.strip().lower().split()
    if not words or words[0] != "%%matrixmarket":
        raise MalformedBannerError(f"not a Matrix Market banner: {line.strip()!r}")
    if len(words) != 5:
        raise MalformedBannerError(f"banner needs 5 tokens, got {len(words)}")
    obj, fmt, field, sym = words[1:]
    if obj != "matrix":
        raise MalformedBannerError(f"unsupported object {obj!r}")
    if fmt not in _VALID["format"]:
        raise MalformedBannerError(f"unsupported format {fmt!r}")
    if field == "complex":
        raise UnsupportedFieldError("complex matrices are not supported")
    if field not in _VALID["field"]:
        raise MalformedBannerError(f"unsupported field {field!r}")
    if sym not in _VALID["symmetry"]:
        raise MalformedBannerError(f"unsupported symmetry {sym!r}")
    if fmt == "array" and field == "pattern":
        raise MalformedBannerError("pattern field requires coordinate format")
    return MatrixMarketHeader("matrix", fmt, field, sym)


def _size_line(fh) -> str:
    for raw in fh:
        text = raw.strip()
        if text and not text.startswith("%"):
            return text
    raise MalformedSizeError("missing size line")


def _parse_size(text: str, count: int) -> list[int]:
    words = text.split()
    if len(words) != count:
        raise MalformedSizeError(f"size line needs {count} integers, got {text!r}")
    try:
        dims = [int(w) for w in words]
    except ValueError:
        raise MalformedSizeError(f"size line is not integral: {text!r}") from None
    if min(dims) < 0:
        raise MalformedSizeError(f"negative size: {text!r}")
    return dims


def _coordinate_body(fh, header, rows, cols, nnz):
    width = 2 if header.field == "pattern" else 3
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # an empty body is legal when nnz == 0
        try:
            table = np.loadtxt(fh, comments="%", dtype=np.float64, ndmin=2)
        except ValueError as exc:
            raise MatrixMarketError(f"cannot parse entry data: {exc}") from None
    if table.size == 0:
        table = np.empty((0, width))
    elif table.shape[1] != width:
        raise MatrixMarketError(f"entries need {width} tokens per line, got {table.shape[1]}")
    if table.shape[0] != nnz:
        raise EntryCountError(f"declared {nnz} entries, file has {table.shape[0]}")
    fr, fc = table[:, 0], table[:, 1]
    r1, c1 = fr.astype(np.int64), fc.astype(np.int64)
    if np.any(fr != r1) or np.any(fc != c1):
        raise MatrixMarketError("non-integral coordinate index")
    bad = np.flatnonzero((r1 < 1) | (r1 > rows) | (c1 < 1) | (c1 > cols))
    if bad.size:
        k = bad[0]
        raise IndexBoundsError(f"entry ({r1[k]}, {c1[k]}) outside declared {rows}x{cols}")
    vals = np.ones(nnz) if width == 2 else table[:, 2].copy()
    return r1 - 1, c1 - 1, vals


def _array_body(fh, header, rows, cols):
    tokens = []
    for raw in fh:
        text = raw.strip()
        if text and not text.startswith("%"):
            tokens.extend(text.split())
    try:
        vals = np.array([float(t) for t in tokens], dtype=np.float64)
    except ValueError:
        bad = next(t for t in tokens if not _is_float(t))
        raise MatrixMarketError(f"cannot parse array value {bad!r}") from None
    # column-major enumeration: column j holds rows i0(j)..rows-1
    if header.symmetry == "general":
        ci, ri = np.divmod(np.arange(rows * cols, dtype=np.int64), max(rows, 1))
    else:  # square; lower triangle (with diagonal unless skew) column by column
        ci, ri = np.triu_indices(rows, k=0 if header.symmetry == "symmetric" else 1)
        ci, ri = ci.astype(np.int64), ri.astype(np.int64)
    if vals.size != ri.size:
        raise EntryCountError(f"declared {ri.size} array values, file has {vals.size}")
    return ri, ci, vals


def _is_float(tok: str) -> bool:
    try:
        float(tok)
    except ValueError:
        return False
    return True


def _mirror(ri, ci, vals, symmetry):
    if symmetry == "general" or ri.size == 0:
        return ri, ci, vals
    off = ri != ci
    sign = -1.0 if symmetry == "skew-symmetric" else 1.0
    return (np.concatenate([ri, ci[off]]), np.concatenate([ci, ri[off]]),
            np.concatenate([vals, sign * vals[off]]))


def _warn_on_duplicates(ri, ci, cols):
    if ri.size < 2:
        return
    w = max(cols, 1)
    key = np.sort(ri * w + ci)
    hit = np.flatnonzero(key[1:] == key[:-1])
    if hit.size:
        i, j = divmod(int(key[hit[0]]), w)
        warnings.warn(f"duplicate entry at ({i + 1}, {j + 1}); duplicates are summed",
                      DuplicateEntryWarning, stacklevel=4)


def read_entries(path):
    """Parse a Matrix Market file into ``(header, rows, cols, row_idxs, col_idxs, values)``:
    the raw (0-based, symmetry-expanded, not yet canonical) triplet stream the reference
    hands to ``coo_from_arrays`` (mmio.py:194-232).  Host-only; no device work."""
    with open(path, "r", encoding="ascii") as fh:
        first = fh.readline()
        if not first:
            raise MalformedBannerError("empty file")
        header = parse_banner(first)
        size = _size_line(fh)
        if header.format == "coordinate":
            rows, cols, nnz = _parse_size(size, 3)
        else:
            rows, cols = _parse_size(size, 2)
        if header.symmetry != "general" and rows != cols:
            raise MalformedSizeError(
                f"{header.symmetry} storage requires a square matrix, got {rows}x{cols}")
        if header.format == "coordinate":
            ri, ci, vals = _coordinate_body(fh, header, rows, cols, nnz)
        else:
            ri, ci, vals = _array_body(fh, header, rows, cols)
    ri, ci, vals = _mirror(ri, ci, vals, header.symmetry)
    _warn_on_duplicates(ri, ci, cols)
    return header, rows, cols, ri, ci, vals


def read_matrix_market(device, path, precision: Precision = Precision.double, format="Csr",
                       index_width: IndexWidth = IndexWidth.i32):
    """Read a Matrix Market file into device CSR (default) or COO storage
    (reference ``read_matrix_market`` mmio.py:194-232); canonicalisation runs on the GPU."""
    target = str(format).lower()
    if target not in ("csr", "coo"):
        raise MatrixMarketError(f"unknown target format {format!r}; expected 'Csr' or 'Coo'")
    _, rows, cols, ri, ci, vals = read_entries(path)
    coo = coo_from_arrays(device, rows, cols, ri, ci, vals, precision, index_width)
    return csr_from_coo(coo) if target == "csr" else coo


def write_matrix_market(m, path) -> None:
    """Write ``m`` as coordinate/real/general, 1-based, ``%.17g`` values, entries in
    canonical (row, column) order (reference mmio.py:235-244)."""
    r, c, v = m._entries_host()
    order = np.lexsort((c, r))
    with open(path, "w", encoding="ascii") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{m.rows} {m.cols} {len(v)}\n")
        fh.writelines("%d %d %.17g\n" % (int(r[k]) + 1, int(c[k]) + 1, float(v[k]))
                      for k in order)
