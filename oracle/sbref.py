"""ctypes + NumPy face of the CPU parity oracle (oracle/sbref.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs, never by the product
package.  Every routine restates a reference function (see sbref.cpp for the
file:line citations); the restatement is pinned against vectors produced by the
reference itself in tests/golden/ (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libsbref.so")

_VN = {np.dtype(np.float32): "float", np.dtype(np.float64): "double"}
_IN = {np.dtype(np.int32): "i32", np.dtype(np.int64): "i64"}

SOLVER_KINDS = {"cg": 0, "cgs": 1, "gmres": 2, "bicgstab": 3}
STOP_REASONS = {0: "residual", 1: "max_iters"}


class _Log(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("converged", ctypes.c_int32),
                ("stop_reason", ctypes.c_int32), ("status", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("status_iteration", ctypes.c_int64),
                ("history_len", ctypes.c_int64)]


class _Criteria(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int64), ("has_residual", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("reduction_factor", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc only; seconds)."""
    src = os.path.join(_HERE, "sbref.cpp")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.ref_hardware_threads.restype = ctypes.c_int
        for vn in ("float", "double"):
            getattr(_lib, f"ref_dot_{vn}").restype = ctypes.c_double
            getattr(_lib, f"ref_norm2_{vn}").restype = ctypes.c_double
            getattr(_lib, f"ref_coo_canonicalize_{vn}").restype = ctypes.c_int64
            for ix in ("i32", "i64"):
                getattr(_lib, f"ref_jacobi_create_{vn}_{ix}").restype = ctypes.c_int64
                getattr(_lib, f"ref_trsv_{vn}_{ix}").restype = ctypes.c_int
                getattr(_lib, f"ref_ilu0_{vn}_{ix}").restype = ctypes.c_int64
                getattr(_lib, f"ref_ic0_{vn}_{ix}").restype = ctypes.c_int64
    return _lib


def hardware_threads() -> int:
    return int(lib().ref_hardware_threads())


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


I64 = ctypes.c_int64
F64 = ctypes.c_double


# ------------------------------------------------------------------ BLAS-1
def dot(x, y, threads=1) -> float:
    x = np.ascontiguousarray(x)
    y = _c(y, x.dtype)
    return float(getattr(lib(), f"ref_dot_{_VN[x.dtype]}")(I64(x.size), _p(x), _p(y), threads))


def norm2(x, threads=1) -> float:
    x = np.ascontiguousarray(x)
    return float(getattr(lib(), f"ref_norm2_{_VN[x.dtype]}")(I64(x.size), _p(x), threads))


def axpy(alpha, x, y, threads=1) -> np.ndarray:
    """Returns a new y := alpha*x + y (inputs untouched)."""
    x = np.ascontiguousarray(x)
    out = np.array(y, dtype=x.dtype, copy=True)
    getattr(lib(), f"ref_axpy_{_VN[x.dtype]}")(I64(x.size), F64(alpha), _p(x), _p(out), threads)
    return out


def scal(alpha, x, threads=1) -> np.ndarray:
    out = np.array(x, copy=True)
    getattr(lib(), f"ref_scal_{_VN[out.dtype]}")(I64(out.size), F64(alpha), _p(out), threads)
    return out


def jacobi_apply(inv, b, threads=1) -> np.ndarray:
    inv = np.ascontiguousarray(inv)
    b = _c(b, inv.dtype)
    x = np.empty_like(b)
    getattr(lib(), f"ref_jacobi_apply_{_VN[inv.dtype]}")(I64(b.size), _p(inv), _p(b), _p(x), threads)
    return x


# ------------------------------------------------------------------ SpMV
def csr_spmv(row_ptrs, col_idxs, values, b, threads=1) -> np.ndarray:
    values = np.ascontiguousarray(values)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    b = _c(b, values.dtype)
    rows = row_ptrs.size - 1
    x = np.empty(rows, dtype=values.dtype)
    fn = getattr(lib(), f"ref_csr_spmv_{_VN[values.dtype]}_{_IN[col_idxs.dtype]}")
    fn(I64(rows), _p(row_ptrs), _p(col_idxs), _p(values), _p(b), _p(x), threads)
    return x


def coo_spmv(rows, row_idxs, col_idxs, values, b) -> np.ndarray:
    values = np.ascontiguousarray(values)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_idxs = _c(row_idxs, col_idxs.dtype)
    b = _c(b, values.dtype)
    x = np.empty(rows, dtype=values.dtype)
    fn = getattr(lib(), f"ref_coo_spmv_{_VN[values.dtype]}_{_IN[col_idxs.dtype]}")
    fn(I64(rows), I64(values.size), _p(row_idxs), _p(col_idxs), _p(values), _p(b), _p(x))
    return x


def jacobi_create(row_ptrs, col_idxs, values):
    """(inv_diag, None) on success, (None, row) on a singular diagonal."""
    values = np.ascontiguousarray(values)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    n = row_ptrs.size - 1
    inv = np.zeros(n, dtype=values.dtype)
    fn = getattr(lib(), f"ref_jacobi_create_{_VN[values.dtype]}_{_IN[col_idxs.dtype]}")
    row = int(fn(I64(n), _p(row_ptrs), _p(col_idxs), _p(values), _p(inv)))
    return (inv, None) if row < 0 else (None, row)


# ------------------------------------------------------------------ canonical layouts
def ell_from_csr(row_ptrs, col_idxs, values, stride_align=32):
    """ELL(w = max row length, stride = round_up(rows, stride_align)), column-major."""
    values = np.ascontiguousarray(values)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    rows = row_ptrs.size - 1
    lens = np.diff(row_ptrs)
    w = int(lens.max()) if rows else 0
    stride = -(-rows // stride_align) * stride_align
    ec = np.empty(w * stride, dtype=col_idxs.dtype)
    ev = np.empty(w * stride, dtype=values.dtype)
    fn = getattr(lib(), f"ref_ell_from_csr_{_VN[values.dtype]}_{_IN[col_idxs.dtype]}")
    fn(I64(rows), _p(row_ptrs), _p(col_idxs), _p(values), I64(w), I64(stride), _p(ec), _p(ev))
    return w, stride, ec, ev


def sellp_from_csr(row_ptrs, col_idxs, values, slice_size=64):
    values = np.ascontiguousarray(values)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    rows = row_ptrs.size - 1
    ns = -(-rows // slice_size)
    lens = np.diff(row_ptrs)
    pad = np.zeros(ns * slice_size, dtype=np.int64)
    pad[:rows] = lens
    total = int(pad.reshape(ns, slice_size).max(axis=1).sum()) if ns else 0
    sl = np.empty(ns, dtype=col_idxs.dtype)
    ss = np.empty(ns + 1, dtype=col_idxs.dtype)
    sc = np.empty(total * slice_size, dtype=col_idxs.dtype)
    sv = np.empty(total * slice_size, dtype=values.dtype)
    fn = getattr(lib(), f"ref_sellp_from_csr_{_VN[values.dtype]}_{_IN[col_idxs.dtype]}")
    fn(I64(rows), _p(row_ptrs), _p(col_idxs), _p(values), I64(slice_size), _p(sl), _p(ss),
       _p(sc), _p(sv))
    return sl, ss, sc, sv


def hybrid_from_csr(row_ptrs, col_idxs, values, ell_width, stride_align=32):
    """Hybrid(w): the first min(len_i, w) entries of each row go to ELL(w) (column-major,
    stride = round_up(rows, stride_align)); the rest go to a canonical COO tail."""
    col_idxs = np.ascontiguousarray(col_idxs)
    values = np.ascontiguousarray(values)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    rows = row_ptrs.size - 1
    w = int(ell_width)
    stride = -(-rows // stride_align) * stride_align
    ec = np.full(w * stride, -1, dtype=col_idxs.dtype)
    ev = np.zeros(w * stride, dtype=values.dtype)
    tail_r, tail_c, tail_v = [], [], []
    for i in range(rows):
        lo, hi = int(row_ptrs[i]), int(row_ptrs[i + 1])
        for k in range(hi - lo):
            if k < w:
                ec[k * stride + i] = col_idxs[lo + k]
                ev[k * stride + i] = values[lo + k]
            else:
                tail_r.append(i)
                tail_c.append(col_idxs[lo + k])
                tail_v.append(values[lo + k])
    return (w, stride, ec, ev, np.asarray(tail_r, dtype=col_idxs.dtype),
            np.asarray(tail_c, dtype=col_idxs.dtype), np.asarray(tail_v, dtype=values.dtype))


def hybrid_ell_width(row_lengths, quantile=0.8) -> int:
    """Hybrid ELL width rule (SURVEY.md §8 proposal): the 80th percentile of row lengths,
    taken as the length at sorted position floor(q*(rows-1))."""
    lens = np.sort(np.asarray(row_lengths, dtype=np.int64))
    if lens.size == 0:
        return 0
    return int(lens[int(np.floor(quantile * (lens.size - 1)))])


def ell_spmv(rows, w, stride, ecol, evals, b) -> np.ndarray:
    evals = np.ascontiguousarray(evals)
    ecol = np.ascontiguousarray(ecol)
    b = _c(b, evals.dtype)
    x = np.empty(rows, dtype=evals.dtype)
    fn = getattr(lib(), f"ref_ell_spmv_{_VN[evals.dtype]}_{_IN[ecol.dtype]}")
    fn(I64(rows), I64(w), I64(stride), _p(ecol), _p(evals), _p(b), _p(x))
    return x


def sellp_spmv(rows, slice_size, sl, ss, sc, sv, b) -> np.ndarray:
    sv = np.ascontiguousarray(sv)
    sc = np.ascontiguousarray(sc)
    b = _c(b, sv.dtype)
    x = np.empty(rows, dtype=sv.dtype)
    fn = getattr(lib(), f"ref_sellp_spmv_{_VN[sv.dtype]}_{_IN[sc.dtype]}")
    fn(I64(rows), I64(slice_size), _p(_c(sl, sc.dtype)), _p(_c(ss, sc.dtype)), _p(sc), _p(sv),
       _p(b), _p(x))
    return x


# ------------------------------------------------------------------ conversions
def coo_canonicalize(row_idxs, col_idxs, values, dtype=np.float64):
    """coo_from_arrays (formats.py:131-166) without the bounds check: returns
    canonical int64 (rows, cols) and summed values in ``dtype``."""
    ri = _c(row_idxs, np.int64)
    ci = _c(col_idxs, np.int64)
    v = _c(values, dtype)
    m = ri.size
    orow = np.empty(max(m, 1), np.int64)
    ocol = np.empty(max(m, 1), np.int64)
    oval = np.empty(max(m, 1), v.dtype)
    nnz = int(getattr(lib(), f"ref_coo_canonicalize_{_VN[v.dtype]}")(
        I64(m), _p(ri), _p(ci), _p(v), _p(orow), _p(ocol), _p(oval)))
    return orow[:nnz].copy(), ocol[:nnz].copy(), oval[:nnz].copy()


def csr_row_ptrs(row_idxs, rows, dtype=np.int32) -> np.ndarray:
    """csr_from_coo (formats.py:184-191): bincount + cumsum."""
    counts = np.bincount(np.asarray(row_idxs, np.int64), minlength=rows) if len(row_idxs) \
        else np.zeros(rows, np.int64)
    rp = np.zeros(rows + 1, dtype=dtype)
    np.cumsum(counts, out=rp[1:])
    return rp


# ------------------------------------------------------------------ solvers
@dataclass
class Log:
    iterations: int
    converged: bool
    stop_reason: str
    status: int                   # 0 ok, 1 breakdown, 2 numeric failure
    status_iteration: int
    residual_history: list = field(default_factory=list)


def solve(kind, row_ptrs, col_idxs, values, b, x0=None, inv_diag=None, max_iters=1000,
          reduction_factor=None, krylov_dim=30, threads=1):
    """Run one of cg / cgs / gmres / bicgstab; returns (Log, x)."""
    values = np.ascontiguousarray(values)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    n = row_ptrs.size - 1
    b = _c(b, values.dtype)
    x = np.zeros(n, values.dtype) if x0 is None else np.array(x0, dtype=values.dtype, copy=True)
    inv = None if inv_diag is None else _c(inv_diag, values.dtype)
    crit = _Criteria(int(max_iters), 0 if reduction_factor is None else 1, 0,
                     float(reduction_factor or 0.0))
    cap = int(max_iters)
    hist = np.zeros(max(cap, 1), np.float64)
    log = _Log()
    fn = getattr(lib(), f"ref_solve_{_VN[values.dtype]}_{_IN[col_idxs.dtype]}")
    fn(ctypes.c_int(SOLVER_KINDS[kind]), I64(n), _p(row_ptrs), _p(col_idxs), _p(values),
       None if inv is None else _p(inv), _p(b), _p(x), ctypes.byref(crit), I64(krylov_dim),
       _p(hist), I64(cap), ctypes.byref(log), ctypes.c_int(threads))
    out = Log(int(log.iterations), bool(log.converged), STOP_REASONS.get(log.stop_reason, "?"),
              int(log.status), int(log.status_iteration),
              hist[: min(int(log.history_len), cap)].tolist())
    return out, x


# ---------------------------------------------------------------- ILU(0) / IC(0) / SpTRSV
def trsv(row_ptrs, col_idxs, values, b, lower=True, unit_diag=False):
    """_kernels.solve_lower / solve_upper: returns (status, row, x) with status 0 ok,
    1 entry on the wrong side of the diagonal, 2 missing / zero diagonal."""
    values = np.ascontiguousarray(values)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    n = row_ptrs.size - 1
    b = _c(b, values.dtype)
    x = np.zeros(n, values.dtype)
    row = I64(0)
    fn = getattr(lib(), f"ref_trsv_{_VN[values.dtype]}_{_IN[col_idxs.dtype]}")
    st = fn(I64(n), _p(row_ptrs), _p(col_idxs), _p(values), _p(b), _p(x), int(lower), int(unit_diag),
            ctypes.byref(row))
    return int(st), int(row.value), x


def ilu0(row_ptrs, col_idxs, values):
    """ilu0_factorize on the stored pattern: (zero_pivot_row or -1, factored values)."""
    vals = np.array(values, copy=True)
    col_idxs = np.ascontiguousarray(col_idxs)
    row_ptrs = _c(row_ptrs, col_idxs.dtype)
    fn = getattr(lib(), f"ref_ilu0_{_VN[vals.dtype]}_{_IN[col_idxs.dtype]}")
    return int(fn(I64(row_ptrs.size - 1), _p(row_ptrs), _p(col_idxs), _p(vals))), vals


def split_lu(row_ptrs, col_idxs, values, lower_incl_diag=False):
    """_split_lu (precond.py:190-202): strict lower (or lower incl. diagonal) / the rest."""
    rp = np.asarray(row_ptrs, np.int64)
    n = rp.size - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    cols = np.asarray(col_idxs)
    m = cols <= rows if lower_incl_diag else cols < rows
    def part(mask):
        ptr = np.concatenate([[0], np.cumsum(np.bincount(rows[mask], minlength=n))])
        return ptr.astype(cols.dtype), cols[mask].copy(), np.asarray(values)[mask].copy()
    return part(m), part(~m)


def ic0(row_ptrs, col_idxs, values):
    """ic0_factorize: (pivot_error_row or -1, (lp, lc, lv)) on the lower pattern of A."""
    (lp, lc, la), _ = split_lu(row_ptrs, col_idxs, values, lower_incl_diag=True)
    out = np.zeros_like(la)
    fn = getattr(lib(), f"ref_ic0_{_VN[la.dtype]}_{_IN[lc.dtype]}")
    st = int(fn(I64(lp.size - 1), _p(lp), _p(lc), _p(la), _p(out)))
    return st, (lp, lc, out)
