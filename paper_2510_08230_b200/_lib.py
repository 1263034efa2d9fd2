"""ctypes binding of libsparseb200.so (the C ABI declared in include/sparseb200.h).

This is the ONLY way the package reaches compute: there is no CPU fallback.  If
the library is missing or cannot be loaded, every operation raises
:class:`LibraryUnavailableError` loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .sparseops import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARSEB200_LIB") or os.path.join(_HERE, "libsparseb200.so")

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t


class LibraryUnavailableError(RuntimeError):
    kind = "library-unavailable"


# ------------------------------------------------------------------ structs (sparseb200.h)
class SbError(ctypes.Structure):
    _fields_ = [("code", c_i32), ("pad", c_i32), ("row", c_i64), ("iteration", c_i64),
                ("msg", ctypes.c_char * 256)]


class SbDense(ctypes.Structure):
    _fields_ = [("data", c_vp), ("rows", c_i64), ("cols", c_i64), ("stride", c_i64)]


class SbRowStats(ctypes.Structure):
    _fields_ = [("rows", c_i64), ("nnz", c_i64), ("min_len", c_i64), ("max_len", c_i64),
                ("empty_rows", c_i64), ("mean_len", c_f64), ("std_len", c_f64),
                ("max_block_nnz", c_i64 * 4)]


class SbCsrPlan(ctypes.Structure):
    _fields_ = [("kernel", c_i32), ("block_rows", c_i32), ("nnz_cap", c_i32), ("nnz_cap256", c_i32),
                ("num_tiles", c_i64), ("items_per_tile", c_i64), ("tile_rows", c_vp),
                ("tile_nnz", c_vp), ("carry_rows", c_vp), ("carry_vals", c_vp)]


class SbCsr(ctypes.Structure):
    _fields_ = [("rows", c_i64), ("cols", c_i64), ("nnz", c_i64), ("row_ptrs", c_vp),
                ("col_idxs", c_vp), ("values", c_vp), ("plan", ctypes.POINTER(SbCsrPlan))]


class SbCooPlan(ctypes.Structure):
    _fields_ = [("num_tiles", c_i64), ("carry_rows", c_vp), ("carry_vals", c_vp),
                ("row_ptrs", c_vp), ("csr_plan", ctypes.c_void_p)]


class SbCoo(ctypes.Structure):
    _fields_ = [("rows", c_i64), ("cols", c_i64), ("nnz", c_i64), ("row_idxs", c_vp),
                ("col_idxs", c_vp), ("values", c_vp), ("plan", ctypes.POINTER(SbCooPlan))]


class SbEll(ctypes.Structure):
    _fields_ = [("rows", c_i64), ("cols", c_i64), ("width", c_i64), ("stride", c_i64),
                ("col_idxs", c_vp), ("values", c_vp)]


class SbSellp(ctypes.Structure):
    _fields_ = [("rows", c_i64), ("cols", c_i64), ("slice_size", c_i64), ("num_slices", c_i64),
                ("slice_lengths", c_vp), ("slice_sets", c_vp), ("col_idxs", c_vp),
                ("values", c_vp), ("max_block_entries", c_i64), ("row_perm", c_vp),
                ("piece_plan", c_vp), ("num_pieces", c_i64), ("num_split", c_i64),
                ("piece_entries", c_i64), ("carry", c_vp)]


class SbHybrid(ctypes.Structure):
    _fields_ = [("ell", SbEll), ("coo", SbCoo)]


class SbMatrix(ctypes.Structure):
    _fields_ = [("format", c_i32), ("pad", c_i32), ("mat", c_vp)]


class SbCriteria(ctypes.Structure):
    _fields_ = [("max_iters", c_i64), ("has_residual", c_i32), ("pad", c_i32),
                ("reduction_factor", c_f64)]


class SbLog(ctypes.Structure):
    _fields_ = [("iterations", c_i64), ("converged", c_i32), ("stop_reason", c_i32),
                ("history_len", c_i64), ("history", ctypes.POINTER(c_f64)),
                ("history_cap", c_i64)]


class SbDistPart(ctypes.Structure):
    _fields_ = [("a", SbMatrix), ("num_views", c_i32), ("num_neighbors", c_i32),
                ("views", SbMatrix * 3), ("view_row0", c_i64 * 3), ("n_local", c_i64),
                ("n_ghost", c_i64), ("nbr", ctypes.POINTER(c_i32)),
                ("send_count", ctypes.POINTER(c_i64)), ("send_lo", ctypes.POINTER(c_i64)),
                ("send_off", ctypes.POINTER(c_i64)), ("recv_count", ctypes.POINTER(c_i64)),
                ("recv_off", ctypes.POINTER(c_i64)), ("send_idx", c_vp), ("send_buf", c_vp),
                ("inv_diag", c_vp), ("b", SbDense), ("x", SbDense), ("workspace", c_vp)]


class SbTriPrecond(ctypes.Structure):
    _fields_ = [("l", ctypes.POINTER(SbCsr)), ("l_unit", c_i32), ("pad", c_i32),
                ("u", ctypes.POINTER(SbCsr)), ("workspace", c_vp)]


FMT_CSR, FMT_COO, FMT_ELL, FMT_SELLP, FMT_HYBRID = 0, 1, 2, 3, 4
CSR_AUTO, CSR_STRICT, CSR_STREAM, CSR_VECTOR, CSR_MERGE, CSR_TILE = 0, 1, 2, 3, 4, 5
CSR_KERNELS = {"auto": CSR_AUTO, "strict": CSR_STRICT, "stream": CSR_STREAM,
               "vector": CSR_VECTOR, "merge": CSR_MERGE, "tile": CSR_TILE}
SOLVER_CG, SOLVER_CGS, SOLVER_GMRES, SOLVER_BICGSTAB = 0, 1, 2, 3

P = ctypes.POINTER
VALUES = ("float", "double")
INDICES = ("i32", "i64")

# name -> (restype, argtypes); the suffixed families are expanded below
_VALUE_PROTOS = {
    "sb_dot_{v}": (c_i32, [P(SbDense), P(SbDense), P(c_f64), c_vp, c_vp, P(SbError)]),
    "sb_norm2_{v}": (c_i32, [P(SbDense), P(c_f64), c_vp, c_vp, P(SbError)]),
    "sb_axpy_{v}": (c_i32, [c_f64, P(SbDense), P(SbDense), c_vp, P(SbError)]),
    "sb_scal_{v}": (c_i32, [c_f64, P(SbDense), c_vp, P(SbError)]),
    "sb_copy_{v}": (c_i32, [P(SbDense), P(SbDense), c_vp, P(SbError)]),
    "sb_fill_{v}": (c_i32, [P(SbDense), c_f64, c_vp, P(SbError)]),
    "sb_jacobi_apply_{v}": (c_i32, [c_vp, P(SbDense), P(SbDense), c_vp, P(SbError)]),
}
_SOLVE = [P(SbMatrix), c_vp, P(SbDense), P(SbDense), P(SbCriteria), c_vp, P(SbLog), c_vp,
          P(SbError)]
_VI_PROTOS = {
    "sb_csr_spmv_{v}_{i}": (c_i32, [P(SbCsr), P(SbDense), P(SbDense), c_vp, P(SbError)]),
    "sb_coo_spmv_{v}_{i}": (c_i32, [P(SbCoo), P(SbDense), P(SbDense), c_vp, P(SbError)]),
    "sb_ell_spmv_{v}_{i}": (c_i32, [P(SbEll), P(SbDense), P(SbDense), c_vp, P(SbError)]),
    "sb_sellp_spmv_{v}_{i}": (c_i32, [P(SbSellp), P(SbDense), P(SbDense), c_vp, P(SbError)]),
    "sb_hybrid_spmv_{v}_{i}": (c_i32, [P(SbHybrid), P(SbDense), P(SbDense), c_vp, P(SbError)]),
    "sb_apply_advanced_{v}_{i}": (c_i32, [P(SbMatrix), c_f64, P(SbDense), c_f64, P(SbDense),
                                          c_vp, c_vp, P(SbError)]),
    "sb_jacobi_create_{v}_{i}": (c_i32, [P(SbCsr), c_vp, c_vp, c_vp, P(SbError)]),
    "sb_ell_from_csr_{v}_{i}": (c_i32, [P(SbCsr), P(SbEll), c_vp, P(SbError)]),
    "sb_sellp_from_csr_{v}_{i}": (c_i32, [P(SbCsr), P(SbSellp), c_vp, P(SbError)]),
    "sb_hybrid_from_csr_{v}_{i}": (c_i32, [P(SbCsr), c_vp, P(SbHybrid), c_vp, P(SbError)]),
    "sb_coo_from_arrays_{v}_{i}": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                           c_vp, c_vp, c_sz, P(c_i64), c_vp, P(SbError)]),
    "sb_cg_solve_{v}_{i}": (c_i32, _SOLVE),
    "sb_cgs_solve_{v}_{i}": (c_i32, _SOLVE),
    "sb_bicgstab_solve_{v}_{i}": (c_i32, _SOLVE),
    "sb_gmres_solve_{v}_{i}": (c_i32, [P(SbMatrix), c_vp, P(SbDense), P(SbDense), P(SbCriteria),
                                       c_i64, c_vp, P(SbLog), c_vp, P(SbError)]),
    "sb_dist_cg_solve_{v}_{i}": (c_i32, [P(SbDistPart), c_i32, c_vp, P(SbCriteria), P(SbLog),
                                         c_vp, P(SbError)]),
    "sb_dist_bicgstab_solve_{v}_{i}": (c_i32, [P(SbDistPart), c_i32, c_vp, P(SbCriteria), P(SbLog),
                                               c_vp, P(SbError)]),
    "sb_dist_gmres_solve_{v}_{i}": (c_i32, [P(SbDistPart), c_i32, c_vp, P(SbCriteria), c_i64,
                                            P(SbLog), c_vp, P(SbError)]),
    "sb_csr_trisolve_{v}_{i}": (c_i32, [P(SbCsr), c_i32, c_i32, P(SbDense), P(SbDense), c_vp, c_vp,
                                        P(SbError)]),
    "sb_csr_tri_check_{v}_{i}": (c_i32, [P(SbCsr), c_i32, c_i32, c_vp, c_vp, P(SbError)]),
    "sb_ilu0_{v}_{i}": (c_i32, [P(SbCsr), c_vp, c_vp, c_vp, c_vp, P(SbError)]),
    "sb_ic0_{v}_{i}": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, P(SbError)]),
    "sb_csr_split_scatter_{v}_{i}": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                             c_vp, c_vp, P(SbError)]),
    "sb_cg_solve_tri_{v}_{i}": (c_i32, [P(SbMatrix), P(SbTriPrecond), P(SbDense), P(SbDense),
                                        P(SbCriteria), c_vp, P(SbLog), c_vp, P(SbError)]),
    "sb_gmres_solve_tri_{v}_{i}": (c_i32, [P(SbMatrix), P(SbTriPrecond), P(SbDense), P(SbDense),
                                           P(SbCriteria), c_i64, c_vp, P(SbLog), c_vp, P(SbError)]),
    "sb_cgs_solve_tri_{v}_{i}": (c_i32, [P(SbMatrix), P(SbTriPrecond), P(SbDense), P(SbDense),
                                         P(SbCriteria), c_vp, P(SbLog), c_vp, P(SbError)]),
    "sb_bicgstab_solve_tri_{v}_{i}": (c_i32, [P(SbMatrix), P(SbTriPrecond), P(SbDense), P(SbDense),
                                              P(SbCriteria), c_vp, P(SbLog), c_vp, P(SbError)]),
}
_I_PROTOS = {
    "sb_csr_row_stats_{i}": (c_i32, [c_i64, c_vp, c_vp, P(SbRowStats), c_vp, P(SbError)]),
    "sb_csr_plan_build_{i}": (c_i32, [c_i64, c_i64, c_vp, P(SbCsrPlan), c_vp, P(SbError)]),
    "sb_csr_row_ptrs_from_coo_{i}": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, P(SbError)]),
    "sb_coo_row_idxs_from_csr_{i}": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, P(SbError)]),
    "sb_sellp_slices_{i}": (c_i32, [c_i64, c_vp, c_i64, c_vp, c_vp, P(c_i64), c_vp, P(SbError)]),
    "sb_hybrid_tail_ptrs_{i}": (c_i32, [c_i64, c_vp, c_i64, c_vp, P(c_i64), c_vp, P(SbError)]),
    "sb_stencil_csr_double_{i}": (c_i32, [c_i64, c_i32, c_f64, c_i64, c_i64, c_vp, c_vp, c_vp,
                                          c_vp, P(SbError)]),
    "sb_stencil_csr_float_{i}": (c_i32, [c_i64, c_i32, c_f64, c_i64, c_i64, c_vp, c_vp, c_vp,
                                         c_vp, P(SbError)]),
    "sb_csr_split_count_{i}": (c_i32, [c_i64, c_vp, c_vp, c_i32, c_vp, c_vp, P(SbError)]),
}
_PLAIN_PROTOS = {
    "sb_version": (c_i32, []),
    "sb_status_string": (ctypes.c_char_p, [c_i32]),
    "sb_set_graph_mode": (None, [c_i32]),
    "sb_set_cg_fused": (None, [c_i32]),
    "sb_set_cg_sync": (None, [c_i32]),
    "sb_set_cg_xw": (None, [c_i32]),
    "sb_cg_last_loop": (c_i32, []),
    "sb_cg_last_block_rows": (c_i32, []),
    "sb_tri_workspace_bytes": (c_sz, [c_i64]),
    "sb_csr_plan_select": (c_i32, [P(SbRowStats), c_i32, c_i32, c_i32, P(SbCsrPlan),
                                   P(SbError)]),
    "sb_coo_tile_entries": (c_i64, []),
    "sb_reduce_workspace_bytes": (c_sz, []),
    "sb_coo_from_arrays_workspace_bytes": (c_sz, [c_i64]),
    "sb_solver_workspace_bytes": (c_sz, [c_i32, c_i32, c_i64, c_i64, c_i64]),
    "sb_nccl_unique_id": (c_i32, [ctypes.c_char_p, P(SbError)]),
    "sb_nccl_comm_init": (c_i32, [c_i32, ctypes.c_char_p, c_i32, P(c_vp), P(SbError)]),
    "sb_nccl_comm_destroy": (c_i32, [c_vp, P(SbError)]),
    "sb_dist_workspace_bytes": (c_sz, [c_i32, c_i64, c_i64, c_i64]),
    "sb_dist_solver_workspace_bytes": (c_sz, [c_i32, c_i32, c_i64, c_i64, c_i64, c_i64]),
}


def all_prototypes() -> dict:
    out = dict(_PLAIN_PROTOS)
    for name, proto in _VALUE_PROTOS.items():
        for v in VALUES:
            out[name.format(v=v)] = proto
    for name, proto in _VI_PROTOS.items():
        for v in VALUES:
            for i in INDICES:
                out[name.format(v=v, i=i)] = proto
    for name, proto in _I_PROTOS.items():
        for i in INDICES:
            out[name.format(i=i)] = proto
    return out


_lock = threading.Lock()
_lib = None
_load_error = None


def load(path: str = LIB_PATH):
    """Load the library (once) and attach prototypes; raises loudly on failure."""
    global _lib, _load_error
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            _load_error = f"{path} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`"
            raise LibraryUnavailableError(_load_error)
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:  # pragma: no cover - environment specific
            _load_error = f"cannot load {path}: {exc}"
            raise LibraryUnavailableError(_load_error) from exc
        for name, (res, args) in all_prototypes().items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if os.environ.get("SPARSEB200_GRAPH", "1") == "0":
            # host-polled solver loops (profilers cannot see kernels inside graphs
            # that contain conditional nodes); same kernels, same order
            lib.sb_set_graph_mode(0)
        _lib = lib
        return lib


def fn(name: str):
    return getattr(load(), name)


# ------------------------------------------------------------------ status -> exceptions
def raise_for(status: int, err: SbError):
    """Map a C status onto the reference's exception classes (errors.py:8-131)."""
    if status == 0:
        return
    msg = err.msg.decode(errors="replace") if err.msg else ""
    if status == 1:
        raise E.InvalidArgumentError(msg)
    if status == 2:
        raise E.DimensionMismatchError(msg)
    if status == 3:
        raise E.PrecisionMismatchError(msg)
    if status == 4:
        raise E.UnsupportedFeatureError(msg)
    if status == 5:
        raise E.IndexBoundsError(msg)
    if status == 6:
        raise E.BreakdownError(int(err.iteration), msg)
    if status == 7:
        raise E.NumericFailureError(msg)
    if status == 8:
        raise E.SingularDiagonalError(int(err.row), msg)
    if status == 10:
        raise E.CommunicationError(msg)
    if status == 11:
        raise E.ZeroPivotError(int(err.row), msg)
    if status == 12:
        raise E.IndefinitePivotError(int(err.row), msg)
    if status == 13:
        raise E.NotTriangularError(int(err.row), msg)
    if status == 14:
        raise E.SingularTriangleError(int(err.row), msg)
    raise E.DeviceError(f"{msg} (status {status})")


def call(name: str, *args):
    """Invoke an sb_* function that takes a trailing sb_error*; raise on failure."""
    err = SbError()
    status = fn(name)(*args, ctypes.byref(err))
    raise_for(status, err)
