"""Row-partitioned Krylov solves across GPUs.

Decomposition: rank r of P owns the contiguous rows ``partition(n, P)[r]`` (the
reference's own row partition, core.py:173-183).  Its local CSR keeps those rows with
columns renumbered to ``[own rows 0..n_local) | ghosts n_local..)``; ghosts are the
off-rank columns it reads, sorted, hence grouped by owner.  The halo pattern per
neighbour: the rows it must send (a contiguous range for banded matrices such as the
stencils, else an index list) and the slot of the rows it receives.  When the rows
that read ghosts form a prefix and a suffix of the local block (true for slab
partitions of the stencils), the SpMV is split into an interior view that runs while
the halo is in flight and the boundary views that run after it.

Solvers (libsparseb200 ``sb_dist_{cg,bicgstab,gmres}_solve_*``, csrc/dist_krylov.cu):
DistCg, DistBicgstab, DistGmres -- the single-GPU solvers' fused steps on the local rows,
every reduction's local totals summed across ranks before the unchanged finaliser runs.

Transports:
* NCCL: one rank per GPU, grouped ncclSend/ncclRecv halos and ncclAllReduce of the fused
  dot partials, captured into CUDA graphs (``NcclComm`` builds the communicator; the
  unique id travels through torch.distributed);
* loopback: all P partitions on ONE GPU, halos as device copies -- the single-GPU test of
  the decomposition (NCCL refuses two ranks on one device).

The host logic (this module) is plain torch and runs on CPU tensors too, which is how
tests/test_dist_host.py checks it with the gloo backend at world size 2.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import gen
from .sparseops import errors as E
from .sparseops.core import Device, IndexWidth, Precision
from .sparseops.formats import CsrMatrix, _ptr, _stream
from .sparseops.solvers import ConvergenceLog, _criteria_struct, validate_criteria

__all__ = ["partition", "LocalPattern", "localize", "exchange_send_lists", "DistPartition",
           "stencil_partition", "csr_partition", "NcclComm", "DistCg", "DistBicgstab", "DistGmres"]


def partition(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous row blocks whose sizes differ by at most one (core.py:173-183)."""
    base, rem = divmod(n, parts)
    out, lo = [], 0
    for t in range(parts):
        hi = lo + base + (1 if t < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


@dataclass
class LocalPattern:
    """Host-side description of one partition (everything but the device matrix)."""

    rank: int
    lo: int
    hi: int
    n_ghost: int
    ghosts: torch.Tensor                     # global indices of the ghost columns (sorted)
    recv: dict = field(default_factory=dict)  # owner -> (offset in ghost region, count)
    send: dict = field(default_factory=dict)  # dest -> local rows to send (int64 tensor)
    boundary_rows: torch.Tensor | None = None  # local rows reading at least one ghost

    @property
    def n_local(self):
        return self.hi - self.lo

    def interior(self):
        """(prefix, suffix) boundary-row counts if boundary rows are exactly a prefix plus
        a suffix of the local block (SpMV overlap possible), else None."""
        b = self.boundary_rows
        if b is None or b.numel() == 0:
            return (0, 0)
        b = b.cpu()
        n = self.n_local
        pre = int((b == torch.arange(b.numel())).sum().item())
        tail = b[pre:]
        suf = tail.numel()
        if suf and not torch.equal(tail, torch.arange(n - suf, n)):
            return None
        return (pre, suf)


def localize(row_ptrs: torch.Tensor, col_idxs: torch.Tensor, lo: int, hi: int, bounds, rank: int):
    """Renumber the global columns of rows [lo, hi) to [own | ghosts]; returns the local
    column index tensor (same dtype) and the LocalPattern (without send lists)."""
    ci = col_idxs.long()
    own = (ci >= lo) & (ci < hi)
    ghosts = torch.unique(ci[~own])  # sorted
    n_local = hi - lo
    local = torch.where(own, ci - lo, n_local + torch.searchsorted(ghosts, ci))
    starts = torch.tensor([b[0] for b in bounds], device=ci.device)
    owners = torch.searchsorted(starts, ghosts, right=True) - 1
    recv = {}
    if ghosts.numel():
        uo, counts = torch.unique_consecutive(owners, return_counts=True)
        off = 0
        for o, c in zip(uo.tolist(), counts.tolist()):
            recv[int(o)] = (off, int(c))
            off += int(c)
    counts_per_row = (row_ptrs[1:] - row_ptrs[:-1]).long()
    row_of = torch.repeat_interleave(torch.arange(n_local, device=ci.device), counts_per_row)
    boundary = torch.unique(row_of[~own])
    pat = LocalPattern(rank, lo, hi, int(ghosts.numel()), ghosts, recv, {}, boundary)
    return local.to(col_idxs.dtype), pat


def send_lists_from(patterns_ghosts: dict, rank: int, lo: int, hi: int, device) -> dict:
    """Rows this rank must send: for every other rank s, the ghosts of s owned here."""
    out = {}
    for s, gh in patterns_ghosts.items():
        if s == rank:
            continue
        g = torch.as_tensor(gh, dtype=torch.int64, device=device)
        mine = g[(g >= lo) & (g < hi)]
        if mine.numel():
            out[int(s)] = mine - lo
    return out


def exchange_send_lists(pat: LocalPattern, group=None) -> LocalPattern:
    """Fill ``pat.send`` by exchanging ghost lists with torch.distributed (any backend)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, pat.ghosts.cpu().numpy(), group=group)
    pat.send = send_lists_from(dict(enumerate(gathered)), pat.rank, pat.lo, pat.hi,
                               pat.ghosts.device)
    return pat


class DistPartition:
    """Device-side partition: local CSR (+ SpMV views), halo buffers, Jacobi, C struct."""

    def __init__(self, device: Device, pat: LocalPattern, row_ptrs, local_cols, values,
                 global_cols=None, jacobi: bool = True):
        self.device = device
        self.pat = pat
        nl, ng = pat.n_local, pat.n_ghost
        dev = device.torch
        self.matrix = CsrMatrix(device, nl, nl + ng, row_ptrs, local_cols, values)
        self.n_local, self.n_ghost = nl, ng
        split = pat.interior()
        self.views, self.view_row0 = [], []
        if split is not None and ng > 0 and nl > 0:
            pre, suf = split
            # view boundaries on multiples of 4 rows: every view's row_ptrs slice (and its
            # output offset) stays 16-byte aligned for the TMA-staged SpMV; moving rows from
            # the interior view into a boundary view is always correct
            pre = min(nl, (pre + 3) // 4 * 4)
            tail0 = max(pre, (nl - suf) // 4 * 4)
            ranges = [(pre, tail0), (0, pre), (tail0, nl)]
            for a, b in ranges:
                if b > a:
                    self.views.append(CsrMatrix(device, b - a, nl + ng, self.matrix.row_ptrs[a:b + 1],
                                                self.matrix.col_idxs, self.matrix.values))
                    self.view_row0.append(a)
            if not ranges[0][1] > ranges[0][0]:  # no interior rows: no overlap
                self.views, self.view_row0 = [], []
        nbrs = sorted(set(pat.recv) | set(pat.send))
        self.nbr = nbrs
        send_cnt, send_lo, send_off, recv_cnt, recv_off, idx = [], [], [], [], [], []
        off = 0
        for s in nbrs:
            rows = pat.send.get(s)
            c = 0 if rows is None else int(rows.numel())
            contiguous = c > 0 and int(rows[-1] - rows[0]) == c - 1 and bool(
                torch.all(rows[1:] - rows[:-1] == 1))
            send_cnt.append(c)
            send_lo.append(int(rows[0]) if contiguous else -1)
            send_off.append(off)
            if c and not contiguous:
                idx.append(rows.to(torch.int64))
            else:
                idx.append(torch.zeros(c, dtype=torch.int64, device=rows.device if c else dev))
            off += c
            ro, rc = pat.recv.get(s, (0, 0))
            recv_cnt.append(rc)
            recv_off.append(ro)
        self.send_idx = (torch.cat(idx).to(dev) if idx else torch.zeros(1, dtype=torch.int64, device=dev))
        self.send_buf = torch.empty(max(off, 1), dtype=values.dtype, device=dev)
        self._host = dict(
            nbr=(ctypes.c_int32 * max(len(nbrs), 1))(*nbrs),
            send_count=(ctypes.c_int64 * max(len(nbrs), 1))(*send_cnt),
            send_lo=(ctypes.c_int64 * max(len(nbrs), 1))(*send_lo),
            send_off=(ctypes.c_int64 * max(len(nbrs), 1))(*send_off),
            recv_count=(ctypes.c_int64 * max(len(nbrs), 1))(*recv_cnt),
            recv_off=(ctypes.c_int64 * max(len(nbrs), 1))(*recv_off))
        self.inv_diag = self._jacobi(global_cols) if jacobi else None
        self.workspace = None

    def _jacobi(self, global_cols) -> torch.Tensor:
        """Local inverse diagonal by the device jacobi_create on the slab with columns
        shifted by -lo: still sorted per row, and the diagonal of local row i sits at
        column i (the renumbered local columns are not sorted)."""
        from .sparseops import jacobi_create

        if global_cols is None:
            raise E.InvalidArgumentError("Jacobi needs the slab's global column indices")
        shifted = (global_cols.long() - self.pat.lo).to(global_cols.dtype)
        sq = CsrMatrix(self.device, self.n_local, self.n_local, self.matrix.row_ptrs, shifted,
                       self.matrix.values, kernel="strict")
        return jacobi_create(sq).inv_diag

    def struct(self, b, x, cap: int, kind: int = _lib.SOLVER_CG, dim: int = 0,
               precond: bool = True) -> _lib.SbDistPart:
        need = self._ws_bytes(cap, kind, dim)
        if self.workspace is None or self.workspace.numel() < need:
            self.workspace = torch.zeros(need, dtype=torch.uint8, device=self.device.torch)
        P = _lib.SbDistPart()
        P.a = self.matrix.matrix_struct()
        P.num_views = len(self.views)
        P.num_neighbors = len(self.nbr)
        self._view_structs = [v.matrix_struct() for v in self.views]
        for k, vs in enumerate(self._view_structs):
            P.views[k] = vs
            P.view_row0[k] = self.view_row0[k]
        P.n_local, P.n_ghost = self.n_local, self.n_ghost
        h = self._host
        P.nbr, P.send_count, P.send_lo, P.send_off = h["nbr"], h["send_count"], h["send_lo"], h["send_off"]
        P.recv_count, P.recv_off = h["recv_count"], h["recv_off"]
        P.send_idx = self.send_idx.data_ptr()
        P.send_buf = self.send_buf.data_ptr()
        P.inv_diag = self.inv_diag.data_ptr() if (precond and self.inv_diag is not None) else None
        P.b = b.struct()
        P.x = x.struct()
        P.workspace = self.workspace.data_ptr()
        return P

    def _ws_bytes(self, cap, kind=_lib.SOLVER_CG, dim=0):
        return int(_lib.fn("sb_dist_solver_workspace_bytes")(kind, self.matrix.precision.itemsize,
                                                              self.n_local, self.n_ghost, dim, cap))


def stencil_partition(device: Device, p: int, rank: int, world: int, dim: int = 3, c: float = 0.0,
                      precision: Precision = Precision.double,
                      index_width: IndexWidth = IndexWidth.i32, exchange=None):
    """This rank's slab of the dim-D stencil, generated directly on its GPU.

    ``exchange``: None -> closed-form send lists (every rank's ghost set is computed
    locally; valid for the stencils), or a callable(LocalPattern) -> LocalPattern
    (e.g. exchange_send_lists) for the general path."""
    n = p ** dim
    bounds = partition(n, world)
    lo, hi = bounds[rank]
    rp, ci, val = gen.stencil_rows(device, p, lo, hi, dim, c, precision, index_width)
    local, pat = localize(rp, ci, lo, hi, bounds, rank)
    if exchange is None:
        ghosts = {}
        for s in range(world):  # ghosts of every rank, from the same generator
            if s == rank:
                continue
            slo, shi = bounds[s]
            if shi == slo:
                continue
            # neighbours in a stencil are within p^(dim-1) rows: only adjacent slabs matter
            if shi <= lo - p ** (dim - 1) or slo >= hi + p ** (dim - 1):
                continue
            srp, sci, _ = gen.stencil_rows(device, p, slo, shi, dim, c, precision, index_width)
            _, spat = localize(srp, sci, slo, shi, bounds, s)
            ghosts[s] = spat.ghosts
        pat.send = send_lists_from(ghosts, rank, lo, hi, device.torch)
    else:
        pat = exchange(pat)
    return DistPartition(device, pat, rp, local, val, global_cols=ci)


def csr_partition(device: Device, row_ptrs, col_idxs, values, rank: int, world: int,
                  all_patterns: dict | None = None, exchange=None):
    """This rank's rows of a global host CSR (NumPy / torch); send lists from
    ``exchange`` (torch.distributed) or from the ghost lists in ``all_patterns``."""
    rp = torch.as_tensor(np.asarray(row_ptrs))
    n = rp.numel() - 1
    bounds = partition(n, world)
    lo, hi = bounds[rank]
    k0, k1 = int(rp[lo]), int(rp[hi])
    lrp = (rp[lo:hi + 1] - k0).to(device.torch)
    ci = torch.as_tensor(np.asarray(col_idxs)[k0:k1]).to(device.torch)
    val = torch.as_tensor(np.asarray(values)[k0:k1]).to(device.torch)
    local, pat = localize(lrp, ci, lo, hi, bounds, rank)
    if exchange is not None:
        pat = exchange(pat)
    elif all_patterns is not None:
        pat.send = send_lists_from(all_patterns, rank, lo, hi, device.torch)
    return DistPartition(device, pat, lrp, local, val, global_cols=ci)


class NcclComm:
    """An NCCL communicator owned by libsparseb200, bootstrapped over torch.distributed."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist

        idbuf = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.call("sb_nccl_unique_id", idbuf)
        obj = [bytes(idbuf.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        idbuf = ctypes.create_string_buffer(obj[0], 128)
        handle = ctypes.c_void_p()
        _lib.call("sb_nccl_comm_init", world, idbuf, rank, ctypes.byref(handle))
        self.handle = handle
        self.rank, self.world = rank, world

    def close(self):
        if self.handle:
            _lib.call("sb_nccl_comm_destroy", self.handle)
            self.handle = ctypes.c_void_p()


class _DistSolver:
    """Row-partitioned Krylov solve.  ``parts``: this rank's DistPartition (with ``comm``)
    or every partition of the system on this GPU (loopback, comm=None).  Jacobi
    preconditioning from each partition's local inverse diagonal (``jacobi=False``: none)."""

    _kind = None
    _name = None

    def __init__(self, parts, criteria, comm: NcclComm | None = None, jacobi: bool = True):
        self.parts = list(parts) if isinstance(parts, (list, tuple)) else [parts]
        self.criteria = validate_criteria(criteria)
        self.comm = comm
        self.jacobi = jacobi
        if comm is not None and len(self.parts) != 1:
            raise E.InvalidArgumentError("NCCL mode takes exactly one partition per rank")

    def _extra(self):
        return ()

    def _dim(self):
        return 0

    def solve(self, bs, xs) -> ConvergenceLog:
        bs = bs if isinstance(bs, (list, tuple)) else [bs]
        xs = xs if isinstance(xs, (list, tuple)) else [xs]
        crit = _criteria_struct(self.criteria)
        cap = int(min(crit.max_iters, 1 << 22))
        hist = np.zeros(max(cap, 1), np.float64)
        log = _lib.SbLog(0, 0, 0, 0, hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap)
        n = len(self.parts)
        arr = (_lib.SbDistPart * n)()
        for k, (part, b, x) in enumerate(zip(self.parts, bs, xs)):
            arr[k] = part.struct(b, x, cap, self._kind, self._dim(), self.jacobi)
        m = self.parts[0].matrix
        comm = self.comm.handle if self.comm is not None else ctypes.c_void_p()
        _lib.call(f"sb_dist_{self._name}_solve_{m.precision.suffix}_{m.index_width.suffix}", arr, n, comm,
                  ctypes.byref(crit), *self._extra(), ctypes.byref(log), _stream(self.parts[0].device))
        hl = min(int(log.history_len), cap)
        return ConvergenceLog(int(log.iterations), hist[:hl].tolist(), bool(log.converged),
                              "residual" if log.stop_reason == 0 else "max_iters")


class DistCg(_DistSolver):
    """Row-partitioned (Jacobi-)CG: 2 allreduces per iteration (p.q; r.r + r.z)."""

    _kind = _lib.SOLVER_CG
    _name = "cg"


class DistBicgstab(_DistSolver):
    """Row-partitioned (Jacobi-)BiCGSTAB: 2 halos and 4 allreduces per iteration."""

    _kind = _lib.SOLVER_BICGSTAB
    _name = "bicgstab"


class DistGmres(_DistSolver):
    """Row-partitioned (Jacobi-)GMRES(krylov_dim): single-pass MGS with one allreduce per
    step (the reference's order, solvers.py:353-358)."""

    _kind = _lib.SOLVER_GMRES
    _name = "gmres"

    def __init__(self, parts, criteria, comm: NcclComm | None = None, krylov_dim: int = 30,
                 jacobi: bool = True):
        if krylov_dim < 1:
            raise E.InvalidArgumentError("krylov_dim must be positive")
        self.krylov_dim = int(krylov_dim)
        super().__init__(parts, criteria, comm, jacobi)

    def _dim(self):
        return self.krylov_dim

    def _extra(self):
        return (self.krylov_dim,)
