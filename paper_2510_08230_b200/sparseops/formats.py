"""Sparse storage on the device: CSR and COO (the reference's formats, formats.py:1-249)
plus ELL, SELL-P and Hybrid (absent from the reference; canonical
layouts pinned in SURVEY.md §8).

Every array is a torch CUDA tensor; construction and conversion run as kernels in
libsparseb200 (canonicalisation = stable radix sort + left-to-right duplicate sums,
bit-exact with coo_from_arrays).  Host inputs (NumPy, SciPy, Python lists, CPU
tensors) are copied to the device once; CUDA tensors are used in place.

SpMV dispatch: ``apply(b, x)`` calls ``sb_<fmt>_spmv_<value>_<index>``.  CSR carries
a plan built on first use from device row statistics: the TMA-staged ``stream``
kernel for regular short rows, ``vector`` (sub-warp per row) for long regular rows,
load-balanced ``merge`` path for irregular rows; ``kernel=`` forces one.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from .. import _lib
from .core import (DenseMatrix, Device, IndexWidth, Precision, _check_apply_shapes,
                   reduce_workspace)
from .errors import (DimensionMismatchError, IndexBoundsError, InvalidArgumentError,
                     PrecisionMismatchError, UnsupportedFeatureError)
from .linop import LinOp

__all__ = ["CooMatrix", "CsrMatrix", "EllMatrix", "SellpMatrix", "HybridMatrix",
           "coo_from_arrays", "coo_from_triplets", "csr_from_coo", "coo_from_csr",
           "csr_from_dense", "ell_from_csr", "sellp_from_csr", "hybrid_from_csr",
           "hybrid_ell_width", "from_scipy", "from_torch", "validate"]

_vp = ctypes.c_void_p


def _ptr(t: torch.Tensor | None):
    return _vp(t.data_ptr() if t is not None and t.numel() else 0)


def _on_device(device: Device, a, dtype: torch.dtype | None = None) -> torch.Tensor:
    """Device tensor view of ``a`` (no copy when it already is one of the right dtype)."""
    if isinstance(a, torch.Tensor):
        t = a
        if t.device.type != "cuda" or t.device.index != device.id:
            t = t.to(device.torch)
    else:
        arr = np.asarray(a)
        if arr.dtype == object:
            arr = arr.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device.torch)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous().reshape(-1)


def _stream(device: Device):
    return _vp(device.stream)


class _SparseBase(LinOp):
    _fmt = None

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    @property
    def device(self) -> Device:
        return self._device

    @property
    def precision(self) -> Precision:
        return Precision.from_dtype(self.values.dtype)

    @property
    def index_width(self) -> IndexWidth:
        return IndexWidth.from_dtype(self.col_idxs.dtype)

    @property
    def nnz(self) -> int:
        return int(self._nnz)

    def _suffix(self):
        return f"{self.precision.suffix}_{self.index_width.suffix}"

    def _check_spmv(self, b: DenseMatrix, x: DenseMatrix):
        _check_apply_shapes(self.shape, b, x)
        if self.values.dtype != b.values.dtype:
            raise PrecisionMismatchError(
                f"matrix/vector precision mismatch: {self.values.dtype} vs {b.values.dtype}")

    def apply(self, b: DenseMatrix, x: DenseMatrix) -> DenseMatrix:
        """x = A*b on the device (linop.spmv_csr / spmv_coo contract)."""
        self._check_spmv(b, x)
        bs, xs = b.struct(), x.struct()
        st = self.struct()
        _lib.call(f"sb_{self._fmt}_spmv_{self._suffix()}", ctypes.byref(st), ctypes.byref(bs),
                  ctypes.byref(xs), _stream(self.device))
        return x

    def _apply_advanced_device(self, alpha, b, beta, x):
        self._check_spmv(b, x)
        tmp = torch.empty(x.rows * x.cols, dtype=x.values.dtype, device=self.device.torch)
        m = self.matrix_struct()
        bs, xs = b.struct(), x.struct()
        _lib.call(f"sb_apply_advanced_{self._suffix()}", ctypes.byref(m), float(alpha),
                  ctypes.byref(bs), float(beta), ctypes.byref(xs), _ptr(tmp),
                  _stream(self.device))
        return x

    def matrix_struct(self) -> _lib.SbMatrix:
        st = self.struct()
        self._keep = st  # the SbMatrix holds a raw pointer to it
        return _lib.SbMatrix(self._fmt_id, 0, ctypes.cast(ctypes.pointer(st), _vp))

    def to_dense(self) -> np.ndarray:
        """Dense float64 host reconstruction (tests and small sizes)."""
        out = np.zeros((self.rows, self.cols))
        r, c, v = self._entries_host()
        np.add.at(out, (r, c), v.astype(np.float64))
        return out


# ------------------------------------------------------------------ COO
class CooMatrix(_SparseBase):
    """Coordinate storage: canonical (row-sorted, unique) parallel arrays."""

    _fmt, _fmt_id = "coo", _lib.FMT_COO

    def __init__(self, device: Device, rows, cols, row_idxs, col_idxs, values, kernel="auto"):
        self._device = device
        if kernel not in ("auto", "segmented"):
            raise InvalidArgumentError(f"unknown COO kernel {kernel!r}; expected 'auto' or 'segmented'")
        self.kernel_request = kernel
        self.rows, self.cols = int(rows), int(cols)
        self.col_idxs = _on_device(device, col_idxs)
        self.row_idxs = _on_device(device, row_idxs)
        self.values = _on_device(device, values)
        if not (self.row_idxs.numel() == self.col_idxs.numel() == self.values.numel()):
            raise InvalidArgumentError("row_idxs, col_idxs and values must have equal length")
        if self.row_idxs.dtype != self.col_idxs.dtype:
            raise InvalidArgumentError("index arrays must share one width")
        IndexWidth.from_dtype(self.col_idxs.dtype)
        Precision.from_dtype(self.values.dtype)
        self._nnz = self.values.numel()
        self._plan = None

    def plan(self) -> _lib.SbCooPlan:
        """Carry buffers of the segmented warp kernel and, for ``kernel="auto"``, a
        row-pointer index of the sorted rows with a CSR plan over it: the SpMV then runs
        the CSR kernels (stream / tile / ...) on (row_ptrs, col_idxs, values) -- the same
        per-row sums as spmv_coo (linop.py:137-159), without re-reading row_idxs."""
        if self._plan is None:
            tiles = -(-self._nnz // int(_lib.fn("sb_coo_tile_entries")()))
            self._carry_rows = torch.empty(max(tiles, 1), dtype=torch.int64, device=self.device.torch)
            self._carry_vals = torch.empty(max(tiles, 1), dtype=torch.float64, device=self.device.torch)
            rp_ptr, csr_plan = 0, None
            if self.kernel_request == "auto" and self.rows > 0 and self._nnz > 0:
                rp = torch.empty(self.rows + 1, dtype=self.col_idxs.dtype, device=self.device.torch)
                _lib.call(f"sb_csr_row_ptrs_from_coo_{self.index_width.suffix}", self.rows, self._nnz,
                          _ptr(self.row_idxs), _ptr(rp), _stream(self.device))
                self._csr_index = CsrMatrix(self.device, self.rows, self.cols, rp, self.col_idxs,
                                            self.values)
                self._csr_plan = self._csr_index.plan()
                rp_ptr, csr_plan = rp.data_ptr(), ctypes.addressof(self._csr_plan)
            self._plan = _lib.SbCooPlan(tiles, self._carry_rows.data_ptr(),
                                        self._carry_vals.data_ptr(), rp_ptr, csr_plan)
        return self._plan

    def with_kernel(self, kernel: str) -> "CooMatrix":
        """Same arrays (shared), "auto" (row-pointer index + CSR kernels) or "segmented"
        (the segmented-reduction warp kernel over the row array)."""
        return CooMatrix(self.device, self.rows, self.cols, self.row_idxs, self.col_idxs,
                         self.values, kernel=kernel)

    @property
    def kernel(self) -> str:
        p = self.plan()
        return "segmented" if not p.row_ptrs else "csr-" + self._csr_index.kernel

    def struct(self) -> _lib.SbCoo:
        return _lib.SbCoo(self.rows, self.cols, self._nnz, _ptr(self.row_idxs).value,
                          _ptr(self.col_idxs).value, _ptr(self.values).value,
                          ctypes.pointer(self.plan()))

    def _entries_host(self):
        return (self.row_idxs.cpu().numpy(), self.col_idxs.cpu().numpy(),
                self.values.cpu().numpy())

    def __repr__(self):
        return f"CooMatrix({self.rows}x{self.cols}, nnz={self.nnz}, {self.precision.value})"


# ------------------------------------------------------------------ CSR
class CsrMatrix(_SparseBase):
    """Compressed sparse row storage; ``row_ptrs`` has rows + 1 entries.

    ``kernel``: "auto" (row-statistics choice), "stream", "vector", "tile" (fixed-nnz
    tiles), "merge" or "strict" (thread-per-row device replica of the reference loop).
    """

    _fmt, _fmt_id = "csr", _lib.FMT_CSR

    def __init__(self, device: Device, rows, cols, row_ptrs, col_idxs, values, kernel="auto"):
        self._device = device
        self.rows, self.cols = int(rows), int(cols)
        self.row_ptrs = _on_device(device, row_ptrs)
        self.col_idxs = _on_device(device, col_idxs)
        self.values = _on_device(device, values)
        if self.row_ptrs.numel() != self.rows + 1:
            raise InvalidArgumentError(
                f"row_ptrs has length {self.row_ptrs.numel()}, expected rows+1 = {self.rows + 1}")
        if self.col_idxs.numel() != self.values.numel():
            raise InvalidArgumentError("col_idxs and values must have equal length")
        if self.row_ptrs.dtype != self.col_idxs.dtype:
            raise InvalidArgumentError("index arrays must share one width")
        IndexWidth.from_dtype(self.col_idxs.dtype)
        Precision.from_dtype(self.values.dtype)
        if kernel not in _lib.CSR_KERNELS:
            raise InvalidArgumentError(f"unknown CSR kernel {kernel!r}; "
                                       f"expected one of {sorted(_lib.CSR_KERNELS)}")
        self._nnz = self.values.numel()
        self.kernel_request = kernel
        self._plan = None
        self._stats = None

    # -- planning ---------------------------------------------------------------
    def row_stats(self) -> _lib.SbRowStats:
        if self._stats is None:
            st = _lib.SbRowStats()
            ws = reduce_workspace(self.device)
            _lib.call(f"sb_csr_row_stats_{self.index_width.suffix}", self.rows,
                      _ptr(self.row_ptrs), _ptr(ws), ctypes.byref(st), _stream(self.device))
            self._stats = st
        return self._stats

    def plan(self) -> _lib.SbCsrPlan:
        if self._plan is None:
            plan = _lib.SbCsrPlan()
            _lib.call("sb_csr_plan_select", ctypes.byref(self.row_stats()),
                      self.precision.itemsize, self.index_width.itemsize,
                      _lib.CSR_KERNELS[self.kernel_request], ctypes.byref(plan))
            if plan.num_tiles > 0:
                dev = self.device.torch
                n = int(plan.num_tiles)
                self._plan_bufs = (torch.empty(n + 1, dtype=torch.int64, device=dev),
                                   torch.empty(n + 1, dtype=torch.int64, device=dev),
                                   torch.empty(n, dtype=torch.int64, device=dev),
                                   torch.empty(n, dtype=torch.float64, device=dev))
                plan.tile_rows, plan.tile_nnz, plan.carry_rows, plan.carry_vals = (
                    t.data_ptr() for t in self._plan_bufs)
                _lib.call(f"sb_csr_plan_build_{self.index_width.suffix}", self.rows, self._nnz,
                          _ptr(self.row_ptrs), ctypes.byref(plan), _stream(self.device))
            self._plan = plan
        return self._plan

    @property
    def kernel(self) -> str:
        """The SpMV kernel the plan selected."""
        k = self.plan().kernel
        return {v: n for n, v in _lib.CSR_KERNELS.items()}[k]

    def with_kernel(self, kernel: str) -> "CsrMatrix":
        """Same arrays (shared, no copy), different forced SpMV kernel."""
        return CsrMatrix(self.device, self.rows, self.cols, self.row_ptrs, self.col_idxs,
                         self.values, kernel=kernel)

    def struct(self) -> _lib.SbCsr:
        return _lib.SbCsr(self.rows, self.cols, self._nnz, _ptr(self.row_ptrs).value,
                          _ptr(self.col_idxs).value, _ptr(self.values).value,
                          ctypes.pointer(self.plan()))

    # -- reference API ------------------------------------------------------------
    def row_slice(self, i: int) -> slice:
        rp = self.row_ptrs[i:i + 2].cpu()
        return slice(int(rp[0]), int(rp[1]))

    def diagonal(self) -> np.ndarray:
        """Stored main-diagonal values (0 where structurally absent), as a host array
        (formats.py:113-122)."""
        n = min(self.rows, self.cols)
        rows = self._row_of_entry()
        mask = (self.col_idxs.long() == rows) & (rows < n)
        diag = torch.zeros(n, dtype=self.values.dtype, device=self.device.torch)
        diag[rows[mask]] = self.values[mask]
        return diag.cpu().numpy()

    def _row_of_entry(self) -> torch.Tensor:
        counts = (self.row_ptrs[1:] - self.row_ptrs[:-1]).long()
        return torch.repeat_interleave(torch.arange(self.rows, device=self.device.torch), counts)

    def _entries_host(self):
        return (self._row_of_entry().cpu().numpy(), self.col_idxs.cpu().numpy(),
                self.values.cpu().numpy())

    def __repr__(self):
        return f"CsrMatrix({self.rows}x{self.cols}, nnz={self.nnz}, {self.precision.value})"


# ------------------------------------------------------------------ ELL / SELL-P / Hybrid
class EllMatrix(_SparseBase):
    """ELL(width, stride): entry k of row i at k*stride + i (column-major); padding has
    col = -1 and val = 0 and is skipped, so results equal CSR's bit for bit."""

    _fmt, _fmt_id = "ell", _lib.FMT_ELL

    def __init__(self, device, rows, cols, width, stride, col_idxs, values, nnz=None):
        self._device = device
        self.rows, self.cols = int(rows), int(cols)
        self.width, self.stride = int(width), int(stride)
        self.col_idxs = _on_device(device, col_idxs)
        self.values = _on_device(device, values)
        if self.col_idxs.numel() != self.width * self.stride or \
                self.values.numel() != self.width * self.stride:
            raise InvalidArgumentError("ELL arrays must hold width*stride entries")
        if self.stride < self.rows:
            raise InvalidArgumentError("ELL stride must be >= rows")
        self._nnz = int((self.col_idxs >= 0).sum()) if nnz is None else int(nnz)

    def struct(self) -> _lib.SbEll:
        return _lib.SbEll(self.rows, self.cols, self.width, self.stride, _ptr(self.col_idxs).value,
                          _ptr(self.values).value)

    @property
    def stored(self) -> int:
        return self.width * self.stride

    def _entries_host(self):
        c = self.col_idxs.view(self.width, self.stride).cpu().numpy()
        v = self.values.view(self.width, self.stride).cpu().numpy()
        k, i = np.nonzero(c >= 0)
        return i, c[k, i], v[k, i]

    def __repr__(self):
        return f"EllMatrix({self.rows}x{self.cols}, width={self.width}, {self.precision.value})"


class SellpMatrix(_SparseBase):
    """SELL-P(slice_size): per-slice ELL; entry k of row i (slice s = i // S) at
    (slice_sets[s] + k)*S + i % S; slice_sets is the exclusive scan of slice_lengths."""

    _fmt, _fmt_id = "sellp", _lib.FMT_SELLP

    def __init__(self, device, rows, cols, slice_size, slice_lengths, slice_sets, col_idxs,
                 values, nnz=None, row_perm=None):
        self._device = device
        # SELL-C-sigma: stored row i holds matrix row row_perm[i] (None: identity)
        self.row_perm = None if row_perm is None else _on_device(device, row_perm)
        self.rows, self.cols = int(rows), int(cols)
        self.slice_size = int(slice_size)
        self.slice_lengths = _on_device(device, slice_lengths)
        self.slice_sets = _on_device(device, slice_sets)
        self.col_idxs = _on_device(device, col_idxs)
        self.values = _on_device(device, values)
        self.num_slices = -(-self.rows // self.slice_size) if self.slice_size else 0
        if self.slice_lengths.numel() != self.num_slices or \
                self.slice_sets.numel() != self.num_slices + 1:
            raise InvalidArgumentError("slice arrays do not match rows / slice_size")
        self._nnz = int((self.col_idxs >= 0).sum()) if nnz is None else int(nnz)
        self.max_block_entries = self._block_entries()
        self.staged = True  # TMA-staged slice kernel when the block fits shared memory
        self._pieces = self._piece_plan()

    def with_staging(self, staged: bool) -> "SellpMatrix":
        """Same arrays (shared), staged (TMA) or direct SpMV kernel."""
        m = SellpMatrix(self.device, self.rows, self.cols, self.slice_size, self.slice_lengths,
                        self.slice_sets, self.col_idxs, self.values, nnz=self._nnz,
                        row_perm=self.row_perm)
        m.staged = staged
        m._pieces = self._pieces
        return m

    def _block_entries(self) -> int:
        """Max stored entries of any aligned group of 128 / S slices (one TMA-staged block
        of the sellp_stream kernel); 0 when the slice size has no staged kernel."""
        S = self.slice_size
        if S not in (32, 64, 128) or self.num_slices == 0:
            return 0
        spb = 128 // S
        ss = self.slice_sets.long()
        idx = torch.arange(0, self.num_slices, spb, device=ss.device)
        hi = torch.clamp(idx + spb, max=self.num_slices)
        return int(((ss[hi] - ss[idx]) * S).max())

    def _piece_plan(self):
        """Split plan of the staged kernel (csrc/spmv.cuh sellp_piece_kernel): blocks of
        128 / S slices larger than one piece (a balanced share of all stored entries, at
        least 8 TMA chunks) are cut into pieces whose partial row sums are added in piece
        order.  None when no block exceeds one piece (the whole-block kernels run)."""
        S = self.slice_size
        if S not in (32, 64, 128) or self.num_slices == 0 or self.max_block_entries == 0:
            return None
        spb = 128 // S
        chunk = min(self.max_block_entries, max(2048 // S * S, S)) // S * S
        ss = self.slice_sets.long()
        idx = torch.arange(0, self.num_slices, spb, device=ss.device)
        ent = (ss[torch.clamp(idx + spb, max=self.num_slices)] - ss[idx]) * S
        sms = torch.cuda.get_device_properties(ss.device).multi_processor_count
        pe = max(8 * chunk, -(-int(ent.sum()) // (sms * 32)))
        pe = -(-pe // chunk) * chunk
        npb = torch.clamp((ent + pe - 1) // pe, min=1)
        if int(npb.max()) <= 1:
            return None
        pstart = torch.zeros(idx.numel() + 1, dtype=torch.int64, device=ss.device)
        pstart[1:] = torch.cumsum(npb, 0)
        pblock = torch.repeat_interleave(torch.arange(idx.numel(), device=ss.device), npb)
        split = torch.nonzero(npb > 1).flatten()
        plan = torch.cat([pstart, pblock, split]).to(torch.int64).contiguous()
        npieces = int(pstart[-1])
        carry = torch.empty(npieces * 128, dtype=torch.float64, device=ss.device)
        return plan, npieces, int(split.numel()), pe, carry

    def struct(self) -> _lib.SbSellp:
        pc = self._pieces if self.staged else None
        return _lib.SbSellp(self.rows, self.cols, self.slice_size, self.num_slices,
                            _ptr(self.slice_lengths).value, _ptr(self.slice_sets).value,
                            _ptr(self.col_idxs).value, _ptr(self.values).value,
                            self.max_block_entries if self.staged else 0,
                            _ptr(self.row_perm).value if self.row_perm is not None else None,
                            _ptr(pc[0]).value if pc else None, pc[1] if pc else 0, pc[2] if pc else 0,
                            pc[3] if pc else 0, _ptr(pc[4]).value if pc else None)

    @property
    def stored(self) -> int:
        return self.values.numel()

    def _entries_host(self):
        S = self.slice_size
        sl = self.slice_lengths.cpu().numpy().astype(np.int64)
        ss = self.slice_sets.cpu().numpy().astype(np.int64)
        c = self.col_idxs.cpu().numpy()
        v = self.values.cpu().numpy()
        rows, cols, vals = [], [], []
        for s in range(self.num_slices):
            blk_c = c[ss[s] * S:(ss[s] + sl[s]) * S].reshape(sl[s], S)
            blk_v = v[ss[s] * S:(ss[s] + sl[s]) * S].reshape(sl[s], S)
            k, l = np.nonzero(blk_c >= 0)
            rows.append(s * S + l)
            cols.append(blk_c[k, l])
            vals.append(blk_v[k, l])
        if not rows:
            return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)
        r = np.concatenate(rows)
        if self.row_perm is not None:
            r = self.row_perm.cpu().numpy().astype(np.int64)[r]
        return r, np.concatenate(cols), np.concatenate(vals)

    def __repr__(self):
        return (f"SellpMatrix({self.rows}x{self.cols}, S={self.slice_size}, "
                f"{self.precision.value})")


class HybridMatrix(_SparseBase):
    """Hybrid(w): the first min(len_i, w) entries of each row in ELL(w), the remainder in a
    canonical COO tail.  SpMV = ELL pass, then the COO tail accumulated into x."""

    _fmt, _fmt_id = "hybrid", _lib.FMT_HYBRID

    def __init__(self, device, ell: EllMatrix, coo: CooMatrix):
        if ell.shape != coo.shape:
            raise DimensionMismatchError("ELL and COO parts must share a shape")
        self._device = device
        self.ell, self.coo = ell, coo
        self.rows, self.cols = ell.rows, ell.cols
        self.col_idxs, self.values = ell.col_idxs, ell.values
        self._nnz = ell.nnz + coo.nnz

    def struct(self) -> _lib.SbHybrid:
        return _lib.SbHybrid(self.ell.struct(), self.coo.struct())

    def _entries_host(self):
        a = self.ell._entries_host()
        b = self.coo._entries_host()
        return tuple(np.concatenate([x, y]) for x, y in zip(a, b))

    def __repr__(self):
        return (f"HybridMatrix({self.rows}x{self.cols}, ell_width={self.ell.width}, "
                f"coo_nnz={self.coo.nnz}, {self.precision.value})")


# ------------------------------------------------------------------ construction
def coo_from_arrays(device, rows, cols, row_idxs, col_idxs, values,
                    precision: Precision = Precision.double,
                    index_width: IndexWidth = IndexWidth.i32) -> CooMatrix:
    """Canonicalise raw triplets on the device (formats.py:131-166): bounds check,
    stable sort by (row, col), duplicates summed left to right in the value dtype,
    explicit zeros kept."""
    rows, cols = int(rows), int(cols)
    if rows < 0 or cols < 0:
        raise InvalidArgumentError("rows and cols must be non-negative")
    vt, it = precision.torch_dtype, index_width.torch_dtype
    ri = _on_device(device, row_idxs, torch.int64)
    ci = _on_device(device, col_idxs, torch.int64)
    if isinstance(values, torch.Tensor):
        vals = _on_device(device, values, vt)
    else:  # np.asarray(values, dtype=vdt) semantics: cast on the host, then copy
        vals = _on_device(device, np.asarray(values, dtype=precision.dtype))
    m = ri.numel()
    if not (ci.numel() == m == vals.numel()):
        raise InvalidArgumentError("row_idxs, col_idxs and values must have equal length")
    dev = device.torch
    if m == 0:
        z = torch.empty(0, dtype=it, device=dev)
        return CooMatrix(device, rows, cols, z, z.clone(), torch.empty(0, dtype=vt, device=dev))
    ws_bytes = int(_lib.fn("sb_coo_from_arrays_workspace_bytes")(m))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    orow = torch.empty(m, dtype=it, device=dev)
    ocol = torch.empty(m, dtype=it, device=dev)
    oval = torch.empty(m, dtype=vt, device=dev)
    nnz = ctypes.c_int64(0)
    err = _lib.SbError()
    status = _lib.fn(f"sb_coo_from_arrays_{precision.suffix}_{index_width.suffix}")(
        rows, cols, m, _ptr(ri), _ptr(ci), _ptr(vals), _ptr(orow), _ptr(ocol), _ptr(oval),
        _ptr(ws), ws_bytes, ctypes.byref(nnz), _stream(device), ctypes.byref(err))
    if status == 5:
        k = int(err.row)
        raise IndexBoundsError(
            f"triplet {k} at ({int(ri[k])}, {int(ci[k])}) outside {rows}x{cols}")
    _lib.raise_for(status, err)
    n = int(nnz.value)
    return CooMatrix(device, rows, cols, orow[:n].clone(), ocol[:n].clone(), oval[:n].clone())


def coo_from_triplets(device, rows, cols, triplets, precision: Precision = Precision.double,
                      index_width: IndexWidth = IndexWidth.i32) -> CooMatrix:
    """Canonical COO from (row, col, value) triplets; duplicates are summed."""
    if len(triplets) == 0:
        return coo_from_arrays(device, rows, cols, [], [], [], precision, index_width)
    ri = [t[0] for t in triplets]
    ci = [t[1] for t in triplets]
    vals = [t[2] for t in triplets]
    return coo_from_arrays(device, rows, cols, ri, ci, vals, precision, index_width)


def csr_from_coo(m: CooMatrix, kernel="auto") -> CsrMatrix:
    """Canonical COO -> CSR (formats.py:184-191): row_ptrs by per-row lower bounds."""
    it = m.col_idxs.dtype
    rp = torch.empty(m.rows + 1, dtype=it, device=m.device.torch)
    _lib.call(f"sb_csr_row_ptrs_from_coo_{m.index_width.suffix}", m.rows, m.nnz,
              _ptr(m.row_idxs), _ptr(rp), _stream(m.device))
    return CsrMatrix(m.device, m.rows, m.cols, rp, m.col_idxs.clone(), m.values.clone(),
                     kernel=kernel)


def coo_from_csr(m: CsrMatrix) -> CooMatrix:
    """CSR -> canonical COO (formats.py:194-199)."""
    ri = torch.empty(m.nnz, dtype=m.col_idxs.dtype, device=m.device.torch)
    _lib.call(f"sb_coo_row_idxs_from_csr_{m.index_width.suffix}", m.rows, m.nnz,
              _ptr(m.row_ptrs), _ptr(ri), _stream(m.device))
    return CooMatrix(m.device, m.rows, m.cols, ri, m.col_idxs.clone(), m.values.clone())


def csr_from_dense(device, array, precision: Precision = Precision.double,
                   index_width: IndexWidth = IndexWidth.i32, keep_zeros: bool = False) -> CsrMatrix:
    """CSR from a dense 2-D array (test / setup helper, formats.py:202-211)."""
    a = np.asarray(array.cpu() if isinstance(array, torch.Tensor) else array, dtype=np.float64)
    if a.ndim != 2:
        raise InvalidArgumentError("expected a 2-D array")
    rows, cols = a.shape
    if keep_zeros:
        r, c = np.divmod(np.arange(rows * cols, dtype=np.int64), cols)
    else:
        r, c = np.nonzero(a != 0.0)
    return csr_from_coo(coo_from_arrays(device, rows, cols, r, c, a[r, c], precision,
                                        index_width))


def from_scipy(device, mat, precision: Precision | None = None,
               index_width: IndexWidth = IndexWidth.i32, format="Csr"):
    """Any scipy.sparse matrix -> canonical CSR / COO on the device (duplicates summed)."""
    coo = mat.tocoo()
    prec = precision or Precision.from_dtype(coo.data.dtype if coo.data.dtype in
                                             (np.float32, np.float64) else np.float64)
    m = coo_from_arrays(device, coo.shape[0], coo.shape[1], coo.row.astype(np.int64),
                        coo.col.astype(np.int64), coo.data, prec, index_width)
    return m if str(format).lower() == "coo" else csr_from_coo(m)


def from_torch(device, t: torch.Tensor, index_width: IndexWidth | None = None, format="Csr"):
    """torch sparse (COO / CSR) or dense tensor -> canonical CSR / COO on the device."""
    if t.layout == torch.sparse_csr:
        t = t.to_sparse_coo()
    if t.layout == torch.sparse_coo:
        t = t.coalesce()
        idx = t.indices()
        ri, ci, vals = idx[0], idx[1], t.values()
    elif t.layout == torch.strided:
        if t.dim() != 2:
            raise InvalidArgumentError("expected a 2-D tensor")
        nz = t.nonzero(as_tuple=True)
        ri, ci, vals = nz[0], nz[1], t[nz]
    else:
        raise UnsupportedFeatureError(f"unsupported torch layout {t.layout}")
    prec = Precision.from_dtype(vals.dtype)
    iw = index_width or IndexWidth.i32
    m = coo_from_arrays(device, t.shape[0], t.shape[1], ri, ci, vals, prec, iw)
    return m if str(format).lower() == "coo" else csr_from_coo(m)


def _row_lengths(m: CsrMatrix) -> torch.Tensor:
    return (m.row_ptrs[1:] - m.row_ptrs[:-1]).long()


def ell_from_csr(m: CsrMatrix, stride_align: int = 32, width: int | None = None) -> EllMatrix:
    """CSR -> ELL(width = max row length, stride = round_up(rows, stride_align))."""
    lens = _row_lengths(m)
    w = int(lens.max()) if m.rows and width is None else int(width or 0)
    if m.rows and w < int(lens.max()):
        raise InvalidArgumentError(f"ELL width {w} < max row length {int(lens.max())}")
    stride = -(-m.rows // stride_align) * stride_align
    dev = m.device.torch
    ec = torch.empty(w * stride, dtype=m.col_idxs.dtype, device=dev)
    ev = torch.empty(w * stride, dtype=m.values.dtype, device=dev)
    out = EllMatrix(m.device, m.rows, m.cols, w, stride, ec, ev, nnz=m.nnz)
    st = out.struct()
    src = m.struct()
    _lib.call(f"sb_ell_from_csr_{m._suffix()}", ctypes.byref(src), ctypes.byref(st),
              _stream(m.device))
    return out


def sellp_from_csr(m: CsrMatrix, slice_size: int = 64, sigma: int = 1) -> SellpMatrix:
    """CSR -> SELL-P(slice_size) with stride factor 1.  ``sigma`` > 1 gives SELL-C-sigma:
    rows sorted by decreasing length (stably) inside windows of ``sigma`` rows (a multiple
    of slice_size) so each slice pads to similar lengths; the kernels write row results
    through the permutation, and every row keeps its stored entry order (results equal
    plain SELL-P / CSR bit for bit)."""
    if slice_size < 1:
        raise InvalidArgumentError("slice_size must be positive")
    if sigma > 1:
        if sigma % slice_size:
            raise InvalidArgumentError("sigma must be a multiple of slice_size")
        perm = _sigma_permutation(m, sigma)
        out = sellp_from_csr(_permute_rows(m, perm), slice_size)
        out.row_perm = perm.to(m.col_idxs.dtype)
        return out
    dev = m.device.torch
    ns = -(-m.rows // slice_size)
    it = m.col_idxs.dtype
    sl = torch.empty(max(ns, 1), dtype=it, device=dev)[:ns]
    ss = torch.empty(ns + 1, dtype=it, device=dev)
    total = ctypes.c_int64(0)
    _lib.call(f"sb_sellp_slices_{m.index_width.suffix}", m.rows, _ptr(m.row_ptrs), slice_size,
              _ptr(sl), _ptr(ss), ctypes.byref(total), _stream(m.device))
    n = int(total.value) * slice_size
    sc = torch.empty(n, dtype=it, device=dev)
    sv = torch.empty(n, dtype=m.values.dtype, device=dev)
    out = SellpMatrix(m.device, m.rows, m.cols, slice_size, sl, ss, sc, sv, nnz=m.nnz)
    st = out.struct()
    src = m.struct()
    _lib.call(f"sb_sellp_from_csr_{m._suffix()}", ctypes.byref(src), ctypes.byref(st),
              _stream(m.device))
    return out


def _sigma_permutation(m: CsrMatrix, sigma: int) -> torch.Tensor:
    """Rows sorted by decreasing length inside consecutive windows of sigma rows (stable)."""
    lens = (m.row_ptrs[1:] - m.row_ptrs[:-1]).long()
    n = m.rows
    window = torch.arange(n, device=lens.device) // sigma
    key = window * (int(lens.max()) + 1 if n else 1) + (lens.max() - lens if n else lens)
    return torch.sort(key, stable=True).indices


def _permute_rows(m: CsrMatrix, perm: torch.Tensor) -> CsrMatrix:
    """Row-permuted copy of m (row p of the result = row perm[p] of m), entries in order."""
    rp = m.row_ptrs.long()
    lens = (rp[1:] - rp[:-1])[perm]
    new_rp = torch.zeros(m.rows + 1, dtype=torch.int64, device=rp.device)
    torch.cumsum(lens, 0, out=new_rp[1:])
    start = torch.repeat_interleave(rp[:-1][perm], lens)
    offs = torch.arange(int(new_rp[-1]), device=rp.device) - torch.repeat_interleave(new_rp[:-1], lens)
    src = start + offs
    it = m.col_idxs.dtype
    return CsrMatrix(m.device, m.rows, m.cols, new_rp.to(it), m.col_idxs[src], m.values[src])


def hybrid_ell_width(row_lengths, quantile: float = 0.8) -> int:
    """Hybrid ELL-width rule: the row length at sorted position floor(q*(rows-1))."""
    lens = row_lengths if isinstance(row_lengths, torch.Tensor) else torch.as_tensor(row_lengths)
    if lens.numel() == 0:
        return 0
    srt = torch.sort(lens.long()).values
    return int(srt[int(math.floor(quantile * (lens.numel() - 1)))])


def hybrid_from_csr(m: CsrMatrix, ell_width: int | None = None,
                    stride_align: int = 32) -> HybridMatrix:
    """CSR -> Hybrid(w): ELL(w) holds each row's first min(len, w) entries, the rest go
    to a canonical COO tail (default w: 80th-percentile row length)."""
    lens = _row_lengths(m)
    w = hybrid_ell_width(lens) if ell_width is None else int(ell_width)
    dev = m.device.torch
    it = m.col_idxs.dtype
    stride = -(-m.rows // stride_align) * stride_align
    tail_ptrs = torch.empty(m.rows + 1, dtype=it, device=dev)
    tail_nnz = ctypes.c_int64(0)
    _lib.call(f"sb_hybrid_tail_ptrs_{m.index_width.suffix}", m.rows, _ptr(m.row_ptrs), w,
              _ptr(tail_ptrs), ctypes.byref(tail_nnz), _stream(m.device))
    t = int(tail_nnz.value)
    ell = EllMatrix(m.device, m.rows, m.cols, w, stride,
                    torch.empty(w * stride, dtype=it, device=dev),
                    torch.empty(w * stride, dtype=m.values.dtype, device=dev), nnz=m.nnz - t)
    coo = CooMatrix(m.device, m.rows, m.cols, torch.empty(t, dtype=it, device=dev),
                    torch.empty(t, dtype=it, device=dev),
                    torch.empty(t, dtype=m.values.dtype, device=dev),
                    kernel="segmented")  # the tail accumulates into x: warp kernel
    out = HybridMatrix(m.device, ell, coo)
    st = out.struct()
    src = m.struct()
    _lib.call(f"sb_hybrid_from_csr_{m._suffix()}", ctypes.byref(src), _ptr(tail_ptrs),
              ctypes.byref(st), _stream(m.device))
    return out


def validate(m) -> list[str]:
    """Check every CSR / COO format invariant on a host copy; returns all violations
    (formats.py:214-249 semantics)."""
    out = []
    if isinstance(m, CsrMatrix):
        rp = m.row_ptrs.cpu().numpy().astype(np.int64)
        ci = m.col_idxs.cpu().numpy().astype(np.int64)
        nnz = m.nnz
        if len(rp) and rp[0] != 0:
            out.append(f"row_ptrs[0] = {rp[0]}, expected 0")
        for i in np.flatnonzero(rp[1:] < rp[:-1]) + 1:
            out.append(f"non-decreasing row_ptrs at {i}")
        if len(rp) and rp[-1] != nnz:
            out.append(f"row_ptrs[rows] = {rp[-1]}, expected nnz = {nnz}")
        for i in range(m.rows):
            lo, hi = int(rp[i]), int(rp[i + 1])
            if lo < 0 or hi > nnz or hi < lo:
                continue
            seg = ci[lo:hi]
            for k in np.flatnonzero((seg < 0) | (seg >= m.cols)):
                out.append(f"column index {seg[k]} out of bounds at entry {lo + k}")
            for k in np.flatnonzero(seg[1:] <= seg[:-1]) + 1:
                out.append(f"columns not strictly increasing in row {i} at entry {lo + k}")
    elif isinstance(m, CooMatrix):
        r = m.row_idxs.cpu().numpy().astype(np.int64)
        c = m.col_idxs.cpu().numpy().astype(np.int64)
        for k in range(m.nnz):
            if r[k] < 0 or r[k] >= m.rows:
                out.append(f"row index {r[k]} out of bounds at entry {k}")
            if c[k] < 0 or c[k] >= m.cols:
                out.append(f"column index {c[k]} out of bounds at entry {k}")
            if k > 0 and (r[k], c[k]) <= (r[k - 1], c[k - 1]):
                out.append(f"entries not sorted/unique at entry {k}")
    else:
        raise InvalidArgumentError(f"expected CsrMatrix or CooMatrix, got {type(m).__name__}")
    return out
