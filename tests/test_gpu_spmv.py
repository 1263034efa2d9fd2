"""GPU parity: SpMV of every format and kernel against the reference's own outputs.

Golden vectors were produced by the reference (tests/golden/make_golden.py).  Kernels
that keep the reference's per-row sequential order (strict, stream, ELL, SELL-P) must
match BIT FOR BIT; row-splitting kernels (vector, merge, COO, Hybrid) must be within
the reference's scale tolerance (test_acceptance.py:80-87): 1e-12 (fp64) / 1e-5 (fp32)
x max_i sum_j |a_ij| x max|b|.
"""

import numpy as np
import pytest

from oracle import fixtures, sbref
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
from tests import golden_io
from tests.gpu_util import assert_close, csr, host, out, vec

pytestmark = pytest.mark.gpu

TYPES = [("float64", "int32"), ("float64", "int64"), ("float32", "int32"), ("float32", "int64")]
EXACT_KERNELS = ["strict", "stream"]
TOL_KERNELS = ["vector", "merge", "tile", "auto"]


@pytest.mark.parametrize("vdt,idt", TYPES)
def test_csr_kernels_on_golden_suite(dev, vdt, idt):
    for m in golden_io.spmv_suite(vdt, idt):
        rows, cols = (int(t) for t in m["shape"])
        b = vec(dev, m["b"])
        for kernel in EXACT_KERNELS + TOL_KERNELS:
            a = csr(dev, m["row_ptrs"], m["col_idxs"], m["values"], cols, kernel=kernel)
            x = out(dev, rows, m["values"].dtype)
            try:
                a.apply(b, x)
            except sp.errors.UnsupportedFeatureError:
                assert kernel == "stream"
                continue
            got = host(x)
            if kernel in EXACT_KERNELS:
                np.testing.assert_array_equal(got, m["x"], err_msg=f"{kernel} {rows}x{cols}")
            else:
                assert_close(got, m["x"], m["row_ptrs"], m["values"], m["b"])


@pytest.mark.parametrize("vdt,idt", TYPES)
def test_coo_ell_sellp_hybrid_on_golden_suite(dev, vdt, idt):
    for m in golden_io.spmv_suite(vdt, idt):
        rows, cols = (int(t) for t in m["shape"])
        a = csr(dev, m["row_ptrs"], m["col_idxs"], m["values"], cols)
        b = vec(dev, m["b"])
        for fmt in ("coo", "coo_seg", "ell", "sellp", "sellp32", "sellp_direct", "sellp_sigma",
                    "sellp_sigma_direct", "hybrid", "hybrid2"):
            if fmt == "coo":
                mat = sp.coo_from_csr(a)
            elif fmt == "coo_seg":
                mat = sp.coo_from_csr(a).with_kernel("segmented")
            elif fmt == "ell":
                mat = sp.ell_from_csr(a)
            elif fmt == "sellp":
                mat = sp.sellp_from_csr(a, 64)
            elif fmt == "sellp32":
                mat = sp.sellp_from_csr(a, 32)
            elif fmt == "sellp_direct":
                mat = sp.sellp_from_csr(a, 64).with_staging(False)
            elif fmt == "sellp_sigma":
                mat = sp.sellp_from_csr(a, 32, sigma=128)
            elif fmt == "sellp_sigma_direct":
                mat = sp.sellp_from_csr(a, 32, sigma=64).with_staging(False)
            elif fmt == "hybrid":
                mat = sp.hybrid_from_csr(a)
            else:
                mat = sp.hybrid_from_csr(a, ell_width=2)
            x = out(dev, rows, m["values"].dtype)
            mat.apply(b, x)
            got = host(x)
            if fmt in ("ell", "sellp", "sellp32", "sellp_direct", "sellp_sigma", "sellp_sigma_direct"):
                np.testing.assert_array_equal(got, m["x"], err_msg=f"{fmt} {rows}x{cols}")
            elif fmt == "coo" and mat.kernel in ("csr-stream", "csr-strict"):
                # row-pointer-indexed COO on a sequential-order CSR kernel: bit-exact
                np.testing.assert_array_equal(got, m["x"], err_msg=f"{fmt} {rows}x{cols}")
            else:
                assert_close(got, m["x"], m["row_ptrs"], m["values"], m["b"])


def test_known_answers(dev):
    """test_linop.py:29-55 known answers."""
    a = sp.csr_from_dense(dev, np.eye(3))
    x = out(dev, 3, np.float64)
    a.apply(vec(dev, [1.0, 2.0, 3.0]), x)
    np.testing.assert_array_equal(host(x), [1.0, 2.0, 3.0])
    a = sp.csr_from_dense(dev, np.array([[1.0, 2.0], [0.0, 3.0]]))
    x = out(dev, 2, np.float64)
    a.apply(vec(dev, [1.0, 1.0]), x)
    np.testing.assert_array_equal(host(x), [3.0, 3.0])
    # empty row writes 0 over a NaN pre-fill, for every kernel and format
    dense = np.array([[1.0, 0.0], [0.0, 0.0], [0.0, 2.0]])
    base = sp.csr_from_dense(dev, dense)
    for kernel in ("strict", "stream", "vector", "merge", "tile"):
        x = out(dev, 3, np.float64)
        base.with_kernel(kernel).apply(vec(dev, [1.0, 1.0]), x)
        np.testing.assert_array_equal(host(x), [1.0, 0.0, 2.0], err_msg=kernel)
    for conv in (sp.coo_from_csr, sp.ell_from_csr, sp.sellp_from_csr, sp.hybrid_from_csr):
        x = out(dev, 3, np.float64)
        conv(base).apply(vec(dev, [1.0, 1.0]), x)
        np.testing.assert_array_equal(host(x), [1.0, 0.0, 2.0], err_msg=conv.__name__)
    # COO with nnz = 0 writes zeros; 1x1
    z = sp.coo_from_arrays(dev, 3, 3, [], [], [])
    x = out(dev, 3, np.float64)
    z.apply(vec(dev, [1.0, 1.0, 1.0]), x)
    np.testing.assert_array_equal(host(x), [0.0, 0.0, 0.0])
    one = sp.csr_from_dense(dev, [[2.0]])
    x = out(dev, 1, np.float64)
    one.apply(vec(dev, [3.0]), x)
    assert host(x)[0] == 6.0


def test_multi_rhs_and_strided(dev):
    """Multi-RHS apply loops the columns like linop.py:115 (test_linop.py:136-141)."""
    rng = np.random.default_rng(3)
    trip = fixtures.random_sparse_triplets(rng, 40, 30, 0.2)
    rp, ci, v = fixtures.canonical_csr(40, *trip)
    a = csr(dev, rp, ci, v, 30)
    bm = rng.standard_normal((30, 3))
    b = sp.dense_from_array(dev, bm.copy())
    x = out(dev, 40, np.float64, cols=3)
    a.apply(b, x)
    got = host(x)
    for j in range(3):
        np.testing.assert_array_equal(got[:, j], sbref.csr_spmv(rp, ci, v, bm[:, j]))


def test_apply_advanced(dev):
    """linop.apply_advanced rounding, beta = 0 overwrites NaN/Inf (test_linop.py:153-180)."""
    rng = np.random.default_rng(4)
    rp, ci, v = fixtures.canonical_csr(50, *fixtures.random_sparse_triplets(rng, 50, 50, 0.1))
    a = csr(dev, rp, ci, v, 50)
    bv = rng.standard_normal(50)
    t = sbref.csr_spmv(rp, ci, v, bv)
    x0 = rng.standard_normal(50)
    x = vec(dev, x0)
    a.apply_advanced(2.5, vec(dev, bv), -0.5, x)
    np.testing.assert_array_equal(host(x), sbref.axpy(2.5, t, sbref.scal(-0.5, x0)))
    x = out(dev, 50, np.float64, fill=np.inf)
    a.apply_advanced(2.5, vec(dev, bv), 0.0, x)
    np.testing.assert_array_equal(host(x), sbref.scal(2.5, t))


def test_linearity_and_determinism(dev):
    rp, ci, v = fixtures.stencil_csr(20, dim=3)
    rng = np.random.default_rng(9)
    b1, b2 = rng.standard_normal(rp.size - 1), rng.standard_normal(rp.size - 1)
    for kernel in ("stream", "vector", "merge", "tile"):
        a = csr(dev, rp, ci, v, kernel=kernel)
        runs = []
        for _ in range(3):
            x = out(dev, a.rows, np.float64)
            a.apply(vec(dev, b1 + b2), x)
            runs.append(host(x))
        np.testing.assert_array_equal(runs[0], runs[1])
        np.testing.assert_array_equal(runs[0], runs[2])
        x1, x2 = out(dev, a.rows, np.float64), out(dev, a.rows, np.float64)
        a.apply(vec(dev, b1), x1)
        a.apply(vec(dev, b2), x2)
        assert_close(runs[0], host(x1) + host(x2), rp, v, np.abs(b1) + np.abs(b2))


def test_heavy_rows_merge_and_coo(dev):
    """Rows far longer than a tile (nnz-tile and merge-path carries across many tiles; COO
    runs across tiles) -- the test_linop.py:108-122 heavy-row case at device scale."""
    rng = np.random.default_rng(12)
    n = 3000
    lens = np.ones(n, np.int64)
    lens[[0, 7, 1500, n - 1]] = [20000, 5000, 12345, 8000]
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size)
    rp, ci, v = fixtures.canonical_csr(n, rows, cols, vals)
    bv = rng.standard_normal(n)
    ref = sbref.csr_spmv(rp, ci, v, bv)
    a = csr(dev, rp, ci, v)
    assert a.kernel == "tile"
    for mat in (a, a.with_kernel("merge"), a.with_kernel("vector"), sp.coo_from_csr(a),
                sp.coo_from_csr(a).with_kernel("segmented"), sp.hybrid_from_csr(a), sp.sellp_from_csr(a)):
        x = out(dev, n, np.float64)
        mat.apply(vec(dev, bv), x)
        assert_close(host(x), ref, rp, v, bv)


@pytest.mark.parametrize("p,dim", [(1000, 2), (128, 3)])
def test_baseline_poisson_bitwise(dev, p, dim):
    """Configs #1/#2 at full size: the production stream kernel is bit-exact with the
    oracle (= the reference's sequential fp64 order)."""
    a = gen.stencil_csr(dev, p, dim=dim)
    assert a.kernel == "stream"
    rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
    frp, fci, fv = fixtures.stencil_csr(p, dim=dim)
    np.testing.assert_array_equal(rp, frp)
    np.testing.assert_array_equal(ci, fci)
    np.testing.assert_array_equal(v, fv)
    bv = np.random.default_rng(0).random(a.rows)
    x = out(dev, a.rows, np.float64)
    a.apply(vec(dev, bv), x)
    np.testing.assert_array_equal(host(x), sbref.csr_spmv(frp, fci, fv, bv, threads=8))
    for conv in (sp.ell_from_csr, sp.sellp_from_csr,
                 lambda m: sp.sellp_from_csr(m).with_staging(False), lambda m: sp.sellp_from_csr(m, 32)):
        y = out(dev, a.rows, np.float64)
        conv(a).apply(vec(dev, bv), y)
        np.testing.assert_array_equal(host(y), host(x))


@pytest.mark.slow
def test_powerlaw_config3_formats(dev):
    """Config #3 (4M rows, power-law) at full size, fp64 and fp32: CSR (auto = nnz tiles,
    and merge-path), COO, SELL-P and Hybrid against the oracle's CSR SpMV; ELL is
    infeasible (560 GB)."""
    n, rows, cols, vals = fixtures.powerlaw_triplets()
    for vdt in (np.float64, np.float32):
        a = gen.powerlaw_csr(dev, precision=sp.Precision.from_dtype(vdt))
        assert a.nnz == 63_958_208
        rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
        bv = np.random.default_rng(0).random(n).astype(vdt)
        ref = sbref.csr_spmv(rp, ci, v, bv, threads=8)
        assert a.kernel == "tile"
        for mat in (a, a.with_kernel("merge"), sp.coo_from_csr(a),
                    sp.coo_from_csr(a).with_kernel("segmented"), sp.sellp_from_csr(a),
                    sp.sellp_from_csr(a, 64, sigma=8192), sp.hybrid_from_csr(a)):
            x = out(dev, n, vdt)
            mat.apply(vec(dev, bv), x)
            assert_close(host(x), ref, rp, v, bv)
            del mat


@pytest.mark.parametrize("vdt", [np.float64, np.float32])  # two-stage / pipelined variants
def test_tile_kernel_edge_cases(dev, vdt):
    """nnz-tile CSR: rows ending exactly on tile boundaries, rows spanning several whole
    tiles, runs of empty rows inside and after the last tile (nnz a multiple of the tile),
    long segments reduced by warps; short rows wholly inside a tile are bit-exact."""
    rng = np.random.default_rng(21)
    C = 2048
    cases = {
        "boundaries": [C, C, 1, C - 1, 3 * C, 0, 0, 5, C + 7, 0],
        "multiple": [C] * 4 + [0] * 9,                      # nnz = 4C, trailing empty rows
        "spanning": [1] * 100 + [5 * C + 3] + [2] * 700 + [0] * 50 + [40] * 90,
        "short": list(rng.integers(0, 33, 5000)),
    }
    for name, lens in cases.items():
        lens = np.asarray(lens, np.int64)
        n = lens.size
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        ci = rng.integers(0, n, int(rp[-1])).astype(np.int32)
        ci = np.concatenate([np.sort(ci[rp[i]:rp[i + 1]]) for i in range(n)]).astype(np.int32) \
            if rp[-1] else ci
        v = rng.standard_normal(int(rp[-1])).astype(vdt)
        bv = rng.standard_normal(n).astype(vdt)
        ref = sbref.csr_spmv(rp, ci, v, bv)
        a = csr(dev, rp, ci, v, n, kernel="tile")
        x = out(dev, n, vdt)
        a.apply(vec(dev, bv), x)
        got = host(x)
        assert_close(got, ref, rp, v, bv)
        # rows of <= 32 entries that do not cross a tile boundary keep the sequential order
        inside = (lens <= 32) & (rp[:-1] // C == np.maximum(rp[1:] - 1, rp[:-1]) // C)
        np.testing.assert_array_equal(got[inside], ref[inside], err_msg=name)


def test_stream_spmm_multi_rhs_bitwise(dev):
    """Multi-RHS apply on stream-CSR matrices uses the SpMM kernel (matrix streamed once
    per 8 / 4 / 2 columns): every column equals the single-vector SpMV bit for bit,
    for k = 2..11 (chunk remainders), strided b / x, fp64 and fp32."""
    rng = np.random.default_rng(31)
    for prec, vdt in ((sp.Precision.double, np.float64), (sp.Precision.single, np.float32)):
        a = gen.stencil_csr(dev, 20, dim=3, precision=prec)
        assert a.kernel == "stream"
        n = a.rows
        for k in (2, 3, 5, 8, 11):
            bm = rng.standard_normal((n, k + 1)).astype(vdt)  # stride k+1: strided view
            b = sp.dense_from_array(dev, bm.copy())
            bview = sp.DenseMatrix(dev, n, k, b.values, stride=k + 1)
            x = out(dev, n, vdt, cols=k)
            a.apply(bview, x)
            got = host(x)
            for j in range(k):
                y = out(dev, n, vdt)
                a.apply(vec(dev, bm[:, j]), y)
                np.testing.assert_array_equal(got[:, j], host(y), err_msg=f"k={k} col={j}")


@pytest.mark.parametrize("vdt", [np.float64, np.float32])
def test_sellp_split_pieces(dev, vdt):
    """SELL-P / SELL-C-sigma blocks far above the average size are cut into pieces
    (sellp_piece_kernel + in-order fix-up): results against the oracle's CSR SpMV within
    the fp tolerance, unsplit blocks bitwise equal to the whole-block kernel, and a CG
    solve through the split operator (row-splitting epilogue pass) matches the CSR run."""
    rng = np.random.default_rng(5)
    n = 40000
    lens = rng.integers(1, 8, n)
    lens[rng.choice(n, 40, replace=False)] = rng.integers(3000, 12000, 40)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    ci = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int32)
    v = rng.standard_normal(rp[-1]).astype(vdt)
    a = csr(dev, rp, ci, v)
    bv = rng.random(n).astype(vdt)
    ref = sbref.csr_spmv(rp, ci, v, bv, threads=8)
    x_whole = out(dev, n, vdt)
    for mat in (sp.sellp_from_csr(a, 64), sp.sellp_from_csr(a, 32), sp.sellp_from_csr(a, 64, sigma=1024)):
        assert mat._pieces is not None and mat._pieces[2] > 0  # some blocks are split
        x = out(dev, n, vdt)
        mat.apply(vec(dev, bv), x)
        assert_close(host(x), ref, rp, v, bv)
        # rows of unsplit blocks: bitwise what the whole-block kernel stores
        whole = sp.SellpMatrix(dev, mat.rows, mat.cols, mat.slice_size, mat.slice_lengths, mat.slice_sets,
                               mat.col_idxs, mat.values, row_perm=mat.row_perm)
        whole._pieces = None
        whole.apply(vec(dev, bv), x_whole)
        plan = mat._pieces[0].cpu().numpy()
        nblk = -(-mat.num_slices // (128 // mat.slice_size))
        one = np.nonzero(np.diff(plan[:nblk + 1]) == 1)[0]
        rows = (one[:, None] * 128 + np.arange(128)[None, :]).ravel()
        rows = rows[rows < n]
        if mat.row_perm is not None:
            rows = mat.row_perm.cpu().numpy()[rows]
        np.testing.assert_array_equal(host(x)[rows], host(x_whole)[rows])
    # a solver through the split operator (row-splitting: epilogue pass), SPD matrix with
    # the same long rows: CG on split SELL-P against CG on CSR
    if vdt == np.float64:
        import scipy.sparse as sps
        B = sps.csr_matrix((np.abs(v).astype(np.float64), ci, rp), shape=(n, n))
        S_ = (B + B.T).tocsr()
        S_ = (S_ + sps.diags(np.asarray(abs(S_).sum(axis=1)).ravel() + 1.0)).tocsr()
        S_.sort_indices()
        spd = csr(dev, S_.indptr.astype(np.int32), S_.indices.astype(np.int32), S_.data)
        sell = sp.sellp_from_csr(spd, 64)
        assert sell._pieces is not None
        crit = [sp.Iteration(500), sp.ResidualNorm(1e-10)]
        logs = []
        for mat in (spd, sell):
            x = vec(dev, np.zeros(n))
            logs.append((sp.Cg(mat, criteria=crit, preconditioner=sp.jacobi_create(spd)).solve(vec(dev, bv), x),
                         host(x)))
        (l0, x0), (l1, x1) = logs
        assert l0.converged and l1.converged and abs(l0.iterations - l1.iterations) <= 1
        np.testing.assert_allclose(x1, x0, rtol=1e-8, atol=1e-10)
        # the other solvers' loops through the row-splitting operator (no gather epilogues)
        for cls, kw in ((sp.Gmres, {"krylov_dim": 20}), (sp.Bicgstab, {}), (sp.Cgs, {})):
            its = []
            for mat in (spd, sell):
                x = vec(dev, np.zeros(n))
                its.append(cls(mat, criteria=crit, preconditioner=sp.jacobi_create(spd), **kw)
                           .solve(vec(dev, bv), x))
            assert its[0].converged and its[1].converged, cls
            assert abs(its[0].iterations - its[1].iterations) <= max(1, its[0].iterations // 50), cls
