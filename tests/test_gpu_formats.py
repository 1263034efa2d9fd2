"""GPU parity: construction, conversion, Jacobi and BLAS-1 against the reference.

Integer / index / layout outputs are compared BIT FOR BIT (the north_star bar for
format conversion and indexing).
"""

import numpy as np
import pytest
import torch

from oracle import fixtures, sbref
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
from tests import golden_io
from tests.gpu_util import csr, host, out, vec

pytestmark = pytest.mark.gpu


def test_coo_from_arrays_matches_reference(dev):
    for m in golden_io.unpack(golden_io.load("canonicalize.npz")):
        rows, cols, vt = (int(t) for t in m["meta"])
        prec = sp.Precision.double if vt == 0 else sp.Precision.single
        coo = sp.coo_from_arrays(dev, rows, cols, m["ri"], m["ci"], m["v"], prec,
                                 sp.IndexWidth.i64)
        np.testing.assert_array_equal(coo.row_idxs.cpu().numpy(), m["out_r"])
        np.testing.assert_array_equal(coo.col_idxs.cpu().numpy(), m["out_c"])
        np.testing.assert_array_equal(coo.values.cpu().numpy().astype(np.float64), m["out_v"])
        a = sp.csr_from_coo(coo)
        np.testing.assert_array_equal(a.row_ptrs.cpu().numpy(), m["row_ptrs"])
        back = sp.coo_from_csr(a)
        np.testing.assert_array_equal(back.row_idxs.cpu().numpy(), m["out_r"])
        assert sp.validate(a) == [] and sp.validate(coo) == []


def test_coo_from_arrays_bounds(dev):
    with pytest.raises(sp.errors.IndexBoundsError) as exc:
        sp.coo_from_arrays(dev, 3, 3, [0, 1, 3], [0, 1, 1], [1.0, 2.0, 3.0])
    assert "triplet 2 at (3, 1) outside 3x3" in str(exc.value)


def test_suite_construction_and_layouts(dev):
    """Every golden matrix: device canonicalisation == reference arrays; ELL / SELL-P /
    Hybrid layouts == the oracle's canonical layouts."""
    suite = fixtures.oracle_suite(60, 2024)
    gold = golden_io.spmv_suite("float64", "int32")
    for (rows, cols, ri, ci, v, _), m in zip(suite, gold):
        a = sp.csr_from_coo(sp.coo_from_arrays(dev, rows, cols, ri, ci, v))
        np.testing.assert_array_equal(a.row_ptrs.cpu().numpy(), m["row_ptrs"])
        np.testing.assert_array_equal(a.col_idxs.cpu().numpy(), m["col_idxs"])
        np.testing.assert_array_equal(a.values.cpu().numpy(), m["values"])
        w, stride, ec, ev = sbref.ell_from_csr(m["row_ptrs"], m["col_idxs"], m["values"])
        e = sp.ell_from_csr(a)
        assert (e.width, e.stride) == (w, stride)
        np.testing.assert_array_equal(e.col_idxs.cpu().numpy(), ec)
        np.testing.assert_array_equal(e.values.cpu().numpy(), ev)
        sl, ss, sc, sv = sbref.sellp_from_csr(m["row_ptrs"], m["col_idxs"], m["values"], 64)
        s = sp.sellp_from_csr(a, 64)
        np.testing.assert_array_equal(s.slice_lengths.cpu().numpy(), sl)
        np.testing.assert_array_equal(s.slice_sets.cpu().numpy(), ss)
        np.testing.assert_array_equal(s.col_idxs.cpu().numpy(), sc)
        np.testing.assert_array_equal(s.values.cpu().numpy(), sv)
        wq = sbref.hybrid_ell_width(np.diff(m["row_ptrs"]))
        hw, hs, hec, hev, tr, tc, tv = sbref.hybrid_from_csr(m["row_ptrs"], m["col_idxs"],
                                                             m["values"], wq)
        h = sp.hybrid_from_csr(a)
        assert h.ell.width == hw
        np.testing.assert_array_equal(h.ell.col_idxs.cpu().numpy(), hec)
        np.testing.assert_array_equal(h.ell.values.cpu().numpy(), hev)
        np.testing.assert_array_equal(h.coo.row_idxs.cpu().numpy(), tr)
        np.testing.assert_array_equal(h.coo.col_idxs.cpu().numpy(), tc)
        np.testing.assert_array_equal(h.coo.values.cpu().numpy(), tv)


@pytest.mark.parametrize("p,dim,c", [(7, 2, 0.0), (33, 2, 0.0), (1, 3, 0.0), (2, 3, 0.0),
                                     (13, 3, 0.0), (13, 3, 0.5)])
def test_stencil_generator(dev, p, dim, c):
    for vdt, idt in ((np.float64, np.int32), (np.float32, np.int64)):
        a = gen.stencil_csr(dev, p, dim=dim, c=c, precision=sp.Precision.from_dtype(vdt),
                            index_width=sp.IndexWidth.from_dtype(idt))
        rp, ci, v = fixtures.stencil_csr(p, dim=dim, c=c, dtype=vdt, index=idt)
        np.testing.assert_array_equal(a.row_ptrs.cpu().numpy(), rp)
        np.testing.assert_array_equal(a.col_idxs.cpu().numpy(), ci)
        np.testing.assert_array_equal(a.values.cpu().numpy(), v)


def test_jacobi_matches_reference(dev):
    g = golden_io.load("stencils.npz")
    for name in ("poisson2d_32", "poisson3d_12", "convdiff3d_12"):
        a = csr(dev, g[f"{name}_row_ptrs"], g[f"{name}_col_idxs"], g[f"{name}_values"])
        m = sp.jacobi_create(a)
        np.testing.assert_array_equal(m.inv_diag.cpu().numpy(), g[f"{name}_inv_diag"])
        np.testing.assert_array_equal(a.diagonal(), 1.0 / g[f"{name}_inv_diag"])
        bv = np.random.default_rng(1).random(a.rows)
        x = out(dev, a.rows, np.float64)
        m.apply(vec(dev, bv), x)
        np.testing.assert_array_equal(host(x), sbref.jacobi_apply(g[f"{name}_inv_diag"], bv))
    # missing and zero diagonals (test_precond.py:31-45)
    a = csr(dev, np.array([0, 1, 2, 3], np.int32), np.array([0, 2, 2], np.int32),
            np.array([2.0, 1.0, 3.0]))
    with pytest.raises(sp.errors.SingularDiagonalError) as exc:
        sp.jacobi_create(a)
    assert exc.value.row == 1
    a = sp.csr_from_dense(dev, np.diag([1.0, 2.0, 0.0, 4.0]), keep_zeros=True)
    with pytest.raises(sp.errors.SingularDiagonalError) as exc:
        sp.jacobi_create(a)
    assert exc.value.row == 2
    with pytest.raises(sp.errors.UnsupportedFeatureError):
        sp.jacobi_create(a, max_block_size=4)
    f32 = sp.csr_from_dense(dev, np.diag([3.0, 7.0]), sp.Precision.single)
    inv = sp.jacobi_create(f32).inv_diag.cpu().numpy()
    np.testing.assert_array_equal(inv, (1.0 / np.array([3.0, 7.0])).astype(np.float32))


@pytest.mark.parametrize("vdt", ["float64", "float32"])
def test_blas1(dev, vdt):
    g = golden_io.load("blas1.npz")
    xv, yv = g[f"{vdt}_x"], g[f"{vdt}_y"]
    x, y = vec(dev, xv), vec(dev, yv)
    # dot / norm2: fp64 accumulation; the device sums in a different (fixed) order
    tol = 1e-12 * np.abs(xv.astype(np.float64) * yv).sum()
    assert abs(sp.dot(x, y) - float(g[f"{vdt}_dot1"])) <= tol
    assert abs(sp.norm2(x) - float(g[f"{vdt}_norm1"])) <= 1e-12 * float(g[f"{vdt}_norm1"])
    assert sp.dot(x, y) == sp.dot(x, y)  # deterministic
    sp.axpy(-0.7310585786300049, x, y)
    np.testing.assert_array_equal(host(y), g[f"{vdt}_axpy"])
    sp.scal(1.0 / 3.0, x)
    np.testing.assert_array_equal(host(x), g[f"{vdt}_scal"])


def test_constructors_from_scipy_and_torch(dev):
    import scipy.sparse as sps

    rng = np.random.default_rng(5)
    m = sps.random(60, 50, density=0.1, random_state=7, format="csr")
    a = sp.from_scipy(dev, m)
    np.testing.assert_allclose(a.to_dense(), m.toarray(), rtol=0, atol=0)
    t = torch.tensor(m.toarray()).to_sparse_csr()
    b = sp.from_torch(dev, t)
    np.testing.assert_array_equal(b.to_dense(), m.toarray())
    dense = torch.tensor(rng.standard_normal((8, 9)))
    c = sp.from_torch(dev, dense.cuda(), format="coo")
    np.testing.assert_array_equal(c.to_dense(), dense.numpy())


def test_matrix_market_roundtrip(dev, tmp_path):
    rng = np.random.default_rng(6)
    rp, ci, v = fixtures.canonical_csr(30, *fixtures.random_sparse_triplets(rng, 30, 30, 0.2))
    a = csr(dev, rp, ci, v)
    path = tmp_path / "a.mtx"
    sp.write_matrix_market(a, path)
    b = sp.read_matrix_market(dev, path)
    np.testing.assert_array_equal(b.row_ptrs.cpu().numpy(), rp)
    np.testing.assert_array_equal(b.values.cpu().numpy(), v)
    (tmp_path / "s.mtx").write_text(
        "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 2\n2 1 -1\n3 2 -1\n3 3 2\n")
    s = sp.read_matrix_market(dev, tmp_path / "s.mtx")
    np.testing.assert_array_equal(s.to_dense(), [[2, -1, 0], [-1, 0, -1], [0, -1, 2]])
