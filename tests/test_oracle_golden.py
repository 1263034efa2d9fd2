"""Pin the CPU oracle (oracle/sbref.cpp) to vectors produced by the reference itself.

The golden files were written by tests/golden/make_golden.py running the
unmodified reference (``sparseops``).  Integer/index outputs and SpMV/BLAS-1/solver
outputs must match BIT FOR BIT: the oracle restates the reference's arithmetic
order exactly, which is what makes it a trustworthy checker for the GPU path.
"""

import os

import numpy as np
import pytest

from oracle import fixtures, sbref
from tests import golden_io

VDTS = ["float64", "float32"]
IDTS = ["int32", "int64"]


@pytest.mark.parametrize("vdt", VDTS)
@pytest.mark.parametrize("idt", IDTS)
def test_spmv_suite_bitwise(vdt, idt):
    for m in golden_io.spmv_suite(vdt, idt):
        x = sbref.csr_spmv(m["row_ptrs"], m["col_idxs"], m["values"], m["b"])
        np.testing.assert_array_equal(x, m["x"])
        rows = int(m["shape"][0])
        ri = np.repeat(np.arange(rows), np.diff(m["row_ptrs"])).astype(m["col_idxs"].dtype)
        y = sbref.coo_spmv(rows, ri, m["col_idxs"], m["values"], m["b"])
        np.testing.assert_array_equal(y, m["x"])
        # any thread count is bitwise identical (reference omp device, test_linop.py:90-106)
        x3 = sbref.csr_spmv(m["row_ptrs"], m["col_idxs"], m["values"], m["b"], threads=3)
        np.testing.assert_array_equal(x3, m["x"])


def test_suite_regenerates_from_fixtures():
    """The fixture generator reproduces the reference suite's matrices exactly."""
    suite = fixtures.oracle_suite(60, 2024)
    gold = golden_io.spmv_suite("float64", "int32")
    for (rows, cols, ri, ci, v, bv), m in zip(suite, gold):
        rp, c, vals = fixtures.canonical_csr(rows, ri, ci, v)
        np.testing.assert_array_equal(rp, m["row_ptrs"])
        np.testing.assert_array_equal(c, m["col_idxs"])
        np.testing.assert_array_equal(vals, m["values"])
        np.testing.assert_array_equal(bv, m["b"])


def test_canonicalization_bitwise():
    for m in golden_io.unpack(golden_io.load("canonicalize.npz")):
        rows, cols, vt = (int(t) for t in m["meta"])
        dt = np.float64 if vt == 0 else np.float32
        r, c, v = sbref.coo_canonicalize(m["ri"], m["ci"], m["v"], dt)
        np.testing.assert_array_equal(r, m["out_r"])
        np.testing.assert_array_equal(c, m["out_c"])
        np.testing.assert_array_equal(v.astype(np.float64), m["out_v"])
        np.testing.assert_array_equal(sbref.csr_row_ptrs(r, rows, np.int64), m["row_ptrs"])


@pytest.mark.parametrize("name,dim,c", [("poisson2d_32", 2, 0.0), ("poisson3d_12", 3, 0.0),
                                        ("convdiff3d_12", 3, 0.5)])
def test_stencils_spmv_and_jacobi(name, dim, c):
    g = golden_io.load("stencils.npz")
    p = int(name.split("_")[1])
    rp, ci, v = fixtures.stencil_csr(p, dim=dim, c=c)
    np.testing.assert_array_equal(rp, g[f"{name}_row_ptrs"])
    np.testing.assert_array_equal(ci, g[f"{name}_col_idxs"])
    np.testing.assert_array_equal(v, g[f"{name}_values"])
    x = sbref.csr_spmv(rp, ci, v, g[f"{name}_b"])
    np.testing.assert_array_equal(x, g[f"{name}_x"])
    inv, row = sbref.jacobi_create(rp, ci, v)
    assert row is None
    np.testing.assert_array_equal(inv, g[f"{name}_inv_diag"])


@pytest.mark.parametrize("vdt", VDTS)
def test_blas1_bitwise(vdt):
    g = golden_io.load("blas1.npz")
    x, y = g[f"{vdt}_x"], g[f"{vdt}_y"]
    assert sbref.dot(x, y) == float(g[f"{vdt}_dot1"])
    assert sbref.dot(x, y, threads=3) == float(g[f"{vdt}_dot3"])
    assert sbref.norm2(x) == float(g[f"{vdt}_norm1"])
    np.testing.assert_array_equal(sbref.axpy(-0.7310585786300049, x, y), g[f"{vdt}_axpy"])
    np.testing.assert_array_equal(sbref.scal(1.0 / 3.0, x), g[f"{vdt}_scal"])


def test_solvers_bitwise():
    meta = golden_io.solver_meta()
    g = golden_io.load("solvers.npz")
    for name, m in meta.items():
        if name.startswith("_"):
            continue
        dt = np.dtype(m["dtype"])
        rp, ci, v = fixtures.stencil_csr(m["p"], c=m["c"], dtype=dt)
        inv, _ = sbref.jacobi_create(rp, ci, v)
        b = np.ones(rp.size - 1, dt)
        log, x = sbref.solve(m["solver"], rp, ci, v, b, inv_diag=inv, max_iters=m["max_iters"],
                             reduction_factor=m["reduction_factor"],
                             krylov_dim=m["krylov_dim"] or 30)
        assert log.status == 0, name
        assert log.iterations == m["iterations"], name
        assert log.converged == m["converged"], name
        assert log.stop_reason == m["stop_reason"], name
        np.testing.assert_array_equal(np.asarray(log.residual_history), g[f"{name}_history"],
                                      err_msg=name)
        np.testing.assert_array_equal(x, g[f"{name}_x"], err_msg=name)


def test_jacobi_singular_row():
    rp = np.array([0, 1, 2, 3], np.int32)
    ci = np.array([0, 2, 2], np.int32)   # row 1 has no diagonal
    v = np.array([2.0, 1.0, 3.0])
    inv, row = sbref.jacobi_create(rp, ci, v)
    assert inv is None and row == 1


def test_cg_breakdown_on_zero_matrix():
    """test_solvers.py:107-112: the zero operator breaks down at iteration 1."""
    rp = np.array([0, 0, 0], np.int32)
    log, _ = sbref.solve("cg", rp, np.zeros(0, np.int32), np.zeros(0), np.array([1.0, 2.0]),
                         max_iters=10)
    assert log.status == 1 and log.status_iteration == 1


def test_ell_sellp_layouts_roundtrip():
    """ELL / SELL-P SpMV over the canonical layouts equal reference CSR SpMV bitwise
    (same per-row order, padding skipped)."""
    for m in golden_io.spmv_suite("float64", "int32")[:30]:
        rp, ci, v, b = m["row_ptrs"], m["col_idxs"], m["values"], m["b"]
        rows = rp.size - 1
        w, stride, ec, ev = sbref.ell_from_csr(rp, ci, v)
        np.testing.assert_array_equal(sbref.ell_spmv(rows, w, stride, ec, ev, b), m["x"])
        sl, ss, sc, sv = sbref.sellp_from_csr(rp, ci, v, 64)
        np.testing.assert_array_equal(sbref.sellp_spmv(rows, 64, sl, ss, sc, sv, b), m["x"])


def _transpose(rp, ci, v):
    n = rp.size - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    order = np.lexsort((rows, ci))
    tp = np.concatenate([[0], np.cumsum(np.bincount(ci, minlength=n))]).astype(rp.dtype)
    return tp, rows[order].astype(ci.dtype), v[order]


@pytest.mark.parametrize("vdt", ["float64", "float32"])
def test_oracle_factorizations_match_reference(vdt):
    """ILU(0) factors + apply, IC(0) factor + apply: the oracle restatement equals the
    reference's outputs (tests/golden/factor_*.npz) bit for bit."""
    for m in golden_io.unpack(golden_io.load(f"factor_{vdt}.npz")):
        rp, ci, v, b = m["row_ptrs"], m["col_idxs"], m["values"], m["b"]
        st, fv = sbref.ilu0(rp, ci, v)
        assert st == -1
        (lp, lc, lv), (up, uc, uv) = sbref.split_lu(rp, ci, fv)
        for got, want in ((lp, m["ilu_l_ptrs"]), (lc, m["ilu_l_cols"]), (lv, m["ilu_l_vals"]),
                          (up, m["ilu_u_ptrs"]), (uc, m["ilu_u_cols"]), (uv, m["ilu_u_vals"])):
            np.testing.assert_array_equal(got, want)
        s1, _, y = sbref.trsv(lp, lc, lv, b, lower=True, unit_diag=True)
        s2, _, x = sbref.trsv(up, uc, uv, y, lower=False)
        assert s1 == s2 == 0
        np.testing.assert_array_equal(x, m["ilu_x"])
        if m["ic_l_ptrs"].size:
            st, (gp, gc, gv) = sbref.ic0(rp, ci, v)
            assert st == -1
            np.testing.assert_array_equal(gp, m["ic_l_ptrs"])
            np.testing.assert_array_equal(gc, m["ic_l_cols"])
            np.testing.assert_array_equal(gv, m["ic_l_vals"])
            s1, _, y = sbref.trsv(gp, gc, gv, b, lower=True)
            tp, tc, tv = _transpose(gp, gc, gv)
            s2, _, x = sbref.trsv(tp, tc, tv, y, lower=False)
            assert s1 == s2 == 0
            np.testing.assert_array_equal(x, m["ic_x"])


def test_oracle_factorization_errors_match_reference():
    import json
    with open(os.path.join(golden_io.GOLDEN, "factor.json")) as fh:
        errs = json.load(fh)["errors"]
    def csr_of(dense, keep=True):
        r, c = np.nonzero(np.ones_like(dense)) if keep else np.nonzero(dense)
        return fixtures.canonical_csr(dense.shape[0], r, c, dense[r, c])
    assert sbref.ilu0(*csr_of(np.array([[0.0, 1.0], [1.0, 0.0]])))[0] == errs["ilu_zero_pivot"][1]
    late = np.eye(5) * 2.0
    late[3, 3] = 0.0
    rr, cc = np.nonzero(np.eye(5))
    rp, ci, v = fixtures.canonical_csr(5, rr, cc, late[rr, cc])
    assert sbref.ilu0(rp, ci, v)[0] == errs["ilu_zero_pivot_row3"][1]
    assert sbref.ic0(*csr_of(np.diag([1.0, 4.0, -1.0, 2.0]), keep=False))[0] == errs["ic_indefinite"][1]
    up = csr_of(np.triu(np.ones((4, 4))), keep=False)
    assert sbref.trsv(*up, np.ones(4), lower=True)[:2] == (1, errs["lower_not_triangular"][1])
    lo = csr_of(np.tril(np.ones((4, 4))), keep=False)
    assert sbref.trsv(*lo, np.ones(4), lower=False)[:2] == (1, errs["upper_not_triangular"][1])
    for lower, z, key in ((True, 2, "lower_singular"), (False, 1, "upper_singular")):
        mask = np.tril(np.ones((4, 4))) if lower else np.triu(np.ones((4, 4)))
        dense = mask.copy()
        dense[z, z] = 0.0
        r, c = np.nonzero(mask)
        rp, ci, v = fixtures.canonical_csr(4, r, c, dense[r, c])
        assert sbref.trsv(rp, ci, v, np.ones(4), lower=lower)[:2] == (2, errs[key][1])
