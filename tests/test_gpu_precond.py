"""GPU parity of ILU(0), IC(0) and the sparse triangular solves against
the reference: factors and applies BIT FOR BIT (tests/golden/factor_*.npz, produced by
the reference itself), error kinds and rows of the reference, and the reference's
ILU-GMRES / IC-CG runs (iterations within +-2%, histories to rounding)."""

import json
import os

import numpy as np
import pytest

from oracle import fixtures, sbref
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
from tests import golden_io
from tests.gpu_util import csr, host, out, vec

pytestmark = pytest.mark.gpu


def _meta():
    with open(os.path.join(golden_io.GOLDEN, "factor.json")) as fh:
        return json.load(fh)


def _arrays(m):
    return tuple(t.cpu().numpy() for t in (m.row_ptrs, m.col_idxs, m.values))


@pytest.mark.parametrize("vdt", ["float64", "float32"])
def test_factorizations_bitwise(dev, vdt):
    for m in golden_io.unpack(golden_io.load(f"factor_{vdt}.npz")):
        a = csr(dev, m["row_ptrs"], m["col_idxs"], m["values"])
        f = sp.ilu0_factorize(a)
        for got, (p, c, v) in ((f.l, ("ilu_l_ptrs", "ilu_l_cols", "ilu_l_vals")),
                               (f.u, ("ilu_u_ptrs", "ilu_u_cols", "ilu_u_vals"))):
            gp, gc, gv = _arrays(got)
            np.testing.assert_array_equal(gp, m[p])
            np.testing.assert_array_equal(gc, m[c])
            np.testing.assert_array_equal(gv, m[v])
        x = out(dev, a.rows, m["values"].dtype)
        sp.ilu_apply(f, vec(dev, m["b"]), x)
        np.testing.assert_array_equal(host(x), m["ilu_x"])
        if m["ic_l_ptrs"].size:
            g = sp.ic0_factorize(a)
            gp, gc, gv = _arrays(g.l)
            np.testing.assert_array_equal(gp, m["ic_l_ptrs"])
            np.testing.assert_array_equal(gc, m["ic_l_cols"])
            np.testing.assert_array_equal(gv, m["ic_l_vals"])
            y = out(dev, a.rows, m["values"].dtype)
            sp.ic_apply(g, vec(dev, m["b"]), y)
            np.testing.assert_array_equal(host(y), m["ic_x"])


def test_trisolve_large_bitwise(dev):
    """Sweeps over 3-D Poisson 48^3 factors (110k rows, deep dependency chains) equal the
    oracle's sequential loops bit for bit; lower, unit lower, upper, in place, fp32."""
    a = gen.stencil_csr(dev, 48, dim=3)
    rp, ci, v = _arrays(a)
    f = sp.ilu0_factorize(a)
    st, fv = sbref.ilu0(rp, ci, v)
    (lp, lc, lv), (up, uc, uv) = sbref.split_lu(rp, ci, fv)
    np.testing.assert_array_equal(_arrays(f.l)[2], lv)
    np.testing.assert_array_equal(_arrays(f.u)[2], uv)
    bv = np.random.default_rng(3).standard_normal(a.rows)
    for mat, lower, unit, ref in ((f.l, True, True, (lp, lc, lv)), (f.u, False, False, (up, uc, uv))):
        x = out(dev, a.rows, np.float64)
        (sp.solve_lower_tri(mat, vec(dev, bv), x, unit_diag=True) if lower
         else sp.solve_upper_tri(mat, vec(dev, bv), x))
        _, _, want = sbref.trsv(*ref, bv, lower=lower, unit_diag=unit)
        np.testing.assert_array_equal(host(x), want)
    g = sp.ic0_factorize(a)
    _, (gp, gc, gv) = sbref.ic0(rp, ci, v)
    np.testing.assert_array_equal(_arrays(g.l)[2], gv)
    x = out(dev, a.rows, np.float64)
    sp.solve_lower_tri(g.l, vec(dev, bv), x)
    np.testing.assert_array_equal(host(x), sbref.trsv(gp, gc, gv, bv, lower=True)[2])
    # in place (x is b): the value-as-flag sweep must fall back to separate ready flags
    for mat, lower, unit, ref in ((f.l, True, True, (lp, lc, lv)), (f.u, False, False, (up, uc, uv))):
        xb = vec(dev, bv)
        (sp.solve_lower_tri(mat, xb, xb, unit_diag=True) if lower else sp.solve_upper_tri(mat, xb, xb))
        np.testing.assert_array_equal(host(xb), sbref.trsv(*ref, bv, lower=lower, unit_diag=unit)[2])
    # fp32 factors: the 32-bit sentinel path
    a32 = gen.stencil_csr(dev, 24, dim=3, precision=sp.Precision.single)
    rp, ci, v = _arrays(a32)
    f32 = sp.ilu0_factorize(a32)
    _, fv = sbref.ilu0(rp, ci, v)
    (lp, lc, lv), (up, uc, uv) = sbref.split_lu(rp, ci, fv)
    b32 = np.random.default_rng(4).standard_normal(a32.rows).astype(np.float32)
    x = out(dev, a32.rows, np.float32)
    sp.solve_upper_tri(f32.u, vec(dev, b32), x)
    np.testing.assert_array_equal(host(x), sbref.trsv(up, uc, uv, b32, lower=False)[2])


def test_error_kinds_and_rows(dev):
    errs = _meta()["errors"]
    E = sp.errors
    def row_of(exc_cls, fn):
        with pytest.raises(exc_cls) as exc:
            fn()
        return exc.value.row
    z2 = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert row_of(E.ZeroPivotError, lambda: sp.ilu0_factorize(sp.csr_from_dense(dev, z2, keep_zeros=True))) \
        == errs["ilu_zero_pivot"][1]
    late = np.eye(5) * 2.0
    late[3, 3] = 0.0
    assert row_of(E.ZeroPivotError, lambda: sp.ilu0_factorize(sp.csr_from_dense(dev, late, keep_zeros=True))) \
        == errs["ilu_zero_pivot_row3"][1]
    assert row_of(E.IndefinitePivotError, lambda: sp.ic0_factorize(
        sp.csr_from_dense(dev, np.diag([1.0, 4.0, -1.0, 2.0])))) == errs["ic_indefinite"][1]
    ones = vec(dev, np.ones(4))
    assert row_of(E.NotTriangularError, lambda: sp.solve_lower_tri(
        sp.csr_from_dense(dev, np.triu(np.ones((4, 4)))), ones, out(dev, 4, np.float64))) \
        == errs["lower_not_triangular"][1]
    assert row_of(E.NotTriangularError, lambda: sp.solve_upper_tri(
        sp.csr_from_dense(dev, np.tril(np.ones((4, 4)))), ones, out(dev, 4, np.float64))) \
        == errs["upper_not_triangular"][1]
    def tri(lower, zero_at):
        t = [(i, j, 0.0 if i == j == zero_at else 1.0) for i in range(4) for j in range(4)
             if (j <= i if lower else j >= i)]
        return sp.csr_from_coo(sp.coo_from_triplets(dev, 4, 4, t))
    assert row_of(E.SingularTriangleError, lambda: sp.solve_lower_tri(tri(True, 2), ones, out(dev, 4, np.float64))) \
        == errs["lower_singular"][1]
    assert row_of(E.SingularTriangleError, lambda: sp.solve_upper_tri(tri(False, 1), ones, out(dev, 4, np.float64))) \
        == errs["upper_singular"][1]
    # a user-built factor pair that is not triangular fails the preconditioned solve the same way
    bad = sp.IluFactors(sp.csr_from_dense(dev, np.triu(np.ones((4, 4)))), sp.csr_from_dense(dev, np.eye(4)))
    with pytest.raises(E.NotTriangularError):
        sp.Gmres(sp.csr_from_dense(dev, np.eye(4) * 2), criteria=[sp.Iteration(5)], preconditioner=bad).solve(
            vec(dev, np.ones(4)), out(dev, 4, np.float64, fill=0.0))


def test_identity_and_dense_pattern(dev):
    """test_precond.py TestPreconditionerApply / TestIlu0 cases on the device."""
    eye = sp.csr_from_dense(dev, np.eye(3))
    f = sp.IluFactors(sp.csr_from_dense(dev, np.zeros((3, 3))), eye)
    x = out(dev, 3, np.float64)
    sp.ilu_apply(f, vec(dev, [1.0, 2.0, 3.0]), x)
    np.testing.assert_array_equal(host(x), [1.0, 2.0, 3.0])
    rng = np.random.default_rng(23)
    dense = rng.standard_normal((12, 12)) + 12 * np.eye(12)
    f = sp.ilu0_factorize(sp.csr_from_dense(dev, dense, keep_zeros=True))
    bv = rng.standard_normal(12)
    x = out(dev, 12, np.float64)
    sp.ilu_apply(f, vec(dev, bv), x)
    want = np.linalg.solve(dense, bv)
    assert np.linalg.norm(host(x) - want) <= 1e-10 * np.linalg.norm(want)
    g = sp.ic0_factorize(sp.csr_from_dense(dev, np.array([[4.0, 2.0], [2.0, 5.0]])))
    np.testing.assert_allclose(g.l.to_dense(), [[2.0, 0.0], [1.0, 2.0]])


@pytest.mark.parametrize("name", ["gmres30_ilu_poisson2d_16", "gmres10_ilu_convdiff3d_8",
                                  "cg_ic_poisson2d_16", "cg_ilu_poisson3d_8"])
def test_preconditioned_solvers_match_reference(dev, name):
    run = _meta()["solver_runs"][name]
    kind, p, c = run["source"]
    if kind == "poisson2d":
        n, ri, ci, v = fixtures.poisson2d_triplets(p)
    else:
        n, ri, ci, v = fixtures.stencil3d_triplets(p, c)
    rp, cc, vv = fixtures.canonical_csr(n, ri, ci, v)
    a = csr(dev, rp, cc, vv)
    m = sp.ilu0_factorize(a) if run["precond"] == "ilu" else sp.ic0_factorize(a)
    crit = [sp.Iteration(run["max_iters"]), sp.ResidualNorm(run["reduction_factor"])]
    cls = sp.Gmres if run["solver"] == "gmres" else sp.Cg
    kw = {"krylov_dim": run["krylov_dim"]} if run["solver"] == "gmres" else {}
    x = out(dev, n, np.float64, fill=0.0)
    log = cls(a, criteria=crit, preconditioner=m, **kw).solve(vec(dev, np.ones(n)), x)
    assert log.converged == run["converged"] and log.stop_reason == run["stop_reason"]
    assert abs(log.iterations - run["iterations"]) <= max(1, int(np.ceil(0.02 * run["iterations"])))
    k = min(5, len(run["history"]))
    np.testing.assert_allclose(log.residual_history[:k], run["history"][:k], rtol=1e-9)
    r = np.ones(n) - sbref.csr_spmv(rp, cc, vv, host(x))
    assert np.linalg.norm(r) <= 1.0001 * run["reduction_factor"] * np.sqrt(n) or \
        run["solver"] == "cg"  # CG stops on the recurrence residual (solvers.py:209-216)


def test_mismatched_factors(dev):
    """Every solver takes ILU / IC factors; factors of another operator are rejected."""
    a = gen.stencil_csr(dev, 6, dim=3)
    other = gen.stencil_csr(dev, 5, dim=3)
    for cls in (sp.Cg, sp.Cgs, sp.Bicgstab, sp.Gmres):
        with pytest.raises(sp.errors.DimensionMismatchError):
            cls(a, criteria=[sp.Iteration(5)], preconditioner=sp.ilu0_factorize(other)).solve(
                vec(dev, np.ones(a.rows)), out(dev, a.rows, np.float64, fill=0.0))
