"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference (``sparseops`` from
/root/reference/pkg/src), feeds it the fixture matrices of oracle/fixtures.py and
records its outputs bit for bit in small ``.npz`` files next to this script.
The GPU box never reads /root/reference: tests there use these committed files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import sparseops as sp  # noqa: E402  (the reference)

from oracle import fixtures  # noqa: E402

REF = sp.create_device("reference")
PREC = {np.float64: sp.Precision.double, np.float32: sp.Precision.single}
WIDTH = {np.int32: sp.IndexWidth.i32, np.int64: sp.IndexWidth.i64}


def ref_csr(rows, cols, ri, ci, v, vdt=np.float64, idt=np.int32):
    coo = sp.coo_from_arrays(REF, rows, cols, ri, ci, v, PREC[vdt], WIDTH[idt])
    return sp.csr_from_coo(coo)


def vec(a, dt):
    return sp.dense_from_array(REF, np.asarray(a, dtype=dt).copy())


def pack(mats):
    """Concatenate a list of dicts of arrays with offsets (one npz instead of hundreds)."""
    out = {}
    keys = mats[0].keys()
    for k in keys:
        arrs = [np.atleast_1d(m[k]) for m in mats]
        out[k] = np.concatenate(arrs) if arrs else np.zeros(0)
        out[k + "_off"] = np.concatenate([[0], np.cumsum([a.size for a in arrs])]).astype(np.int64)
    return out


def spmv_suite():
    """First 60 matrices of the acceptance oracle suite (seed 2024), every
    value/index instantiation: CSR and COO SpMV outputs of the reference."""
    suite = fixtures.oracle_suite(60, 2024)
    for vdt in (np.float64, np.float32):
        for idt in (np.int32, np.int64):
            mats = []
            for rows, cols, ri, ci, v, bv in suite:
                a = ref_csr(rows, cols, ri, ci, v, vdt, idt)
                b = vec(bv, vdt)
                x = sp.dense_create(REF, rows, 1, PREC[vdt], np.nan)
                sp.spmv_csr(a, b, x)
                y = sp.dense_create(REF, rows, 1, PREC[vdt], np.nan)
                sp.spmv_coo(sp.coo_from_csr(a), b, y)
                assert np.array_equal(x.values, y.values)
                mats.append(dict(shape=np.array([rows, cols], np.int64), row_ptrs=a.row_ptrs,
                                 col_idxs=a.col_idxs, values=a.values, b=b.values, x=x.values))
            name = f"spmv_suite_{np.dtype(vdt).name}_{np.dtype(idt).name}.npz"
            np.savez_compressed(os.path.join(HERE, name), **pack(mats))


def canonicalization():
    """coo_from_arrays on raw triplets with duplicates, out of order, explicit zeros."""
    rng = np.random.default_rng(11)
    cases = []
    for rows, cols, m in ((7, 5, 40), (50, 60, 900), (1, 1, 5), (300, 3, 2000)):
        ri = rng.integers(0, rows, m)
        ci = rng.integers(0, cols, m)
        v = rng.standard_normal(m)
        v[rng.random(m) < 0.1] = 0.0
        cases.append((rows, cols, ri, ci, v))
    mats = []
    for vdt in (np.float64, np.float32):
        for rows, cols, ri, ci, v in cases:
            coo = sp.coo_from_arrays(REF, rows, cols, ri, ci, v, PREC[vdt], sp.IndexWidth.i64)
            csr = sp.csr_from_coo(coo)
            mats.append(dict(meta=np.array([rows, cols, 0 if vdt == np.float64 else 1], np.int64),
                             ri=ri.astype(np.int64), ci=ci.astype(np.int64), v=v,
                             out_r=coo.row_idxs, out_c=coo.col_idxs,
                             out_v=coo.values.astype(np.float64), row_ptrs=csr.row_ptrs))
    np.savez_compressed(os.path.join(HERE, "canonicalize.npz"), **pack(mats))


def stencils_and_jacobi():
    out = {}
    for name, (p, dim, c) in {"poisson2d_32": (32, 2, 0.0), "poisson3d_12": (12, 3, 0.0),
                              "convdiff3d_12": (12, 3, 0.5)}.items():
        if dim == 2:
            n, ri, ci, v = fixtures.poisson2d_triplets(p)
        else:
            n, ri, ci, v = fixtures.stencil3d_triplets(p, c)
        a = ref_csr(n, n, ri, ci, v)
        bv = np.random.default_rng(0).random(n)
        x = sp.dense_create(REF, n, 1, sp.Precision.double, 0.0)
        sp.spmv_csr(a, vec(bv, np.float64), x)
        jac = sp.jacobi_create(a)
        out[f"{name}_row_ptrs"] = a.row_ptrs
        out[f"{name}_col_idxs"] = a.col_idxs
        out[f"{name}_values"] = a.values
        out[f"{name}_b"] = bv
        out[f"{name}_x"] = x.values
        out[f"{name}_inv_diag"] = jac.inv_diag
    np.savez_compressed(os.path.join(HERE, "stencils.npz"), **out)


def solver_goldens():
    """Reference solver runs: iteration counts, residual histories and final x."""
    out, meta = {}, {}
    runs = [
        # name, generator args, solver class, precision, criteria, krylov_dim
        ("cg_jacobi_poisson3d_16", (16, 0.0), "Cg", np.float64, 100000, 1e-8, None),
        ("cg_jacobi_poisson3d_16_f32", (16, 0.0), "Cg", np.float32, 100000, 1e-5, None),
        ("gmres30_jacobi_convdiff3d_16", (16, 0.5), "Gmres", np.float64, 5000, 1e-8, 30),
        ("cgs_jacobi_convdiff3d_16", (16, 0.5), "Cgs", np.float64, 5000, 1e-8, None),
        ("cg_fixed25_poisson3d_12", (12, 0.0), "Cg", np.float64, 25, None, None),
        ("gmres5_fixed45_poisson3d_12", (12, 0.0), "Gmres", np.float64, 45, None, 5),
        ("gmres10_jacobi_convdiff3d_12", (12, 0.5), "Gmres", np.float64, 5000, 1e-9, 10),
        ("cg_jacobi_poisson3d_32", (32, 0.0), "Cg", np.float64, 100000, 1e-8, None),
        ("gmres30_jacobi_convdiff3d_32", (32, 0.5), "Gmres", np.float64, 5000, 1e-8, 30),
    ]
    for name, (p, c), cls, vdt, max_iters, rf, dim in runs:
        n, ri, ci, v = fixtures.stencil3d_triplets(p, c)
        a = ref_csr(n, n, ri, ci, v, vdt)
        crit = [sp.Iteration(max_iters)] + ([sp.ResidualNorm(rf)] if rf else [])
        m = sp.jacobi_create(a)
        b = sp.dense_create(REF, n, 1, PREC[vdt], 1.0)
        x = sp.dense_create(REF, n, 1, PREC[vdt], 0.0)
        kw = {"krylov_dim": dim} if cls == "Gmres" else {}
        log = getattr(sp, cls)(a, criteria=crit, preconditioner=m, **kw).solve(b, x)
        meta[name] = dict(p=p, c=c, solver=cls.lower(), dtype=np.dtype(vdt).name,
                          max_iters=max_iters, reduction_factor=rf, krylov_dim=dim,
                          iterations=log.iterations, converged=log.converged,
                          stop_reason=log.stop_reason)
        out[f"{name}_history"] = np.asarray(log.residual_history, np.float64)
        out[f"{name}_x"] = x.values.copy()
    np.savez_compressed(os.path.join(HERE, "solvers.npz"), **out)
    # counts measured with this same reference in the survey container;
    # too slow to rerun here, recorded as constants.
    meta["_survey_probe"] = {
        "cg_jacobi_poisson3d_rtol1e-8": {"16": 39, "32": 79, "64": 159, "96": 239,
                                         "128": 319, "256": 611},
        "gmres30_jacobi_convdiff3d_c0.5_rtol1e-8": {"16": 81, "32": 227, "64": 330, "128": 585},
    }
    with open(os.path.join(HERE, "solvers.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def blas1():
    """dot / axpy / scal / norm2 bit patterns (reference device and omp[3])."""
    rng = np.random.default_rng(5)
    out = {}
    for vdt in (np.float64, np.float32):
        nm = np.dtype(vdt).name
        xv = rng.standard_normal(20001).astype(vdt)
        yv = rng.standard_normal(20001).astype(vdt)
        x, y = vec(xv, vdt), vec(yv, vdt)
        out[f"{nm}_x"], out[f"{nm}_y"] = xv, yv
        out[f"{nm}_dot1"] = np.float64(sp.dot(x, y))
        omp3 = sp.create_device("omp", threads=3)
        x3 = sp.dense_from_array(omp3, xv.copy())
        y3 = sp.dense_from_array(omp3, yv.copy())
        out[f"{nm}_dot3"] = np.float64(sp.dot(x3, y3))
        out[f"{nm}_norm1"] = np.float64(sp.norm2(x))
        yy = vec(yv, vdt)
        sp.axpy(-0.7310585786300049, x, yy)
        out[f"{nm}_axpy"] = yy.values.copy()
        xx = vec(xv, vdt)
        sp.scal(1.0 / 3.0, xx)
        out[f"{nm}_scal"] = xx.values.copy()
    np.savez_compressed(os.path.join(HERE, "blas1.npz"), **out)


def factorizations():
    """ILU(0), IC(0) and the triangular solves (precond.py:155-287, _kernels.py:91-137):
    factor values, apply outputs and the error rows of the reference, for fp64 and fp32
    on stencils and random diagonally dominant / SPD matrices; plus ILU-preconditioned
    GMRES and IC-preconditioned CG runs (the README's Listing 1 pipeline)."""
    rng = np.random.default_rng(77)
    mats, meta = [], []
    cases = []
    for vdt in (np.float64, np.float32):
        cases.append(("poisson2d_9", fixtures.poisson2d_triplets(9), vdt, True))
        cases.append(("convdiff3d_6", fixtures.stencil3d_triplets(6, 0.5), vdt, False))
        for t in range(3):
            n = int(rng.integers(20, 90))
            rows, cols, vals = fixtures.random_sparse_triplets(rng, n, n, 0.08)
            d = np.arange(n)
            # diagonally dominant nonsymmetric (ILU) and its symmetric part (IC)
            rr = np.concatenate([rows, d]); cc = np.concatenate([cols, d])
            vv = np.concatenate([vals, np.full(n, 0.0)])
            a0 = ref_csr(n, n, rr, cc, vv, np.float64).to_dense()
            dense = a0 + np.diag(np.abs(a0).sum(axis=1) + 1.0)
            r2, c2 = np.nonzero(dense)
            cases.append((f"rand{t}", (n, r2, c2, dense[r2, c2]), vdt, False))
            sym = dense + dense.T
            r3, c3 = np.nonzero(sym)
            cases.append((f"randspd{t}", (n, r3, c3, sym[r3, c3]), vdt, True))
    for name, (n, ri, ci, v), vdt, spd in cases:
        a = ref_csr(n, n, ri, ci, v, vdt)
        bv = rng.standard_normal(n).astype(vdt)
        f = sp.ilu0_factorize(a)
        y = sp.dense_create(REF, n, 1, PREC[vdt], 0.0)
        sp.ilu_apply(f, vec(bv, vdt), y)
        rec = dict(row_ptrs=a.row_ptrs, col_idxs=a.col_idxs, values=a.values, b=bv,
                   ilu_l_ptrs=f.l.row_ptrs, ilu_l_cols=f.l.col_idxs, ilu_l_vals=f.l.values,
                   ilu_u_ptrs=f.u.row_ptrs, ilu_u_cols=f.u.col_idxs, ilu_u_vals=f.u.values,
                   ilu_x=y.values.copy())
        if spd:
            g = sp.ic0_factorize(a)
            z = sp.dense_create(REF, n, 1, PREC[vdt], 0.0)
            sp.ic_apply(g, vec(bv, vdt), z)
            rec.update(ic_l_ptrs=g.l.row_ptrs, ic_l_cols=g.l.col_idxs, ic_l_vals=g.l.values,
                       ic_x=z.values.copy())
        else:
            for k in ("ic_l_ptrs", "ic_l_cols"):
                rec[k] = np.zeros(0, a.col_idxs.dtype)
            rec["ic_l_vals"] = np.zeros(0, vdt)
            rec["ic_x"] = np.zeros(0, vdt)
        mats.append({k: np.asarray(v_) for k, v_ in rec.items()})
        meta.append(dict(name=name, dtype=np.dtype(vdt).name, spd=spd))
    for vdt in (np.float64, np.float32):
        sel = [m for m, md in zip(mats, meta) if md["dtype"] == np.dtype(vdt).name]
        np.savez_compressed(os.path.join(HERE, f"factor_{np.dtype(vdt).name}.npz"), **pack(sel))
    # error rows: zero pivots, indefinite pivots, wrong-side entries, singular triangles
    errs = {}
    def err_row(fn):
        try:
            fn()
        except sp.errors.SparseOpsError as exc:
            return type(exc).__name__, int(getattr(exc, "row", -1))
        return None, -1
    z2 = np.array([[0.0, 1.0], [1.0, 0.0]])
    errs["ilu_zero_pivot"] = err_row(lambda: sp.ilu0_factorize(sp.csr_from_dense(REF, z2, keep_zeros=True)))
    late = np.eye(5) * 2.0
    late[3, 3] = 0.0
    errs["ilu_zero_pivot_row3"] = err_row(lambda: sp.ilu0_factorize(sp.csr_from_dense(REF, late, keep_zeros=True)))
    errs["ic_indefinite"] = err_row(lambda: sp.ic0_factorize(sp.csr_from_dense(REF, np.diag([1.0, 4.0, -1.0, 2.0]))))
    upper = np.triu(np.ones((4, 4)))
    errs["lower_not_triangular"] = err_row(lambda: sp.solve_lower_tri(
        sp.csr_from_dense(REF, upper), vec(np.ones(4), np.float64), sp.dense_create(REF, 4, 1, sp.Precision.double, 0.0)))
    def tri(lower, zero_at):  # triangle of ones with an explicit zero on one diagonal slot
        t = [(i, j, 0.0 if (i == j == zero_at) else 1.0) for i in range(4) for j in range(4)
             if (j <= i if lower else j >= i)]
        return sp.csr_from_coo(sp.coo_from_triplets(REF, 4, 4, t))
    errs["lower_singular"] = err_row(lambda: sp.solve_lower_tri(
        tri(True, 2), vec(np.ones(4), np.float64), sp.dense_create(REF, 4, 1, sp.Precision.double, 0.0)))
    errs["upper_not_triangular"] = err_row(lambda: sp.solve_upper_tri(
        sp.csr_from_dense(REF, np.tril(np.ones((4, 4)))), vec(np.ones(4), np.float64),
        sp.dense_create(REF, 4, 1, sp.Precision.double, 0.0)))
    errs["upper_singular"] = err_row(lambda: sp.solve_upper_tri(
        tri(False, 1), vec(np.ones(4), np.float64), sp.dense_create(REF, 4, 1, sp.Precision.double, 0.0)))
    # preconditioned solver runs
    runs = {}
    n2, r2, c2, v2 = fixtures.poisson2d_triplets(16)
    a = ref_csr(n2, n2, r2, c2, v2)
    for name, cls, pre, crit, kw in (
            ("gmres30_ilu_poisson2d_16", "Gmres", "ilu", [sp.Iteration(1000), sp.ResidualNorm(1e-6)], {"krylov_dim": 30}),
            ("gmres10_ilu_convdiff3d_8", "Gmres", "ilu", [sp.Iteration(1000), sp.ResidualNorm(1e-8)], {"krylov_dim": 10}),
            ("cg_ic_poisson2d_16", "Cg", "ic", [sp.Iteration(1000), sp.ResidualNorm(1e-8)], {}),
            ("cg_ilu_poisson3d_8", "Cg", "ilu", [sp.Iteration(1000), sp.ResidualNorm(1e-8)], {})):
        if "convdiff" in name:
            n, ri, ci, v = fixtures.stencil3d_triplets(8, 0.5)
            m_ = ref_csr(n, n, ri, ci, v)
            src = ("stencil3d", 8, 0.5)
        elif "poisson3d" in name:
            n, ri, ci, v = fixtures.stencil3d_triplets(8, 0.0)
            m_ = ref_csr(n, n, ri, ci, v)
            src = ("stencil3d", 8, 0.0)
        else:
            m_, n, src = a, n2, ("poisson2d", 16, 0.0)
        prec = sp.ilu0_factorize(m_) if pre == "ilu" else sp.ic0_factorize(m_)
        b = sp.dense_create(REF, n, 1, sp.Precision.double, 1.0)
        x = sp.dense_create(REF, n, 1, sp.Precision.double, 0.0)
        log = getattr(sp, cls)(m_, criteria=crit, preconditioner=prec, **kw).solve(b, x)
        runs[name] = dict(source=list(src), solver=cls.lower(), precond=pre,
                          max_iters=1000, reduction_factor=crit[1].reduction_factor,
                          krylov_dim=kw.get("krylov_dim"), iterations=log.iterations,
                          converged=log.converged, stop_reason=log.stop_reason,
                          history=list(map(float, log.residual_history)))
    with open(os.path.join(HERE, "factor.json"), "w") as fh:
        json.dump({"cases": meta, "errors": errs, "solver_runs": runs}, fh, indent=1, sort_keys=True)


def _mmio_corpus():
    """Matrix Market inputs: the bodies of the reference's own tests/test_mmio.py:26-191
    plus the cases its parser distinguishes (explicit zeros in array bodies, several values
    per line, non-integral / out-of-range indices, non-square symmetric shapes, ragged
    lines, duplicates created by symmetry expansion) and a few larger random files."""
    H = "%%MatrixMarket matrix "
    cases = [
        # (name, text, format, precision, index width)
        ("basic", H + "coordinate real general\n2 2 2\n1 1 1.0\n2 2 3.0\n", "Csr"),
        ("coo_target", H + "coordinate real general\n2 2 1\n2 1 -4.5\n", "Coo"),
        ("symmetric", H + "coordinate real symmetric\n2 2 3\n1 1 2.0\n2 1 -1.0\n2 2 2.0\n", "Csr"),
        ("symmetric_offdiag_only", H + "coordinate real symmetric\n2 2 2\n1 1 2.0\n2 1 -1.0\n", "Csr"),
        ("skew", H + "coordinate real skew-symmetric\n2 2 1\n2 1 5.0\n", "Csr"),
        ("banner_case", "%%matrixmarket MATRIX Coordinate Real General\n1 1 1\n1 1 2.0\n", "Csr"),
        ("bad_banner", "%%Matrix matrix coordinate real general\n1 1 0\n", "Csr"),
        ("comments_blank", H + "coordinate real general\n% a comment\n\n2 2 2\n% another\n1 1 1.5\n\n2 2 2.5\n", "Csr"),
        ("pattern", H + "coordinate pattern general\n2 2 2\n1 2\n2 1\n", "Csr"),
        ("integer_f32", H + "coordinate integer general\n1 2 2\n1 1 3\n1 2 -7\n", "Csr", "single"),
        ("complex", H + "coordinate complex general\n1 1 1\n1 1 1.0 0.0\n", "Csr"),
        ("count_mismatch", H + "coordinate real general\n2 2 3\n1 1 1.0\n", "Csr"),
        ("index_oob", H + "coordinate real general\n2 2 1\n3 1 1.0\n", "Csr"),
        ("index_zero", H + "coordinate real general\n2 2 1\n0 1 1.0\n", "Csr"),
        ("bad_size", H + "coordinate real general\n2 2\n", "Csr"),
        ("duplicates", H + "coordinate real general\n2 2 2\n1 1 1.0\n1 1 2.0\n", "Csr"),
        ("array", H + "array real general\n2 2\n1.0\n2.0\n3.0\n4.0\n", "Csr"),
        ("array_symmetric", H + "array real symmetric\n2 2\n1.0\n2.0\n3.0\n", "Csr"),
        ("garbage_entry", H + "coordinate real general\n1 1 1\n1 1 abc\n", "Csr"),
        # beyond test_mmio.py: what the parser decides that changes the canonical arrays
        ("array_zeros", H + "array real general\n3 3\n1\n0\n0\n0\n2\n0\n5\n0\n3\n", "Csr"),
        ("array_zeros_coo", H + "array real general\n2 3\n0\n1\n0\n0\n2\n0\n", "Coo"),
        ("array_multi_per_line", H + "array real general\n2 2\n1.0 0.0\n3.0 4.0\n", "Csr"),
        ("array_symmetric_zeros", H + "array real symmetric\n3 3\n4\n0\n-1\n4\n0\n4\n", "Csr"),
        ("array_skew", H + "array real skew-symmetric\n3 3\n1\n2\n3\n", "Csr"),
        ("array_integer", H + "array integer general\n1 3\n7\n-2\n0\n", "Csr"),
        ("array_count", H + "array real general\n2 2\n1\n2\n3\n", "Csr"),
        ("array_bad_token", H + "array real general\n1 2\n1\nx\n", "Csr"),
        ("array_pattern", H + "array pattern general\n1 1\n1\n", "Csr"),
        ("array_empty", H + "array real general\n0 0\n", "Csr"),
        ("coord_explicit_zero", H + "coordinate real general\n2 3 3\n1 1 0.0\n2 3 1.5\n1 2 0\n", "Csr"),
        ("coord_unsorted", H + "coordinate real general\n3 3 4\n3 1 1\n1 3 2\n2 2 3\n1 1 4\n", "Coo"),
        ("coord_inline_comment", H + "coordinate real general\n2 2 1\n1 2 7.5 % note\n", "Csr"),
        ("coord_float_index", H + "coordinate real general\n2 2 1\n1e0 2.0 7.5\n", "Csr"),
        ("coord_nonintegral", H + "coordinate real general\n2 2 1\n1.5 1 1.0\n", "Csr"),
        ("coord_ragged", H + "coordinate real general\n2 2 2\n1 1 1.0\n2 2\n", "Csr"),
        ("coord_pattern_3cols", H + "coordinate pattern general\n2 2 1\n1 1 1.0\n", "Csr"),
        ("coord_real_2cols", H + "coordinate real general\n2 2 1\n1 1\n", "Csr"),
        ("coord_empty_body", H + "coordinate real general\n4 5 0\n", "Csr"),
        ("coord_empty_but_declared", H + "coordinate real general\n4 5 1\n", "Csr"),
        ("sym_nonsquare", H + "coordinate real symmetric\n2 3 1\n1 1 1.0\n", "Csr"),
        ("array_sym_nonsquare", H + "array real symmetric\n2 3\n1\n2\n3\n", "Csr"),
        ("sym_mirror_duplicate", H + "coordinate real symmetric\n2 2 2\n2 1 1.0\n1 2 2.0\n", "Csr"),
        ("skew_diagonal", H + "coordinate real skew-symmetric\n2 2 2\n1 1 3.0\n2 1 1.0\n", "Coo"),
        ("negative_size", H + "coordinate real general\n-2 2 0\n", "Csr"),
        ("float_size", H + "coordinate real general\n2.0 2 0\n", "Csr"),
        ("four_tokens", "%%MatrixMarket matrix coordinate real\n1 1 0\n", "Csr"),
        ("field_double", H + "coordinate double general\n1 1 1\n1 1 1.0\n", "Csr"),
        ("bad_symmetry", H + "coordinate real hermitian\n1 1 1\n1 1 1.0\n", "Csr"),
        ("bad_object", "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1.0\n", "Csr"),
        ("empty_file", "", "Csr"),
        ("missing_size", H + "coordinate real general\n% only a comment\n", "Csr"),
        ("bad_target", H + "coordinate real general\n1 1 1\n1 1 1.0\n", "Ell"),
        ("i64", H + "coordinate real general\n3 3 3\n3 3 1\n1 2 2\n2 1 3\n", "Csr", "double", "i64"),
        ("f32_rounding", H + "coordinate real general\n1 2 2\n1 1 0.1\n1 2 3.4028235677973366e+38\n", "Coo", "single"),
    ]
    rng = np.random.default_rng(31)
    # larger random files: coordinate general with duplicates and zeros, symmetric, array
    n = 200
    r = rng.integers(1, n + 1, 1500); c = rng.integers(1, n + 1, 1500)
    v = rng.standard_normal(1500); v[rng.random(1500) < 0.05] = 0.0
    body = "".join("%d %d %.17g\n" % t for t in zip(r, c, v))
    cases.append(("random_general_dups", H + f"coordinate real general\n{n} {n} 1500\n" + body, "Csr"))
    lo = r >= c
    body = "".join("%d %d %.17g\n" % t for t in zip(r[lo], c[lo], v[lo]))
    cases.append(("random_symmetric", H + f"coordinate real symmetric\n{n} {n} {int(lo.sum())}\n" + body, "Csr"))
    st = r > c
    body = "".join("%d %d %.17g\n" % t for t in zip(r[st], c[st], v[st]))
    cases.append(("random_skew_coo", H + f"coordinate real skew-symmetric\n{n} {n} {int(st.sum())}\n" + body, "Coo"))
    a = rng.standard_normal((20, 30)); a[rng.random((20, 30)) < 0.3] = 0.0
    body = "".join("%.17g\n" % t for t in a.T.ravel())
    cases.append(("random_array", H + "array real general\n20 30\n" + body, "Csr"))
    s_ = rng.standard_normal((25, 25)); s_[rng.random((25, 25)) < 0.4] = 0.0
    body = "".join("%.17g\n" % s_[i, j] for j in range(25) for i in range(j, 25))
    cases.append(("random_array_symmetric", H + "array real symmetric\n25 25\n" + body, "Csr", "single"))
    return cases


def mmio_corpus():
    """Run the reference reader on every corpus file; record canonical arrays, warnings
    and error classes (tests/golden/mmio_corpus.json)."""
    import tempfile
    import warnings as _w
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        for case in _mmio_corpus():
            name, text, fmt = case[:3]
            prec = case[3] if len(case) > 3 else "double"
            width = case[4] if len(case) > 4 else "i32"
            path = os.path.join(tmp, name + ".mtx")
            with open(path, "w") as fh:
                fh.write(text)
            rec = dict(name=name, text=text, format=fmt, precision=prec, index_width=width)
            with _w.catch_warnings(record=True) as caught:
                _w.simplefilter("always")
                try:
                    m = sp.read_matrix_market(REF, path, getattr(sp.Precision, prec), fmt,
                                              getattr(sp.IndexWidth, width))
                except Exception as exc:  # noqa: BLE001 -- the class name IS the golden
                    rec["error"] = type(exc).__name__
                else:
                    rec["type"] = type(m).__name__
                    rec["shape"] = [m.rows, m.cols]
                    if isinstance(m, sp.CsrMatrix):
                        rec["row_ptrs"] = m.row_ptrs.tolist()
                    else:
                        rec["row_idxs"] = m.row_idxs.tolist()
                    rec["col_idxs"] = m.col_idxs.tolist()
                    rec["values_hex"] = [float(x).hex() for x in m.values.astype(np.float64)]
                    rec["dtype"] = str(m.values.dtype)
                    rec["index_dtype"] = str(m.col_idxs.dtype)
            rec["warnings"] = sorted({type(w.message).__name__ for w in caught
                                      if issubclass(w.category, UserWarning)})
            out.append(rec)
        # writer: exact text for the reference's own cases and a round trip
        wr = {}
        m = sp.csr_from_dense(REF, np.array([[1.0, 0.0], [0.0, 3.0]]))
        sp.write_matrix_market(m, os.path.join(tmp, "w1.mtx"))
        wr["dense2"] = open(os.path.join(tmp, "w1.mtx")).read()
        awkward = [0.1, 1.0 / 3.0, np.pi, 1e-300, 1e300, -2.2250738585072014e-308]
        m = sp.coo_from_triplets(REF, 6, 1, [(i, 0, v) for i, v in enumerate(awkward)])
        sp.write_matrix_market(m, os.path.join(tmp, "w2.mtx"))
        wr["awkward"] = open(os.path.join(tmp, "w2.mtx")).read()
        m = sp.coo_from_triplets(REF, 3, 3, [])
        sp.write_matrix_market(m, os.path.join(tmp, "w3.mtx"))
        wr["empty"] = open(os.path.join(tmp, "w3.mtx")).read()
        m = sp.csr_from_coo(sp.coo_from_triplets(REF, 2, 2, [(0, 1, 0.5), (1, 0, 0.25)],
                                                  sp.Precision.single))
        sp.write_matrix_market(m, os.path.join(tmp, "w4.mtx"))
        wr["single"] = open(os.path.join(tmp, "w4.mtx")).read()
    with open(os.path.join(HERE, "mmio_corpus.json"), "w") as fh:
        json.dump({"source": "reference sparseops.mmio (pkg/src/sparseops/mmio.py), "
                             "generated by tests/golden/make_golden.py mmio_corpus",
                   "cases": out, "writer": wr}, fh, indent=0)


def parity_matrix():
    """Reference runs for the solver x preconditioner parity matrix (pkg/tests/
    test_config.py:237-273: {Cg, Cgs, Gmres} x {None, Jacobi, Ilu, Ic} on laplacian_2d(8),
    b = 1, [Iteration(1000), ResidualNorm(1e-6)]), the same on a nonsymmetric 3-D
    convection-diffusion operator, generic LinOp preconditioners / operators (a solver
    as a preconditioner, a dense operator) and GMRES trace events
    (pkg/tests/test_acceptance.py:149-173)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from helpers import random_spd_csr  # noqa: E402  (the reference's own generator)

    out, meta = {}, {}

    def run(name, a, bvec, cls, precond, crit, dim=None, arrays=True):
        n = a.rows
        b = vec(bvec, np.float64)
        x = sp.dense_create(REF, n, 1, sp.Precision.double, 0.0)
        kw = {"krylov_dim": dim} if dim else {}
        log = getattr(sp, cls)(a, criteria=crit, preconditioner=precond, **kw).solve(b, x)
        meta[name] = dict(solver=cls, iterations=log.iterations, converged=log.converged,
                          stop_reason=log.stop_reason)
        out[f"{name}_history"] = np.asarray(log.residual_history, np.float64)
        out[f"{name}_x"] = x.values.copy()

    crit = [sp.Iteration(1000), sp.ResidualNorm(1e-6)]
    n, ri, ci, v = fixtures.poisson2d_triplets(8)
    lap = ref_csr(n, n, ri, ci, v)
    p3, ri, ci, v = fixtures.stencil3d_triplets(10, 0.5)
    cd = ref_csr(p3, p3, ri, ci, v)
    makers = {"none": lambda a: None, "jacobi": sp.jacobi_create, "ilu": sp.ilu0_factorize,
              "ic": sp.ic0_factorize}
    for cls in ("Cg", "Cgs", "Gmres"):
        for pname, make in makers.items():
            run(f"lap8_{cls.lower()}_{pname}", lap, np.ones(n), cls, make(lap), crit,
                30 if cls == "Gmres" else None)
    for cls in ("Cgs", "Gmres"):
        for pname in ("jacobi", "ilu"):
            run(f"convdiff10_{cls.lower()}_{pname}", cd, np.ones(p3), cls, makers[pname](cd),
                [sp.Iteration(1000), sp.ResidualNorm(1e-8)], 30 if cls == "Gmres" else None)
    # a solver as the preconditioner (LinOp composition, solvers.py:172-176)
    n16, ri, ci, v = fixtures.poisson2d_triplets(16)
    lap16 = ref_csr(n16, n16, ri, ci, v)
    inner = sp.Cg(lap16, criteria=[sp.Iteration(8)], preconditioner=sp.jacobi_create(lap16))
    run("lap16_gmres10_innercg8", lap16, np.ones(n16), "Gmres", inner,
        [sp.Iteration(300), sp.ResidualNorm(1e-6)], 10)
    # a dense operator (the reference registers DenseMatrix as a LinOp, linop.py:78)
    dense = sp.dense_from_array(REF, lap.to_dense())
    run("lap8dense_cg_none", dense, np.ones(n), "Cg", None, crit)
    # GMRES trace events (test_acceptance.py:149-173)
    problems = [("trace_lap8", lap, np.random.default_rng(31).standard_normal(n), 5),
                ("trace_spd50", random_spd_csr(REF, np.random.default_rng(32), 50), np.ones(50), 7)]
    for name, a, bvec, dim in problems:
        events = []
        x = sp.dense_create(REF, a.rows, 1, sp.Precision.double, 0.0)
        log, _ = sp.gmres_solve(a, vec(bvec, np.float64), x, sp.SolverParams(400, 1e-9, krylov_dim=dim),
                                trace=events.append)
        meta[name] = dict(solver="Gmres", iterations=log.iterations, converged=log.converged,
                          stop_reason=log.stop_reason, krylov_dim=dim,
                          cycles=[e.cycle for e in events], inner=[e.inner for e in events])
        out[f"{name}_rp"], out[f"{name}_ci"], out[f"{name}_v"] = a.row_ptrs, a.col_idxs, a.values
        out[f"{name}_b"] = bvec
        out[f"{name}_estimates"] = np.array([e.estimate for e in events])
        out[f"{name}_solutions"] = np.stack([e.solution for e in events])
    np.savez_compressed(os.path.join(HERE, "parity_matrix.npz"), **out)
    meta["_source"] = "reference sparseops run by tests/golden/make_golden.py parity_matrix"
    with open(os.path.join(HERE, "parity_matrix.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def large_pins(which):
    """Config #4 pin: run the REFERENCE GMRES(30) + Jacobi on the
    256^3 convection-diffusion operator (c = 0.5), b = 1, x0 = 0, rtol 1e-8, on the
    reference's own single-thread device, and record iterations / stop reason / history.
    Slow (~40 min); run with ``python tests/golden/make_golden.py large <name>``."""
    import time
    path = os.path.join(HERE, "reference_large.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    specs = {
        "gmres30_jacobi_convdiff3d_256": (256, 0.5, "Gmres", 5000, 30),
        "gmres30_jacobi_convdiff3d_128": (128, 0.5, "Gmres", 5000, 30),
        "cg_jacobi_poisson3d_256": (256, 0.0, "Cg", 100000, None),
    }
    for name in which:
        p, c, cls, max_iters, dim = specs[name]
        n, ri, ci, v = fixtures.stencil3d_triplets(p, c)
        t0 = time.time()
        a = ref_csr(n, n, ri, ci, v)
        del ri, ci, v
        m = sp.jacobi_create(a)
        t1 = time.time()
        b = sp.dense_create(REF, n, 1, sp.Precision.double, 1.0)
        x = sp.dense_create(REF, n, 1, sp.Precision.double, 0.0)
        kw = {"krylov_dim": dim} if dim else {}
        crit = [sp.Iteration(max_iters), sp.ResidualNorm(1e-8)]
        log = getattr(sp, cls)(a, criteria=crit, preconditioner=m, **kw).solve(b, x)
        t2 = time.time()
        data[name] = dict(p=p, c=c, solver=cls.lower(), krylov_dim=dim, max_iters=max_iters,
                          reduction_factor=1e-8, device="reference (1 thread)",
                          iterations=log.iterations, converged=log.converged,
                          stop_reason=log.stop_reason,
                          final_estimate=float(log.residual_history[-1]),
                          history_head=list(map(float, log.residual_history[:5])),
                          setup_s=round(t1 - t0, 1), solve_s=round(t2 - t1, 1))
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
        print(name, data[name]["iterations"], data[name]["solve_s"], flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "large":
        large_pins(sys.argv[2:])
        sys.exit(0)
    if len(sys.argv) > 1:
        globals()[sys.argv[1]]()
        sys.exit(0)
    spmv_suite()
    canonicalization()
    stencils_and_jacobi()
    blas1()
    solver_goldens()
    factorizations()
    mmio_corpus()
    print("golden fixtures written to", HERE)
