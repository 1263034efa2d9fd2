"""GPU parity: the device Krylov solvers against the reference.

Bar (north_star): iteration counts within +-2% of the reference, same stop reason,
recurrence residual below the tolerance; the true residual is reported beside it.
The only numerical difference from the reference is the order of the fp64 dot sums,
so histories agree to ~1e-10 relative in the early iterations.
"""

import numpy as np
import pytest

from oracle import fixtures, sbref
from paper_2510_08230_b200 import gen
from paper_2510_08230_b200 import sparseops as sp
from tests import golden_io
from tests.gpu_util import csr, host, out, vec

pytestmark = pytest.mark.gpu

SOLVERS = {"cg": sp.Cg, "cgs": sp.Cgs, "gmres": sp.Gmres, "bicgstab": sp.Bicgstab}


def within(n, ref, pct=0.02):
    return abs(n - ref) <= max(1, int(np.ceil(pct * ref)))


ENVELOPE_THREADS = (1, 2, 3, 4, 5, 6, 7, 8, 12, 16)


def oracle_envelope(kind, a, b, precond=True, **kw):
    """Iteration counts of the oracle restatement of the reference when only the dot
    summation order changes (its thread count): CGS and BiCGSTAB are sensitive enough
    that the reference's own algorithm spreads over several iterations."""
    rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
    inv = sbref.jacobi_create(rp, ci, v)[0] if precond else None
    its = [sbref.solve(kind, rp, ci, v, b, inv_diag=inv, threads=t, **kw)[0].iterations
           for t in ENVELOPE_THREADS]
    return min(its), max(its)


def within_envelope(n, env, pct=0.02):
    lo, hi = env
    return lo - max(1, int(np.ceil(pct * lo))) <= n <= hi + max(1, int(np.ceil(pct * hi)))


def true_residual(rp, ci, v, b, x):
    r = b.astype(np.float64) - sbref.csr_spmv(rp, ci, v.astype(np.float64), x.astype(np.float64))
    return np.linalg.norm(r) / max(np.linalg.norm(b), 1e-300)


def solve(dev, kind, a, bvec, criteria, precond=True, x0=None, **kw):
    if precond is True:
        m = sp.jacobi_create(a)
    else:
        m = precond or None
    b = vec(dev, bvec)
    x = vec(dev, np.zeros(a.rows, bvec.dtype) if x0 is None else x0)
    log = SOLVERS[kind](a, criteria=criteria, preconditioner=m, **kw).solve(b, x)
    return log, host(x), b


def test_reference_solver_goldens(dev):
    """Every reference run recorded in tests/golden/solvers.json."""
    meta = golden_io.solver_meta()
    g = golden_io.load("solvers.npz")
    for name, m in meta.items():
        if name.startswith("_"):
            continue
        dt = np.dtype(m["dtype"])
        a = gen.stencil_csr(dev, m["p"], dim=3, c=m["c"], precision=sp.Precision.from_dtype(dt))
        crit = [sp.Iteration(m["max_iters"])] + (
            [sp.ResidualNorm(m["reduction_factor"])] if m["reduction_factor"] else [])
        kw = {"krylov_dim": m["krylov_dim"]} if m["solver"] == "gmres" else {}
        log, x, _ = solve(dev, m["solver"], a, np.ones(a.rows, dt), crit, **kw)
        assert log.stop_reason == m["stop_reason"], name
        assert log.converged == m["converged"], name
        if m["stop_reason"] == "max_iters":
            assert log.iterations == m["iterations"], name
        else:
            assert within(log.iterations, m["iterations"]), (name, log.iterations, m["iterations"])
        hist = np.asarray(log.residual_history)
        ref = g[f"{name}_history"]
        k = min(10, len(ref), len(hist))
        np.testing.assert_allclose(hist[:k], ref[:k], rtol=1e-6 if dt == np.float32 else 1e-9,
                                   err_msg=name)
        xref = g[f"{name}_x"]
        rel = np.abs(x.astype(np.float64) - xref).max() / np.abs(xref).max()
        assert rel <= (1e-3 if dt == np.float32 else 1e-6), (name, rel)


@pytest.mark.parametrize("p,iters", [(64, 159), (128, 319)])
def test_cg_poisson_config2_iteration_parity(dev, p, iters):
    """Config #2 (and 64^3): Jacobi-CG, b = 1, x0 = 0, rtol 1e-8 -> the reference's
    iteration count (SURVEY.md §8c golden, 319 at 128^3) within +-2%."""
    a = gen.poisson3d(dev, p)
    log, x, _ = solve(dev, "cg", a, np.ones(a.rows), [sp.Iteration(100000), sp.ResidualNorm(1e-8)])
    assert log.converged and within(log.iterations, iters), log.iterations
    assert log.residual_history[-1] <= 1e-8 * np.sqrt(a.rows)
    rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
    assert true_residual(rp, ci, v, np.ones(a.rows), x) <= 2e-8


def test_gmres_convdiff_64(dev):
    a = gen.convdiff3d(dev, 64)
    log, x, _ = solve(dev, "gmres", a, np.ones(a.rows), [sp.Iteration(5000), sp.ResidualNorm(1e-8)],
                      krylov_dim=30)
    assert log.converged and within(log.iterations, 330), log.iterations


@pytest.mark.parametrize("p", [16, 32])
def test_bicgstab_against_oracle(dev, p):
    """BiCGSTAB has no reference implementation: parity with the oracle restatement."""
    for c in (0.0, 0.5):
        a = gen.stencil_csr(dev, p, dim=3, c=c)
        rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
        inv, _ = sbref.jacobi_create(rp, ci, v)
        ref, xref = sbref.solve("bicgstab", rp, ci, v, np.ones(a.rows), inv_diag=inv,
                                max_iters=5000, reduction_factor=1e-8)
        env = oracle_envelope("bicgstab", a, np.ones(a.rows), max_iters=5000,
                              reduction_factor=1e-8)
        log, x, _ = solve(dev, "bicgstab", a, np.ones(a.rows),
                          [sp.Iteration(5000), sp.ResidualNorm(1e-8)])
        assert log.converged and ref.converged
        assert within_envelope(log.iterations, env), (log.iterations, env)
        np.testing.assert_allclose(log.residual_history[:5], ref.residual_history[:5], rtol=1e-9)
        assert true_residual(rp, ci, v, np.ones(a.rows), x) <= 1e-7


@pytest.mark.parametrize("kind", ["cg", "cgs", "gmres", "bicgstab"])
def test_every_format_same_iterations(dev, kind):
    """One problem, every storage format and CSR kernel: each run's iteration count lies
    in the reference algorithm's reduction-order envelope (+-2%)."""
    c = 0.0 if kind == "cg" else 0.5
    a = gen.stencil_csr(dev, 20, dim=3, c=c)
    crit = [sp.Iteration(3000), sp.ResidualNorm(1e-8)]
    env = oracle_envelope(kind, a, np.ones(a.rows), max_iters=3000, reduction_factor=1e-8)
    m = sp.jacobi_create(a)
    base, _, _ = solve(dev, kind, a, np.ones(a.rows), crit, precond=m)
    assert base.converged and within_envelope(base.iterations, env), (base.iterations, env)
    mats = [a.with_kernel("strict"), a.with_kernel("vector"), a.with_kernel("merge"),
            a.with_kernel("tile"), sp.coo_from_csr(a), sp.coo_from_csr(a).with_kernel("segmented"),
            sp.ell_from_csr(a), sp.sellp_from_csr(a), sp.sellp_from_csr(a, 32, sigma=256),
            sp.hybrid_from_csr(a, 5)]
    for mat in mats:
        log, _, _ = solve(dev, kind, mat, np.ones(a.rows), crit, precond=m)
        assert log.converged and within_envelope(log.iterations, env), \
            (repr(mat), log.iterations, env)
    # the polled (non-graph) loop gives the identical run
    from paper_2510_08230_b200 import _lib
    _lib.fn("sb_set_graph_mode")(0)
    try:
        polled, _, _ = solve(dev, kind, a, np.ones(a.rows), crit, precond=m)
    finally:
        _lib.fn("sb_set_graph_mode")(1)
    assert polled.iterations == base.iterations
    assert polled.residual_history == base.residual_history


def test_semantics(dev):
    """test_solvers.py:79-145 behaviours on the device."""
    one = sp.csr_from_dense(dev, np.eye(4))
    log, x, _ = solve(dev, "cg", one, np.ones(4), [sp.Iteration(1000), sp.ResidualNorm(1e-6)],
                      precond=False)
    assert log.iterations == 1 and log.converged and log.residual_history[-1] == 0.0
    np.testing.assert_allclose(x, 1.0)
    zero = sp.csr_from_dense(dev, np.zeros((2, 2)), keep_zeros=False)
    with pytest.raises(sp.errors.BreakdownError) as exc:
        solve(dev, "cg", zero, np.array([1.0, 2.0]), [sp.Iteration(10)], precond=False)
    assert exc.value.iteration == 1
    with pytest.raises(sp.errors.BreakdownError) as exc:
        solve(dev, "cgs", zero, np.array([1.0, 2.0]), [sp.Iteration(10)], precond=False)
    assert exc.value.iteration == 1
    d = sp.csr_from_dense(dev, np.diag([2.0, 4.0]))
    for kind in SOLVERS:
        log, _, _ = solve(dev, kind, d, np.array([2.0, 4.0]), [sp.Iteration(10), sp.ResidualNorm(1e-6)],
                          precond=False, x0=np.array([1.0, 1.0]))
        assert log.iterations == 0 and log.converged and log.residual_history == [0.0], kind
    # fixed-iteration mode runs exactly max_iters (test_solvers.py:296-313)
    a = gen.poisson3d(dev, 8)
    for kind in SOLVERS:
        log, _, _ = solve(dev, kind, a, np.ones(a.rows), [sp.Iteration(7)], krylov_dim=3) \
            if kind == "gmres" else solve(dev, kind, a, np.ones(a.rows), [sp.Iteration(7)])
        assert log.iterations == 7 and log.stop_reason == "max_iters", kind
        assert len(log.residual_history) == 7
    # b untouched, x overwritten
    bv = np.random.default_rng(2).random(a.rows)
    b = vec(dev, bv)
    x = vec(dev, np.full(a.rows, 0.5))
    sp.Cg(a, criteria=[sp.Iteration(100), sp.ResidualNorm(1e-10)]).solve(b, x)
    np.testing.assert_array_equal(host(b), bv)


def test_fp32_cg(dev):
    a = gen.poisson3d(dev, 16, precision=sp.Precision.single)
    log, x, _ = solve(dev, "cg", a, np.ones(a.rows, np.float32),
                      [sp.Iteration(1000), sp.ResidualNorm(1e-5)])
    assert log.converged and within(log.iterations, 28)


def test_config_solve_listing2(dev):
    tree = {"type": "solver::Gmres", "krylov_dim": 30,
            "preconditioner": {"type": "preconditioner::Jacobi"},
            "criteria": [{"type": "Iteration", "max_iters": 1000},
                         {"type": "ResidualNorm", "reduction_factor": 1e-8}]}
    a = gen.convdiff3d(dev, 16)
    b = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 1.0)
    x = sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0)
    log, res = sp.config_solve(tree, dev, a, b, x)
    assert res is x and log.converged and within(log.iterations, 81)
    tree["type"] = "solver::Bicgstab"
    del tree["krylov_dim"]
    log, _ = sp.config_solve(tree, dev, a, b, sp.dense_create(dev, a.rows, 1, sp.Precision.double, 0.0))
    assert log.converged


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cg_fused_direction_bitwise(dev, dtype):
    """The two-kernel CG loop (search direction evaluated inside the SpMV gather, x update
    deferred to the next SpMV) reproduces the three-kernel loop bit for bit: same
    iterations, residual history and solution, for every row-owning format and kernel,
    odd and even final iterations, max_iters stops, x0 != 0, and without a
    preconditioner; also in the polled (non-graph) loop."""
    from paper_2510_08230_b200 import _lib
    prec = sp.Precision.from_dtype(np.dtype(dtype))
    a = gen.stencil_csr(dev, 18, dim=3, precision=prec)
    rng = np.random.default_rng(5)
    b = rng.random(a.rows).astype(dtype)
    x0 = rng.random(a.rows).astype(dtype)
    mats = [a, a.with_kernel("strict"), a.with_kernel("vector"), sp.ell_from_csr(a),
            sp.sellp_from_csr(a), sp.coo_from_csr(a)]
    cases = [([sp.Iteration(2000), sp.ResidualNorm(1e-7)], True, None),
             ([sp.Iteration(7)], True, x0),             # odd max_iters stop
             ([sp.Iteration(8)], False, None),          # even, identity preconditioner
             ([sp.Iteration(2000), sp.ResidualNorm(1e-6)], False, x0)]
    fn_fused, fn_graph = _lib.fn("sb_set_cg_fused"), _lib.fn("sb_set_graph_mode")
    try:
        for crit, pre, xi in cases:
            runs = []
            for fused, graph in ((0, 1), (1, 1), (1, 0), (0, 0)):
                fn_fused(fused)
                fn_graph(graph)
                for k, mat in enumerate(mats):
                    log, x, _ = solve(dev, "cg", mat, b, crit, precond=sp.jacobi_create(a) if pre else False,
                                      x0=xi)
                    runs.append((k, fused, graph, log, x))
            for name, fused, graph, log, x in runs[len(mats):]:
                ref = runs[name]  # same matrix / kernel, three-kernel graph loop
                assert log.iterations == ref[3].iterations, (name, fused, graph)
                assert log.residual_history == ref[3].residual_history, (name, fused, graph)
                np.testing.assert_array_equal(x, ref[4], err_msg=f"{name} fused={fused} graph={graph}")
    finally:
        fn_fused(3)
        fn_graph(1)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cg_persistent_kernel(dev, dtype):
    """The single-launch persistent CG (CSR stream matrices) against the graph loop and the
    oracle: same iteration counts and stop reasons, residual histories equal up to the
    dot-product summation order, same solutions to rounding; odd / even max_iters stops,
    x0 != 0, identity preconditioner, breakdown and exact-solution exits."""
    from paper_2510_08230_b200 import _lib
    prec = sp.Precision.from_dtype(np.dtype(dtype))
    a = gen.stencil_csr(dev, 24, dim=3, precision=prec)
    rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
    rng = np.random.default_rng(9)
    b = rng.random(a.rows).astype(dtype)
    x0 = rng.random(a.rows).astype(dtype)
    inv = sbref.jacobi_create(rp, ci, v)[0]
    rtol = 1e-9 if dtype == np.float64 else 1e-4
    set_mode = _lib.fn("sb_set_cg_fused")
    set_sync = _lib.fn("sb_set_cg_sync")
    try:
        for crit, pre, xi, its, rf in (([sp.Iteration(5000), sp.ResidualNorm(1e-7)], True, None, 5000, 1e-7),
                                       ([sp.Iteration(7)], True, x0, 7, None),
                                       ([sp.Iteration(8)], False, x0, 8, None),
                                       ([sp.Iteration(5000), sp.ResidualNorm(1e-6)], False, None, 5000, 1e-6)):
            logs = {}
            for mode in (1, 3, 4):  # 3: two-barrier persistent kernel, 4: single-sync kernel
                set_mode(min(mode, 3))
                set_sync(1 if mode == 4 else 2)
                logs[mode] = solve(dev, "cg", a, b, crit, precond=sp.jacobi_create(a) if pre else False, x0=xi)
                assert _lib.fn("sb_cg_last_loop")() == min(mode, 3)
            set_sync(2)
            ref, xr = sbref.solve("cg", rp, ci, v, b, x0=xi, inv_diag=inv if pre else None, max_iters=its,
                                  reduction_factor=rf)
            l1, x1, _ = logs[1]
            for m3 in (3, 4):
                l3, x3, _ = logs[m3]
                assert l3.iterations == l1.iterations or (rf and within(l3.iterations, ref.iterations))
                assert l3.stop_reason == l1.stop_reason == ref.stop_reason
                n = min(5, len(ref.residual_history))
                np.testing.assert_allclose(l3.residual_history[:n], ref.residual_history[:n], rtol=rtol)
                if rf is None:
                    np.testing.assert_allclose(x3, x1, rtol=rtol * 10, atol=rtol)
                else:
                    assert l3.residual_history[-1] <= rf * np.linalg.norm(b.astype(np.float64)) * 1.0001
        set_mode(3)
        if dtype == np.float64:
            zero = sp.csr_from_dense(dev, np.zeros((300, 300)), keep_zeros=False).with_kernel("stream")
            with pytest.raises(sp.errors.BreakdownError) as exc:
                solve(dev, "cg", zero, np.ones(300), [sp.Iteration(10)], precond=False)
            assert exc.value.iteration == 1
        exact, _, _ = solve(dev, "cg", a, np.zeros(a.rows, dtype), [sp.Iteration(10), sp.ResidualNorm(1e-6)])
        assert exact.iterations == 0 and exact.converged
    finally:
        set_mode(3)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cg_persistent_x_update_in_barrier_waits(dev, dtype):
    """The persistent CG's x update deferred into the grid-barrier waits (sb_set_cg_xw(1),
    the default) changes only WHEN x += alpha p runs, not its per-element order or
    rounding: x and the residual history are bitwise those of the in-phase update, for
    converged, odd / even max_iters, x0 != 0 and breakdown exits."""
    from paper_2510_08230_b200 import _lib
    prec = sp.Precision.from_dtype(np.dtype(dtype))
    a = gen.stencil_csr(dev, 40, dim=3, precision=prec)
    rng = np.random.default_rng(11)
    b = rng.random(a.rows).astype(dtype)
    x0 = rng.random(a.rows).astype(dtype)
    set_xw = _lib.fn("sb_set_cg_xw")
    try:
        for crit, xi in (([sp.Iteration(5000), sp.ResidualNorm(1e-7)], None),
                         ([sp.Iteration(7)], x0), ([sp.Iteration(8)], x0),
                         ([sp.Iteration(5000), sp.ResidualNorm(1e-6)], x0)):
            out = {}
            for xw in (0, 1):
                set_xw(xw)
                out[xw] = solve(dev, "cg", a, b, crit, x0=xi)
                assert _lib.fn("sb_cg_last_loop")() == 3
            (l0, x0r, _), (l1, x1r, _) = out[0], out[1]
            assert l0.iterations == l1.iterations and l0.stop_reason == l1.stop_reason
            np.testing.assert_array_equal(np.asarray(l1.residual_history), np.asarray(l0.residual_history))
            np.testing.assert_array_equal(x1r, x0r)
    finally:
        set_xw(1)


@pytest.mark.parametrize("kind", ["cg", "cgs", "bicgstab", "gmres"])
def test_graph_cache_tracks_workspace_layout(dev, kind):
    """A captured solver loop is reused only for the same buffers: the workspace's vector
    offsets depend on the history capacity (max_iters), so two solves with the same
    pointers but different criteria must not share a graph (regression: a stale graph
    iterated on the previous solve's vector offsets when x0 != 0)."""
    a = gen.stencil_csr(dev, 16, dim=3)
    rng = np.random.default_rng(11)
    b, x0 = rng.random(a.rows), rng.random(a.rows)
    rp, ci, v = (t.cpu().numpy() for t in (a.row_ptrs, a.col_idxs, a.values))
    inv = sbref.jacobi_create(rp, ci, v)[0]
    kw = {"krylov_dim": 30} if kind == "gmres" else {}
    for crit, its in (([sp.Iteration(3000), sp.ResidualNorm(1e-8)], 3000), ([sp.Iteration(5)], 5),
                      ([sp.Iteration(40)], 40)):
        for _ in range(2):  # the second solve hits the graph cache with recycled buffers
            log, x, _ = solve(dev, kind, a, b, crit, x0=x0, **kw)
        ref, xr = sbref.solve(kind, rp, ci, v, b, x0=x0, inv_diag=inv, max_iters=its,
                              reduction_factor=1e-8 if its == 3000 else None, **kw)
        n = min(4, len(ref.residual_history))
        np.testing.assert_allclose(log.residual_history[:n], ref.residual_history[:n], rtol=1e-9,
                                   err_msg=f"{kind} max_iters={its}")
        if its < 3000:
            assert log.iterations == its


@pytest.mark.slow
def test_config4_bicgstab_converges(dev):
    """BASELINE config #4: BiCGSTAB + Jacobi on the 256^3 convection-diffusion system.  The
    recurrence's residual grows by ~20 orders of magnitude before it recovers, so only
    near-exact dots follow the exact-arithmetic trajectory: the device's compensated dots
    converge within the oracle's envelope (1045 with 8-chunk sequential sums, 1059 with
    compensated sums; tests/golden/oracle_probe_256.json)."""
    import json
    import os
    with open(os.path.join(golden_io.GOLDEN, "oracle_probe_256.json")) as fh:
        probe = json.load(fh)["config4_convdiff3d_256_c0.5_jacobi_rtol1e-8"]
    lo = min(probe["bicgstab"]["iterations"], probe["bicgstab_compensated_dots"]["iterations"])
    hi = max(probe["bicgstab"]["iterations"], probe["bicgstab_compensated_dots"]["iterations"])
    a = gen.convdiff3d(dev, 256)
    log, _, _ = solve(dev, "bicgstab", a, np.ones(a.rows), [sp.Iteration(5000), sp.ResidualNorm(1e-8)])
    assert log.converged and log.stop_reason == "residual"
    assert within_envelope(log.iterations, (lo, hi)), (log.iterations, lo, hi)


@pytest.mark.parametrize("kind", ["cg", "gmres", "bicgstab", "cgs"])
def test_int64_indices_identical(dev, kind):
    """i64 index instantiations (persistent CG, graph loops, ILU path) give bitwise the same
    runs as i32: the index width never enters the arithmetic."""
    c = 0.0 if kind == "cg" else 0.5
    runs = []
    for iw in (sp.IndexWidth.i32, sp.IndexWidth.i64):
        a = gen.stencil_csr(dev, 14, dim=3, c=c, index_width=iw)
        log, x, _ = solve(dev, kind, a, np.ones(a.rows), [sp.Iteration(2000), sp.ResidualNorm(1e-8)])
        runs.append((log, x))
        if kind in ("cg", "gmres"):
            xi = out(dev, a.rows, np.float64, fill=0.0)
            li = SOLVERS[kind](a, criteria=[sp.Iteration(2000), sp.ResidualNorm(1e-8)],
                               preconditioner=sp.ilu0_factorize(a)).solve(vec(dev, np.ones(a.rows)), xi)
            runs.append((li, host(xi)))
    half = len(runs) // 2
    for (l32, x32), (l64, x64) in zip(runs[:half], runs[half:]):
        assert l32.iterations == l64.iterations and l32.residual_history == l64.residual_history
        np.testing.assert_array_equal(x32, x64)


def test_persistent_cg_on_indexed_coo(dev):
    """Row-pointer-indexed COO runs the persistent CG like its CSR: same iterations."""
    from paper_2510_08230_b200 import _lib
    a = gen.stencil_csr(dev, 20, dim=3)
    c = sp.coo_from_csr(a)
    lc, xc, _ = solve(dev, "cg", c, np.ones(a.rows), [sp.Iteration(2000), sp.ResidualNorm(1e-8)])
    assert int(_lib.fn("sb_cg_last_loop")()) == 3
    assert int(_lib.fn("sb_cg_last_block_rows")()) == 512  # small system, stencil stage fits
    la, xa, _ = solve(dev, "cg", a, np.ones(a.rows), [sp.Iteration(2000), sp.ResidualNorm(1e-8)])
    assert lc.iterations == la.iterations and lc.residual_history == la.residual_history
    np.testing.assert_array_equal(xc, xa)
