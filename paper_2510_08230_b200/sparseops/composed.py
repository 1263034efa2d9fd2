"""Host-composed Krylov loops over device primitives, for operands the fused device
loops cannot take: a generic ``LinOp`` operator or preconditioner (a solver used as a
preconditioner, a user-defined operator, a dense matrix), and GMRES ``trace=``.

These are the reference's own loops (solvers.py:188-224 CG, :231-284 CGS, :322-399
GMRES, and the builder's BiCGSTAB recurrence of oracle/sbref.cpp) composed from the
library's device BLAS-1 (``core.dot/norm2/axpy/scal/copy_into`` -> ``sb_dot_*`` ...)
and ``LinOp.apply``: every vector operation runs as a CUDA kernel on the device; only
the scalars (dots, Givens rotations, the small Hessenberg system) live on the host,
exactly as in the reference.  There is no CPU path: every vector stays in HBM.

The fused device loops (``sb_<solver>_solve_*``) remain the path for sparse operators
with Jacobi / ILU / IC / no preconditioner; these loops only widen the operand types.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .core import DenseMatrix, axpy, copy_into, dense_create, dot, norm2, scal
from .errors import BreakdownError, InvalidArgumentError, NumericFailureError

BREAKDOWN_RTOL = 1e-30
STOP_RESIDUAL = "residual"
STOP_MAX_ITERS = "max_iters"


@dataclass
class GmresTraceEvent:
    """One inner-iteration snapshot handed to a GMRES trace callback (solvers.py:291-298):
    ``solution`` is a host copy of the iterate x would be if the cycle stopped here."""

    cycle: int
    inner: int
    estimate: float
    solution: np.ndarray


def _check_system(a, b: DenseMatrix, x: DenseMatrix):
    from .errors import DimensionMismatchError, PrecisionMismatchError

    rows, cols = a.shape
    if rows != cols:
        raise DimensionMismatchError(f"solver needs a square operator, got {rows}x{cols}")
    if b.shape != (rows, 1) or x.shape != (rows, 1):
        raise DimensionMismatchError(f"expected {rows}x1 vectors, got b {b.shape} and x {x.shape}")
    if b.values.dtype != x.values.dtype:
        raise PrecisionMismatchError("b and x must share one precision")


def _fresh(b: DenseMatrix) -> DenseMatrix:
    return dense_create(b.device, b.rows, 1, b.precision, 0.0)


def _residual(a, b, x, r, t) -> float:
    """r := b - A x, returning ||r|| (solvers.py:164-169)."""
    a.apply(x, t)
    copy_into(b, r)
    axpy(-1.0, t, r)
    return norm2(r)


def _apply_precond(m, r, z):
    if m is None:
        copy_into(r, z)
    else:
        m.apply(r, z)


def _log(cls, it, history, reason):
    return cls(it, history, reason == STOP_RESIDUAL, reason)


def _exact(cls):
    return cls(0, [0.0], True, STOP_RESIDUAL)


def run_cg(a, b, x, criteria, m, check, log_cls):
    """solvers.py:188-224."""
    _check_system(a, b, x)
    bnorm = norm2(b)
    r, z, p, q, t = (_fresh(b) for _ in range(5))
    rnorm = _residual(a, b, x, r, t)
    if rnorm == 0.0:
        return _exact(log_cls)
    _apply_precond(m, r, z)
    copy_into(z, p)
    rz = dot(r, z)
    history: list = []
    it = 0
    while True:
        it += 1
        a.apply(p, q)
        pq = dot(p, q)
        if not np.isfinite(pq) or pq <= BREAKDOWN_RTOL * abs(rz):
            raise BreakdownError(it, f"p'Ap = {pq} at iteration {it}; operator not SPD?")
        alpha = rz / pq
        axpy(alpha, p, x)
        axpy(-alpha, q, r)
        rnorm = norm2(r)
        history.append(rnorm)
        reason = check(criteria, it, rnorm, bnorm)
        if reason is None and rnorm == 0.0:
            reason = STOP_RESIDUAL
        if reason is not None:
            return _log(log_cls, it, history, reason)
        _apply_precond(m, r, z)
        rz_new = dot(r, z)
        if not np.isfinite(rz_new) or rz == 0.0:
            raise BreakdownError(it, f"r'z = {rz_new} at iteration {it}")
        beta = rz_new / rz
        scal(beta, p)
        axpy(1.0, z, p)
        rz = rz_new


def run_cgs(a, b, x, criteria, m, check, log_cls):
    """solvers.py:231-284."""
    _check_system(a, b, x)
    bnorm = norm2(b)
    r, r_shadow, u, p, q, v, uq, uhat, phat, t = (_fresh(b) for _ in range(10))
    rnorm = _residual(a, b, x, r, t)
    if rnorm == 0.0:
        return _exact(log_cls)
    copy_into(r, r_shadow)
    shadow_norm = rnorm
    history: list = []
    rho_prev = 0.0
    it = 0
    while True:
        it += 1
        rho = dot(r_shadow, r)
        if not np.isfinite(rho) or abs(rho) <= BREAKDOWN_RTOL * shadow_norm * rnorm:
            raise BreakdownError(it, f"rho = {rho} at iteration {it}")
        if it == 1:
            copy_into(r, u)
            copy_into(u, p)
        else:
            beta = rho / rho_prev
            copy_into(q, u)
            scal(beta, u)
            axpy(1.0, r, u)
            scal(beta * beta, p)
            axpy(beta, q, p)
            axpy(1.0, u, p)
        _apply_precond(m, p, phat)
        a.apply(phat, v)
        sigma = dot(r_shadow, v)
        if not np.isfinite(sigma) or abs(sigma) <= BREAKDOWN_RTOL * abs(rho):
            raise BreakdownError(it, f"r_shadow'Ap = {sigma} at iteration {it}")
        alpha = rho / sigma
        copy_into(u, q)
        axpy(-alpha, v, q)
        copy_into(u, uq)
        axpy(1.0, q, uq)
        _apply_precond(m, uq, uhat)
        axpy(alpha, uhat, x)
        a.apply(uhat, t)
        axpy(-alpha, t, r)
        rnorm = norm2(r)
        history.append(rnorm)
        reason = check(criteria, it, rnorm, bnorm)
        if reason is None and rnorm == 0.0:
            reason = STOP_RESIDUAL
        if reason is not None:
            return _log(log_cls, it, history, reason)
        rho_prev = rho


def run_bicgstab(a, b, x, criteria, m, check, log_cls):
    """Right-preconditioned BiCGSTAB (van der Vorst), the recurrence of oracle/sbref.cpp
    ``bicgstab`` in the reference's composition style."""
    _check_system(a, b, x)
    bnorm = norm2(b)
    r, rs, p, v, s, t, ph, sh, tmp = (_fresh(b) for _ in range(9))
    rnorm = _residual(a, b, x, r, tmp)
    if rnorm == 0.0:
        return _exact(log_cls)
    copy_into(r, rs)
    shadow_norm = rnorm
    history: list = []
    rho_prev = alpha = omega = 1.0
    it = 0
    while True:
        it += 1
        rho = dot(rs, r)
        if not np.isfinite(rho) or abs(rho) <= BREAKDOWN_RTOL * shadow_norm * rnorm:
            raise BreakdownError(it, f"rho = {rho} at iteration {it}")
        if it == 1:
            copy_into(r, p)
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            axpy(-omega, v, p)  # p = r + beta (p - omega v)
            scal(beta, p)
            axpy(1.0, r, p)
        _apply_precond(m, p, ph)
        a.apply(ph, v)
        sigma = dot(rs, v)
        if not np.isfinite(sigma) or abs(sigma) <= BREAKDOWN_RTOL * abs(rho):
            raise BreakdownError(it, f"r_shadow'Ap = {sigma} at iteration {it}")
        alpha = rho / sigma
        copy_into(r, s)
        axpy(-alpha, v, s)
        snorm = norm2(s)
        if check(criteria, it, snorm, bnorm) == STOP_RESIDUAL:
            axpy(alpha, ph, x)
            history.append(snorm)
            return _log(log_cls, it, history, STOP_RESIDUAL)
        _apply_precond(m, s, sh)
        a.apply(sh, t)
        tt = dot(t, t)
        ts = dot(t, s)
        if not np.isfinite(tt) or not np.isfinite(ts) or tt == 0.0:
            raise BreakdownError(it, f"t't = {tt}, t's = {ts} at iteration {it}")
        omega = ts / tt
        axpy(alpha, ph, x)
        axpy(omega, sh, x)
        copy_into(s, r)
        axpy(-omega, t, r)
        rnorm = norm2(r)
        history.append(rnorm)
        reason = check(criteria, it, rnorm, bnorm)
        if reason is None and rnorm == 0.0:
            reason = STOP_RESIDUAL
        if reason is not None:
            return _log(log_cls, it, history, reason)
        if omega == 0.0:
            raise BreakdownError(it, f"omega = 0 at iteration {it}")
        rho_prev = rho


def givens_rotation(a: float, b: float):
    import math

    if a == 0.0 and b == 0.0:
        return 1.0, 0.0, 0.0
    r = math.hypot(a, b)
    return a / r, b / r, r


def _back_substitute(r: np.ndarray, g: np.ndarray, k: int) -> np.ndarray:
    """solvers.py:301-308."""
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        acc = g[i]
        for j in range(i + 1, k):
            acc -= r[i, j] * y[j]
        y[i] = acc / r[i, i]
    return y


def _gmres_update(x, basis, r_mat, g, k, m, b):
    """x += M^{-1} (V_k y), solvers.py:311-319."""
    y = _back_substitute(r_mat, g, k)
    z_acc = _fresh(b)
    for i in range(k):
        axpy(float(y[i]), basis[i], z_acc)
    dx = _fresh(b)
    _apply_precond(m, z_acc, dx)
    axpy(1.0, dx, x)


def run_gmres(a, b, x, criteria, m, krylov_dim, check, log_cls,
              trace: Optional[Callable[[GmresTraceEvent], None]] = None):
    """solvers.py:322-399, including the per-inner-iteration trace snapshots."""
    _check_system(a, b, x)
    if krylov_dim < 1:
        raise InvalidArgumentError("krylov_dim must be positive")
    bnorm = norm2(b)
    dim = krylov_dim
    history: list = []
    total_inner = 0
    cycle = 0
    r, t, z, w = (_fresh(b) for _ in range(4))
    while True:
        beta = _residual(a, b, x, r, t)
        if beta == 0.0:
            if total_inner == 0:
                return _exact(log_cls)
            return log_cls(total_inner, history, True, STOP_RESIDUAL)
        v0 = _fresh(b)
        copy_into(r, v0)
        scal(1.0 / beta, v0)
        basis = [v0]
        r_mat = np.zeros((dim, dim))
        g = np.zeros(dim + 1)
        g[0] = beta
        cs = np.zeros(dim)
        sn = np.zeros(dim)
        for j in range(dim):
            _apply_precond(m, basis[j], z)
            a.apply(z, w)
            hcol = np.zeros(j + 2)
            for i in range(j + 1):
                hij = dot(basis[i], w)
                axpy(-hij, basis[i], w)
                hcol[i] = hij
            hnorm = norm2(w)
            hcol[j + 1] = hnorm
            if not np.all(np.isfinite(hcol)):
                raise NumericFailureError(
                    f"non-finite Hessenberg column at inner iteration {total_inner + 1}")
            for i in range(j):
                hi, hi1 = hcol[i], hcol[i + 1]
                hcol[i] = cs[i] * hi + sn[i] * hi1
                hcol[i + 1] = -sn[i] * hi + cs[i] * hi1
            c, s, rr = givens_rotation(float(hcol[j]), float(hcol[j + 1]))
            cs[j], sn[j] = c, s
            hcol[j] = rr
            r_mat[: j + 1, j] = hcol[: j + 1]
            g[j + 1] = -s * g[j]
            g[j] = c * g[j]
            estimate = abs(float(g[j + 1]))
            if not np.isfinite(estimate):
                raise NumericFailureError(
                    f"non-finite residual estimate at inner iteration {total_inner + 1}")
            total_inner += 1
            history.append(estimate)
            if trace is not None:
                xs = x.copy()
                _gmres_update(xs, basis, r_mat, g, j + 1, m, b)
                trace(GmresTraceEvent(cycle, total_inner, estimate, xs.column(0).cpu().numpy()))
            reason = check(criteria, total_inner, estimate, bnorm)
            happy = hnorm <= 1e-30 * bnorm
            if reason is not None or happy or j + 1 == dim:
                _gmres_update(x, basis, r_mat, g, j + 1, m, b)
                if reason is not None:
                    return log_cls(total_inner, history, reason == STOP_RESIDUAL, reason)
                break
            vnext = _fresh(b)
            copy_into(w, vnext)
            scal(1.0 / hnorm, vnext)
            basis.append(vnext)
        cycle += 1
