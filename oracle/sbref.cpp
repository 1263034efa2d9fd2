// sbref.cpp -- CPU restatement of the reference (the pyGinkgo artifact `sparseops`) hot path.
//
// TEST INFRASTRUCTURE ONLY.  This is the parity oracle: only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs
// may load it.  The product package (paper_2510_08230_b200) never links, imports
// or calls anything here.
//
// Each function restates one reference routine and cites it (paths relative to
// /root/reference/pkg/src/sparseops).  Numerics follow the reference exactly
// (SURVEY.md §0, §9 P8/P9):
//   * all accumulation in fp64; for fp32 buffers each product is rounded to fp32
//     before the fp64 add (numba float32*float32 -> float32);
//   * no FMA contraction (compiled with -ffp-contract=off);
//   * per-row accumulation is sequential in stored order;
//   * dot partials over core.partition(n, threads) are summed in chunk order, so
//     a `threads`-way run equals the reference `omp` device with that thread count.
// The restatement is pinned against vectors produced by the reference itself
// (tests/golden/make_golden.py -> tests/golden/*.npz; tests/test_oracle_golden.py).
#include <cmath>
#include <cstdlib>
#include <string>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <algorithm>

namespace {

constexpr double kBreakdownRtol = 1e-30;  // solvers.py:46
constexpr int64_t kParallelCutoff = 8192; // core.py:47

enum { ST_OK = 0, ST_BREAKDOWN = 1, ST_NUMERIC = 2 };
enum { STOP_NONE = -1, STOP_RESIDUAL = 0, STOP_MAX_ITERS = 1 };

}  // namespace

extern "C" {
struct ref_log {
    int64_t iterations;
    int32_t converged;
    int32_t stop_reason;       // STOP_RESIDUAL / STOP_MAX_ITERS
    int32_t status;            // ST_*
    int32_t pad;
    int64_t status_iteration;  // BreakdownError.iteration
    int64_t history_len;
};
struct ref_criteria {
    int64_t max_iters;         // min over Iteration entries
    int32_t has_residual;      // any ResidualNorm entry
    int32_t pad;
    double reduction_factor;   // max over ResidualNorm entries (OR semantics)
};
}

namespace {

// core.partition (core.py:173-183): contiguous chunks whose sizes differ by <= 1.
inline void partition(int64_t n, int parts, int t, int64_t &lo, int64_t &hi) {
    int64_t base = n / parts, rem = n % parts;
    lo = t * base + std::min<int64_t>(t, rem);
    hi = lo + base + (t < rem ? 1 : 0);
}

// core.run_chunks (core.py:186-196): one contiguous chunk per thread.
template <class F>
void run_partitioned(int threads, int64_t n, F &&fn) {
    if (threads <= 1 || n < kParallelCutoff) {
        if (threads <= 1) { fn(0, 0, n); return; }
        for (int t = 0; t < threads; ++t) {
            int64_t lo, hi;
            partition(n, threads, t, lo, hi);
            fn(t, lo, hi);
        }
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(threads);
    for (int t = 0; t < threads; ++t) {
        int64_t lo, hi;
        partition(n, threads, t, lo, hi);
        pool.emplace_back([&fn, t, lo, hi] { fn(t, lo, hi); });
    }
    for (auto &th : pool) th.join();
}

// numba arithmetic: float32*float32 -> float32 (rounded), then widened to fp64.
inline double mul(float a, float b) { return (double)(a * b); }
inline double mul(double a, double b) { return a * b; }

// solvers.check_criteria (solvers.py:121-135); the residual reason wins ties.
inline int check_criteria(const ref_criteria &c, int64_t it, double res, double rhs_norm) {
    if (c.has_residual) {
        double thr = rhs_norm > 0 ? c.reduction_factor * rhs_norm : c.reduction_factor;
        if (res <= thr) return STOP_RESIDUAL;
    }
    if (it >= c.max_iters) return STOP_MAX_ITERS;
    return STOP_NONE;
}

// ---------------------------------------------------------------- BLAS-1
// _kernels.dot_range (_kernels.py:44-49) + core.dot (core.py:358-373)
// Diagnostics only (tools/): SBREF_DOT=neumaier switches every dot to compensated
// (Neumaier) summation, to separate rounding sensitivity from algorithmic failure.
inline bool compensated_dots() {
    static const bool on = [] {
        const char *e = getenv("SBREF_DOT");
        return e && std::string(e) == "neumaier";
    }();
    return on;
}
inline void neumaier(double &s, double &c, double v) {
    const double t = s + v;
    c += std::fabs(s) >= std::fabs(v) ? (s - t) + v : (v - t) + s;
    s = t;
}

template <class V>
double dot(int64_t n, const V *x, const V *y, int th) {
    th = std::max(th, 1);
    if (compensated_dots()) {
        std::vector<double> ps(th, 0.0), pc(th, 0.0);
        run_partitioned(th, n, [&](int t, int64_t lo, int64_t hi) {
            double s = 0.0, c = 0.0;
            for (int64_t i = lo; i < hi; ++i) neumaier(s, c, mul(x[i], y[i]));
            ps[t] = s;
            pc[t] = c;
        });
        double s = 0.0, c = 0.0;
        for (int t = 0; t < th; ++t) {
            neumaier(s, c, ps[t]);
            neumaier(s, c, pc[t]);
        }
        return s + c;
    }
    std::vector<double> part(th, 0.0);
    run_partitioned(th, n, [&](int t, int64_t lo, int64_t hi) {
        double acc = 0.0;
        for (int64_t i = lo; i < hi; ++i) acc += mul(x[i], y[i]);
        part[t] = acc;
    });
    double acc = 0.0;
    for (int t = 0; t < th; ++t) acc += part[t];
    return acc;
}
// core.norm2 (core.py:376-378)
template <class V>
double norm2(int64_t n, const V *x, int th) { return std::sqrt(dot(n, x, x, th)); }
// _kernels.axpy_rows (_kernels.py:30-34): y = alpha*x + y with fp64 alpha, no FMA.
template <class V>
void axpy(int64_t n, double alpha, const V *x, V *y, int th) {
    run_partitioned(th, n, [&](int, int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            double p = alpha * (double)x[i];
            y[i] = (V)(p + (double)y[i]);
        }
    });
}
// _kernels.scal_rows (_kernels.py:37-41)
template <class V>
void scal(int64_t n, double alpha, V *x, int th) {
    run_partitioned(th, n, [&](int, int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) x[i] = (V)(alpha * (double)x[i]);
    });
}
// _kernels.copy_rows (_kernels.py:23-27)
template <class V>
void copy(int64_t n, const V *src, V *dst, int th) {
    run_partitioned(th, n, [&](int, int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) dst[i] = src[i];
    });
}
// JacobiPreconditioner.apply (precond.py:57-63): np.multiply in the value dtype.
template <class V>
void jacobi_apply(int64_t n, const V *inv, const V *b, V *x, int th) {
    run_partitioned(th, n, [&](int, int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) x[i] = (V)(b[i] * inv[i]);
    });
}

// ---------------------------------------------------------------- SpMV
// linop.spmv_csr (linop.py:102-121) -> _kernels.spmv_csr_rows (_kernels.py:62-68)
template <class V, class I>
void csr_spmv(int64_t rows, const I *rp, const I *ci, const V *val, const V *b, V *x, int th) {
    run_partitioned(th, rows, [&](int, int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            double acc = 0.0;
            for (int64_t k = rp[i]; k < (int64_t)rp[i + 1]; ++k) acc += mul(val[k], b[ci[k]]);
            x[i] = (V)acc;
        }
    });
}

// linop.spmv_coo (linop.py:137-159) with zero_range / spmv_coo_entries (_kernels.py:71-88)
template <class V, class I>
void coo_spmv(int64_t rows, int64_t nnz, const I *ri, const I *ci, const V *val, const V *b, V *x) {
    for (int64_t i = 0; i < rows; ++i) x[i] = (V)0;
    int64_t k = 0;
    while (k < nnz) {
        int64_t i = ri[k];
        double acc = 0.0;
        while (k < nnz && (int64_t)ri[k] == i) {
            acc += mul(val[k], b[ci[k]]);
            ++k;
        }
        x[i] = (V)acc;
    }
}

// CsrMatrix.diagonal (formats.py:113-122) + jacobi_create (precond.py:66-84).
// Returns -1 on success, else the first singular row (SingularDiagonalError.row).
template <class V, class I>
int64_t jacobi_create(int64_t n, const I *rp, const I *ci, const V *val, V *inv) {
    std::vector<V> diag(n, (V)0);
    for (int64_t i = 0; i < n; ++i) {
        const I *b0 = ci + rp[i], *b1 = ci + rp[i + 1];
        const I *p = std::lower_bound(b0, b1, (I)i);  // np.searchsorted (left)
        if (p < b1 && (int64_t)*p == i) diag[i] = val[p - ci];
    }
    for (int64_t i = 0; i < n; ++i)
        if (diag[i] == (V)0) return i;
    for (int64_t i = 0; i < n; ++i) inv[i] = (V)(1.0 / (double)diag[i]);
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite((double)inv[i])) return i;
    return -1;
}

// ---------------------------------------------------------------- formats the reference lacks
// Canonical layouts (SURVEY.md §8 "Proposed canonical layouts"); all derive from canonical CSR.
// ELL(w, stride): entry k of row i at k*stride + i; padding col = -1, val = 0.
template <class V, class I>
void ell_from_csr(int64_t rows, const I *rp, const I *ci, const V *val, int64_t w, int64_t stride,
                  I *ecol, V *evals) {
    for (int64_t k = 0; k < w; ++k)
        for (int64_t i = 0; i < stride; ++i) {
            int64_t len = i < rows ? (int64_t)(rp[i + 1] - rp[i]) : 0;
            int64_t dst = k * stride + i;
            if (k < len) { ecol[dst] = ci[rp[i] + k]; evals[dst] = val[rp[i] + k]; }
            else { ecol[dst] = (I)-1; evals[dst] = (V)0; }
        }
}
// SELL-P(S): slice_lengths[s] = max row length in slice; slice_sets = exclusive scan
// (length n_slices + 1); entry k of row i (slice s = i / S) at (slice_sets[s] + k)*S + i%S.
template <class V, class I>
void sellp_from_csr(int64_t rows, const I *rp, const I *ci, const V *val, int64_t S,
                    I *slice_lengths, I *slice_sets, I *scol, V *svals) {
    int64_t ns = (rows + S - 1) / S;
    slice_sets[0] = 0;
    for (int64_t s = 0; s < ns; ++s) {
        int64_t m = 0;
        for (int64_t i = s * S; i < std::min((s + 1) * S, rows); ++i)
            m = std::max<int64_t>(m, rp[i + 1] - rp[i]);
        slice_lengths[s] = (I)m;
        slice_sets[s + 1] = (I)(slice_sets[s] + m);
    }
    for (int64_t s = 0; s < ns; ++s)
        for (int64_t k = 0; k < (int64_t)slice_lengths[s]; ++k)
            for (int64_t l = 0; l < S; ++l) {
                int64_t i = s * S + l;
                int64_t dst = ((int64_t)slice_sets[s] + k) * S + l;
                int64_t len = i < rows ? (int64_t)(rp[i + 1] - rp[i]) : 0;
                if (k < len) { scol[dst] = ci[rp[i] + k]; svals[dst] = val[rp[i] + k]; }
                else { scol[dst] = (I)-1; svals[dst] = (V)0; }
            }
}
// ELL / SELL-P SpMV: same per-row sequential order as CSR, padding skipped.
template <class V, class I>
void ell_spmv(int64_t rows, int64_t w, int64_t stride, const I *ecol, const V *evals, const V *b, V *x) {
    for (int64_t i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int64_t k = 0; k < w; ++k) {
            I c = ecol[k * stride + i];
            if (c >= 0) acc += mul(evals[k * stride + i], b[c]);
        }
        x[i] = (V)acc;
    }
}
template <class V, class I>
void sellp_spmv(int64_t rows, int64_t S, const I *slice_lengths, const I *slice_sets, const I *scol,
                const V *svals, const V *b, V *x) {
    for (int64_t i = 0; i < rows; ++i) {
        int64_t s = i / S, l = i % S;
        double acc = 0.0;
        for (int64_t k = 0; k < (int64_t)slice_lengths[s]; ++k) {
            int64_t p = ((int64_t)slice_sets[s] + k) * S + l;
            if (scol[p] >= 0) acc += mul(svals[p], b[scol[p]]);
        }
        x[i] = (V)acc;
    }
}

// ---------------------------------------------------------------- Krylov solvers
template <class V, class I>
struct System {
    int64_t n;
    const I *rp, *ci;
    const V *val, *inv;
    int th;
    void apply(const V *b, V *x) const { csr_spmv(n, rp, ci, val, b, x, th); }
    // solvers._apply_precond (solvers.py:172-176): identity is a copy
    void precond(const V *r, V *z) const {
        if (inv) jacobi_apply(n, inv, r, z, th);
        else copy(n, r, z, th);
    }
    // solvers._residual (solvers.py:164-169): r := b - A x via t, copy and axpy(-1)
    double residual(const V *b, const V *x, V *r, V *t) const {
        apply(x, t);
        copy(n, b, r, th);
        axpy(n, -1.0, t, r, th);
        return norm2(n, r, th);
    }
    std::vector<V> fresh() const { return std::vector<V>(std::max<int64_t>(n, 1), (V)0); }
};

// solvers._exact_log (solvers.py:179-181)
void exact_log(ref_log *log, double *hist, int64_t cap) {
    log->iterations = 0;
    log->converged = 1;
    log->stop_reason = STOP_RESIDUAL;
    log->history_len = 1;
    if (cap > 0) hist[0] = 0.0;
}
void breakdown(ref_log *log, int64_t it) {
    log->status = ST_BREAKDOWN;
    log->status_iteration = it;
    log->iterations = it;
}
void record(double *hist, int64_t cap, ref_log *log, int64_t it, double res) {
    if (it - 1 < cap) hist[it - 1] = res;
    log->history_len = it;
}
bool finish(ref_log *log, int64_t it, int reason) {
    if (reason == STOP_NONE) return false;
    log->iterations = it;
    log->converged = reason == STOP_RESIDUAL;
    log->stop_reason = reason;
    return true;
}

// solvers._run_cg (solvers.py:188-224)
template <class V, class I>
void cg(const System<V, I> &A, const V *b, V *x, const ref_criteria &crit, double *hist, int64_t cap,
        ref_log *log) {
    const int64_t n = A.n;
    const int th = A.th;
    std::memset(log, 0, sizeof(*log));
    double bnorm = norm2(n, b, th);
    auto r = A.fresh(), z = A.fresh(), p = A.fresh(), q = A.fresh(), t = A.fresh();
    double rnorm = A.residual(b, x, r.data(), t.data());
    if (rnorm == 0.0) return exact_log(log, hist, cap);
    A.precond(r.data(), z.data());
    copy(n, z.data(), p.data(), th);
    double rz = dot(n, r.data(), z.data(), th);
    for (int64_t it = 1;; ++it) {
        A.apply(p.data(), q.data());
        double pq = dot(n, p.data(), q.data(), th);
        if (!std::isfinite(pq) || pq <= kBreakdownRtol * std::fabs(rz)) return breakdown(log, it);
        double alpha = rz / pq;
        axpy(n, alpha, p.data(), x, th);
        axpy(n, -alpha, q.data(), r.data(), th);
        rnorm = norm2(n, r.data(), th);
        record(hist, cap, log, it, rnorm);
        int reason = check_criteria(crit, it, rnorm, bnorm);
        if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
        if (finish(log, it, reason)) return;
        A.precond(r.data(), z.data());
        double rz_new = dot(n, r.data(), z.data(), th);
        if (!std::isfinite(rz_new) || rz == 0.0) return breakdown(log, it);
        double beta = rz_new / rz;
        scal(n, beta, p.data(), th);
        axpy(n, 1.0, z.data(), p.data(), th);
        rz = rz_new;
    }
}

// solvers._run_cgs (solvers.py:231-284)
template <class V, class I>
void cgs(const System<V, I> &A, const V *b, V *x, const ref_criteria &crit, double *hist, int64_t cap,
         ref_log *log) {
    const int64_t n = A.n;
    const int th = A.th;
    std::memset(log, 0, sizeof(*log));
    double bnorm = norm2(n, b, th);
    auto r = A.fresh(), rs = A.fresh(), u = A.fresh(), p = A.fresh(), q = A.fresh(), v = A.fresh(),
         uq = A.fresh(), uhat = A.fresh(), phat = A.fresh(), t = A.fresh();
    double rnorm = A.residual(b, x, r.data(), t.data());
    if (rnorm == 0.0) return exact_log(log, hist, cap);
    copy(n, r.data(), rs.data(), th);
    const double shadow_norm = rnorm;
    double rho_prev = 0.0;
    for (int64_t it = 1;; ++it) {
        double rho = dot(n, rs.data(), r.data(), th);
        if (!std::isfinite(rho) || std::fabs(rho) <= kBreakdownRtol * shadow_norm * rnorm)
            return breakdown(log, it);
        if (it == 1) {
            copy(n, r.data(), u.data(), th);
            copy(n, u.data(), p.data(), th);
        } else {
            double beta = rho / rho_prev;
            copy(n, q.data(), u.data(), th);
            scal(n, beta, u.data(), th);
            axpy(n, 1.0, r.data(), u.data(), th);
            scal(n, beta * beta, p.data(), th);
            axpy(n, beta, q.data(), p.data(), th);
            axpy(n, 1.0, u.data(), p.data(), th);
        }
        A.precond(p.data(), phat.data());
        A.apply(phat.data(), v.data());
        double sigma = dot(n, rs.data(), v.data(), th);
        if (!std::isfinite(sigma) || std::fabs(sigma) <= kBreakdownRtol * std::fabs(rho))
            return breakdown(log, it);
        double alpha = rho / sigma;
        copy(n, u.data(), q.data(), th);
        axpy(n, -alpha, v.data(), q.data(), th);
        copy(n, u.data(), uq.data(), th);
        axpy(n, 1.0, q.data(), uq.data(), th);
        A.precond(uq.data(), uhat.data());
        axpy(n, alpha, uhat.data(), x, th);
        A.apply(uhat.data(), t.data());
        axpy(n, -alpha, t.data(), r.data(), th);
        rnorm = norm2(n, r.data(), th);
        record(hist, cap, log, it, rnorm);
        int reason = check_criteria(crit, it, rnorm, bnorm);
        if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
        if (finish(log, it, reason)) return;
        rho_prev = rho;
    }
}

// Right-preconditioned BiCGSTAB (van der Vorst).  NOT in the reference (
// parity unpinned by the reference's tests).  Builder-written in the reference's style: the
// same primitives (copy/scal/axpy/dot/apply), criteria (solvers.py:121-135), breakdown rule
// (solvers.py:46) and recurrence-residual stop as _run_cgs (solvers.py:231-284).
// One iteration = two SpMVs:
//   rho = rhat.r                       (breakdown if |rho| <= 1e-30 ||rhat|| ||r||)
//   it == 1: p = r;  else beta = (rho/rho_prev)(alpha/omega);
//            p = r + beta (p - omega v)  as axpy(-omega, v, p); scal(beta, p); axpy(1, r, p)
//   phat = M p; v = A phat; sigma = rhat.v  (breakdown if |sigma| <= 1e-30 |rho|)
//   alpha = rho/sigma; s = r - alpha v      (copy + axpy)
//   ||s|| meets a ResidualNorm criterion -> x += alpha phat; history gets ||s||; stop
//   shat = M s; t = A shat; tt = t.t; ts = t.s (breakdown if tt == 0); omega = ts/tt
//   x += alpha phat; x += omega shat; r = s - omega t (copy + axpy); history ||r||; check
//   omega == 0 without a stop -> breakdown (the next beta would divide by it)
template <class V, class I>
void bicgstab(const System<V, I> &A, const V *b, V *x, const ref_criteria &crit, double *hist,
              int64_t cap, ref_log *log) {
    const int64_t n = A.n;
    const int th = A.th;
    std::memset(log, 0, sizeof(*log));
    double bnorm = norm2(n, b, th);
    auto r = A.fresh(), rh = A.fresh(), p = A.fresh(), v = A.fresh(), s = A.fresh(), ph = A.fresh(),
         sh = A.fresh(), t = A.fresh();
    double rnorm = A.residual(b, x, r.data(), t.data());
    if (rnorm == 0.0) return exact_log(log, hist, cap);
    copy(n, r.data(), rh.data(), th);
    const double rh_norm = rnorm;
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    for (int64_t it = 1;; ++it) {
        double rho = dot(n, rh.data(), r.data(), th);
        if (!std::isfinite(rho) || std::fabs(rho) <= kBreakdownRtol * rh_norm * rnorm)
            return breakdown(log, it);
        if (it == 1) {
            copy(n, r.data(), p.data(), th);
        } else {
            double beta = (rho / rho_prev) * (alpha / omega);
            axpy(n, -omega, v.data(), p.data(), th);
            scal(n, beta, p.data(), th);
            axpy(n, 1.0, r.data(), p.data(), th);
        }
        A.precond(p.data(), ph.data());
        A.apply(ph.data(), v.data());
        double sigma = dot(n, rh.data(), v.data(), th);
        if (!std::isfinite(sigma) || std::fabs(sigma) <= kBreakdownRtol * std::fabs(rho))
            return breakdown(log, it);
        alpha = rho / sigma;
        copy(n, r.data(), s.data(), th);
        axpy(n, -alpha, v.data(), s.data(), th);
        double snorm = norm2(n, s.data(), th);
        if (crit.has_residual && check_criteria(crit, it, snorm, bnorm) == STOP_RESIDUAL) {
            axpy(n, alpha, ph.data(), x, th);
            record(hist, cap, log, it, snorm);
            finish(log, it, STOP_RESIDUAL);
            return;
        }
        A.precond(s.data(), sh.data());
        A.apply(sh.data(), t.data());
        double tt = dot(n, t.data(), t.data(), th);
        double ts = dot(n, t.data(), s.data(), th);
        if (!std::isfinite(tt) || !std::isfinite(ts) || tt == 0.0) return breakdown(log, it);
        omega = ts / tt;
        axpy(n, alpha, ph.data(), x, th);
        axpy(n, omega, sh.data(), x, th);
        copy(n, s.data(), r.data(), th);
        axpy(n, -omega, t.data(), r.data(), th);
        rnorm = norm2(n, r.data(), th);
        record(hist, cap, log, it, rnorm);
        int reason = check_criteria(crit, it, rnorm, bnorm);
        if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
        if (finish(log, it, reason)) return;
        if (omega == 0.0) return breakdown(log, it);
        rho_prev = rho;
    }
}

// solvers._run_gmres (solvers.py:322-399) with givens_rotation (:138-143),
// _back_substitute (:301-308) and _gmres_update (:311-319).
template <class V, class I>
void gmres(const System<V, I> &A, const V *b, V *x, const ref_criteria &crit, int64_t dim,
           double *hist, int64_t cap, ref_log *log) {
    const int64_t n = A.n;
    const int th = A.th;
    std::memset(log, 0, sizeof(*log));
    double bnorm = norm2(n, b, th);
    auto r = A.fresh(), t = A.fresh(), z = A.fresh(), w = A.fresh();
    std::vector<std::vector<V>> basis;
    std::vector<double> rmat(dim * dim), g(dim + 1), cs(dim), sn(dim), hcol(dim + 1), y(dim);
    int64_t total = 0;
    for (;;) {
        double beta = A.residual(b, x, r.data(), t.data());
        if (beta == 0.0) {
            if (total == 0) return exact_log(log, hist, cap);
            finish(log, total, STOP_RESIDUAL);
            return;
        }
        basis.clear();
        basis.push_back(A.fresh());
        copy(n, r.data(), basis[0].data(), th);
        scal(n, 1.0 / beta, basis[0].data(), th);
        std::fill(rmat.begin(), rmat.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        std::fill(cs.begin(), cs.end(), 0.0);
        std::fill(sn.begin(), sn.end(), 0.0);
        g[0] = beta;
        for (int64_t j = 0; j < dim; ++j) {
            A.precond(basis[j].data(), z.data());
            A.apply(z.data(), w.data());
            std::fill(hcol.begin(), hcol.end(), 0.0);
            for (int64_t i = 0; i <= j; ++i) {  // modified Gram-Schmidt, single pass
                double hij = dot(n, basis[i].data(), w.data(), th);
                axpy(n, -hij, basis[i].data(), w.data(), th);
                hcol[i] = hij;
            }
            double hnorm = norm2(n, w.data(), th);
            hcol[j + 1] = hnorm;
            for (int64_t i = 0; i <= j + 1; ++i)
                if (!std::isfinite(hcol[i])) {
                    log->status = ST_NUMERIC;
                    log->status_iteration = total + 1;
                    log->iterations = total;
                    return;
                }
            for (int64_t i = 0; i < j; ++i) {
                double hi = hcol[i], hi1 = hcol[i + 1];
                hcol[i] = cs[i] * hi + sn[i] * hi1;
                hcol[i + 1] = -sn[i] * hi + cs[i] * hi1;
            }
            double c, s, rr;
            if (hcol[j] == 0.0 && hcol[j + 1] == 0.0) {
                c = 1.0; s = 0.0; rr = 0.0;
            } else {
                rr = std::hypot(hcol[j], hcol[j + 1]);
                c = hcol[j] / rr;
                s = hcol[j + 1] / rr;
            }
            cs[j] = c;
            sn[j] = s;
            hcol[j] = rr;
            for (int64_t i = 0; i <= j; ++i) rmat[i * dim + j] = hcol[i];
            g[j + 1] = -s * g[j];
            g[j] = c * g[j];
            double est = std::fabs(g[j + 1]);
            if (!std::isfinite(est)) {
                log->status = ST_NUMERIC;
                log->status_iteration = total + 1;
                log->iterations = total;
                return;
            }
            total += 1;
            record(hist, cap, log, total, est);
            int reason = check_criteria(crit, total, est, bnorm);
            bool happy = hnorm <= 1e-30 * bnorm;
            if (reason != STOP_NONE || happy || j + 1 == dim) {
                int64_t k = j + 1;
                for (int64_t i = k - 1; i >= 0; --i) {
                    double acc = g[i];
                    for (int64_t q = i + 1; q < k; ++q) acc -= rmat[i * dim + q] * y[q];
                    y[i] = acc / rmat[i * dim + i];
                }
                auto zacc = A.fresh(), dx = A.fresh();
                for (int64_t i = 0; i < k; ++i) axpy(n, y[i], basis[i].data(), zacc.data(), th);
                A.precond(zacc.data(), dx.data());
                axpy(n, 1.0, dx.data(), x, th);
                if (finish(log, total, reason)) return;
                break;  // restart
            }
            basis.push_back(A.fresh());
            copy(n, w.data(), basis[j + 1].data(), th);
            scal(n, 1.0 / hnorm, basis[j + 1].data(), th);
        }
    }
}

// coo_from_arrays (formats.py:131-166): stable lexsort by (row, col); duplicates summed
// strictly left to right in sorted order in the value dtype; explicit zeros kept.
template <class V>
int64_t coo_canonicalize(int64_t m, const int64_t *ri, const int64_t *ci, const V *vals,
                         int64_t *out_r, int64_t *out_c, V *out_v) {
    std::vector<int64_t> order(m);
    for (int64_t k = 0; k < m; ++k) order[k] = k;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return ri[a] != ri[b] ? ri[a] < ri[b] : ci[a] < ci[b];
    });
    int64_t nnz = 0;
    for (int64_t k = 0; k < m;) {
        int64_t s = order[k], e = k + 1;
        while (e < m && ri[order[e]] == ri[s] && ci[order[e]] == ci[s]) ++e;
        V acc = vals[s];
        for (int64_t q = k + 1; q < e; ++q) acc = acc + vals[order[q]];
        out_r[nnz] = ri[s];
        out_c[nnz] = ci[s];
        out_v[nnz] = acc;
        ++nnz;
        k = e;
    }
    return nnz;
}

// ---------------------------------------------------------------- triangular solves
// _kernels.solve_lower / solve_upper (_kernels.py:91-137): acc = b[i] + 0.0 in fp64;
// acc -= values[k] * x[j] (product in the value dtype, like numba float32 * float32);
// x[i] = acc (unit) or acc / diag in fp64, cast on store.  Returns status 0 ok, 1 entry
// on the wrong side of the diagonal (row), 2 missing / zero diagonal (row).
template <class V, class I>
int trsv(int64_t n, const I *rp, const I *ci, const V *val, const V *b, V *x, bool lower, bool unit,
         int64_t *row) {
    for (int64_t t = 0; t < n; ++t) {
        const int64_t i = lower ? t : n - 1 - t;
        double acc = (double)b[i] + 0.0;
        double diag = 0.0;
        bool has_diag = false;
        for (int64_t k = rp[i]; k < (int64_t)rp[i + 1]; ++k) {
            const int64_t j = ci[k];
            if (lower ? j < i : j > i) {
                acc -= mul(val[k], x[j]);
            } else if (j == i) {
                diag = (double)val[k];
                has_diag = true;
            } else {
                *row = i;
                return 1;
            }
        }
        if (lower && unit) {
            x[i] = (V)acc;
        } else {
            if (!has_diag || diag == 0.0) {
                *row = i;
                return 2;
            }
            x[i] = (V)(acc / diag);
        }
    }
    *row = -1;
    return 0;
}

// ilu0_factorize (precond.py:155-187): IKJ elimination on the stored pattern, in place on
// a copy of the values, arithmetic in the value dtype.  Returns -1 or the zero-pivot row.
template <class V, class I>
int64_t ilu0(int64_t n, const I *rp, const I *ci, V *vals) {
    std::vector<int64_t> dpos(n, -1);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < (int64_t)rp[i + 1]; ++k)
            if ((int64_t)ci[k] == i) dpos[i] = k;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t s = rp[i], e = rp[i + 1];
        for (int64_t idx = s; idx < e; ++idx) {
            const int64_t k = ci[idx];
            if (k >= i) break;
            const int64_t dk = dpos[k];
            const V ukk = dk >= 0 ? vals[dk] : (V)0;
            if (ukk == (V)0) return k;
            const V lik = vals[idx] / ukk;
            vals[idx] = lik;
            for (int64_t idx2 = dk + 1; idx2 < (int64_t)rp[k + 1]; ++idx2) {
                const I j = ci[idx2];
                const I *pos = std::lower_bound(ci + s, ci + e, j);
                if (pos != ci + e && *pos == j) {
                    V &a = vals[pos - ci];
                    a = a - lik * vals[idx2];
                }
            }
        }
        if (dpos[i] < 0 || vals[dpos[i]] == (V)0) return i;
    }
    return -1;
}

// ic0_factorize (precond.py:205-256) on the lower pattern (cols <= i, diagonal last):
// Python-float (fp64) arithmetic throughout, cast to the value dtype at the end.
// Returns -1 or the row of the first non-positive / missing pivot.
template <class V, class I>
int64_t ic0(int64_t n, const I *lp, const I *lc, const V *a_lower, V *out) {
    std::vector<double> lv((size_t)lp[n], 0.0);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t si = lp[i], ei = lp[i + 1];
        for (int64_t pos = si; pos < ei; ++pos) {
            const int64_t j = lc[pos];
            double s = (double)a_lower[pos];
            const int64_t sj = lp[j], ej = lp[j + 1];
            int64_t pi = si, pj = sj;
            while (pi < ei && pj < ej) {
                const int64_t c1 = lc[pi], c2 = lc[pj];
                if (c1 >= j || c2 >= j) break;
                if (c1 == c2) {
                    s -= lv[pi] * lv[pj];
                    ++pi;
                    ++pj;
                } else if (c1 < c2) {
                    ++pi;
                } else {
                    ++pj;
                }
            }
            if (j == i) {
                if (s <= 0.0) return i;
                lv[pos] = std::sqrt(s);
            } else {
                if (ej == sj || (int64_t)lc[ej - 1] != j || lv[ej - 1] == 0.0) return j;
                lv[pos] = s / lv[ej - 1];
            }
        }
        if (ei == si || (int64_t)lc[ei - 1] != i) return i;
    }
    for (int64_t k = 0; k < (int64_t)lp[n]; ++k) out[k] = (V)lv[k];
    return -1;
}

}  // namespace

// ---------------------------------------------------------------- exported C ABI (ctypes)
#define SBREF_VALUE(V, VN)                                                                        \
    extern "C" double ref_dot_##VN(int64_t n, const V *x, const V *y, int th) {                   \
        return dot(n, x, y, th);                                                                  \
    }                                                                                             \
    extern "C" double ref_norm2_##VN(int64_t n, const V *x, int th) { return norm2(n, x, th); }   \
    extern "C" void ref_axpy_##VN(int64_t n, double a, const V *x, V *y, int th) {                \
        axpy(n, a, x, y, th);                                                                     \
    }                                                                                             \
    extern "C" void ref_scal_##VN(int64_t n, double a, V *x, int th) { scal(n, a, x, th); }       \
    extern "C" void ref_jacobi_apply_##VN(int64_t n, const V *inv, const V *b, V *x, int th) {    \
        jacobi_apply(n, inv, b, x, th);                                                           \
    }                                                                                             \
    extern "C" int64_t ref_coo_canonicalize_##VN(int64_t m, const int64_t *ri, const int64_t *ci, \
                                                 const V *v, int64_t *orow, int64_t *ocol,        \
                                                 V *oval) {                                       \
        return coo_canonicalize(m, ri, ci, v, orow, ocol, oval);                                  \
    }

#define SBREF_INDEX(V, VN, I, IN)                                                                  \
    extern "C" void ref_csr_spmv_##VN##_##IN(int64_t rows, const I *rp, const I *ci,               \
                                             const V *val, const V *b, V *x, int th) {             \
        csr_spmv(rows, rp, ci, val, b, x, th);                                                     \
    }                                                                                              \
    extern "C" void ref_coo_spmv_##VN##_##IN(int64_t rows, int64_t nnz, const I *ri, const I *ci,  \
                                             const V *val, const V *b, V *x) {                     \
        coo_spmv(rows, nnz, ri, ci, val, b, x);                                                    \
    }                                                                                              \
    extern "C" int64_t ref_jacobi_create_##VN##_##IN(int64_t n, const I *rp, const I *ci,          \
                                                     const V *val, V *inv) {                       \
        return jacobi_create(n, rp, ci, val, inv);                                                 \
    }                                                                                              \
    extern "C" void ref_ell_from_csr_##VN##_##IN(int64_t rows, const I *rp, const I *ci,           \
                                                 const V *val, int64_t w, int64_t stride, I *ec,   \
                                                 V *ev) {                                          \
        ell_from_csr(rows, rp, ci, val, w, stride, ec, ev);                                        \
    }                                                                                              \
    extern "C" void ref_sellp_from_csr_##VN##_##IN(int64_t rows, const I *rp, const I *ci,         \
                                                   const V *val, int64_t S, I *sl, I *ss, I *sc,   \
                                                   V *sv) {                                        \
        sellp_from_csr(rows, rp, ci, val, S, sl, ss, sc, sv);                                      \
    }                                                                                              \
    extern "C" void ref_ell_spmv_##VN##_##IN(int64_t rows, int64_t w, int64_t stride, const I *ec, \
                                             const V *ev, const V *b, V *x) {                      \
        ell_spmv(rows, w, stride, ec, ev, b, x);                                                   \
    }                                                                                              \
    extern "C" void ref_sellp_spmv_##VN##_##IN(int64_t rows, int64_t S, const I *sl, const I *ss,  \
                                               const I *sc, const V *sv, const V *b, V *x) {       \
        sellp_spmv(rows, S, sl, ss, sc, sv, b, x);                                                 \
    }                                                                                              \
    extern "C" int ref_trsv_##VN##_##IN(int64_t n, const I *rp, const I *ci, const V *val,         \
                                        const V *b, V *x, int lower, int unit, int64_t *row) {     \
        return trsv(n, rp, ci, val, b, x, lower != 0, unit != 0, row);                             \
    }                                                                                              \
    extern "C" int64_t ref_ilu0_##VN##_##IN(int64_t n, const I *rp, const I *ci, V *vals) {        \
        return ilu0(n, rp, ci, vals);                                                              \
    }                                                                                              \
    extern "C" int64_t ref_ic0_##VN##_##IN(int64_t n, const I *lp, const I *lc, const V *al,       \
                                           V *out) {                                               \
        return ic0(n, lp, lc, al, out);                                                            \
    }                                                                                              \
    extern "C" void ref_solve_##VN##_##IN(int kind, int64_t n, const I *rp, const I *ci,           \
                                          const V *val, const V *inv, const V *b, V *x,            \
                                          const ref_criteria *crit, int64_t dim, double *hist,     \
                                          int64_t cap, ref_log *log, int th) {                     \
        System<V, I> A{n, rp, ci, val, inv, std::max(th, 1)};                                      \
        switch (kind) {                                                                            \
        case 0: cg(A, b, x, *crit, hist, cap, log); break;                                         \
        case 1: cgs(A, b, x, *crit, hist, cap, log); break;                                        \
        case 2: gmres(A, b, x, *crit, dim, hist, cap, log); break;                                 \
        default: bicgstab(A, b, x, *crit, hist, cap, log); break;                                  \
        }                                                                                          \
    }

SBREF_VALUE(float, float)
SBREF_VALUE(double, double)
SBREF_INDEX(float, float, int32_t, i32)
SBREF_INDEX(float, float, int64_t, i64)
SBREF_INDEX(double, double, int32_t, i32)
SBREF_INDEX(double, double, int64_t, i64)

extern "C" int ref_hardware_threads(void) {
    unsigned h = std::thread::hardware_concurrency();
    return h ? (int)h : 1;
}
