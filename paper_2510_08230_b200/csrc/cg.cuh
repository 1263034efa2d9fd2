// cg.cuh -- the CG iteration's fused elementwise steps and reduction finalisers
// (solvers.py:188-224), shared by the single-GPU loops (cg.cu) and the row-partitioned
// solver (dist_krylov.cu, where the finalisers run after the cross-rank allreduce).
#pragma once
#include <cmath>

#include "solver_common.cuh"

namespace sb {

// ================================================================ CG
// setup: r = b - A x (t = A x first), z = M r, p = z; dots b.b, r.r, r.z
template <class V>
struct CgInit : SkipNone {
    using value_type = V;
    const V *b, *t, *inv;
    V *r, *z, *p;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[3]) const {
        const auto B = ldp<W>(b, i), T = ldp<W>(t, i), D = ldp_or_one<W>(inv, i);
        Pk<V, W> R, Z;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-1.0, T.v[w], B.v[w]);
            Z.v[w] = inv ? vmul(R.v[w], D.v[w]) : R.v[w];
            part[0] = addd(part[0], mulp(B.v[w], B.v[w]));
            part[1] = addd(part[1], mulp(R.v[w], R.v[w]));
            part[2] = addd(part[2], mulp(R.v[w], Z.v[w]));
        }
        stp<W>(r, i, R);
        stp<W>(z, i, Z);
        if (p) stp<W>(p, i, Z);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[3]) const {
        c->bnorm = sqrt(tot[0]);
        c->rnorm = sqrt(tot[1]);
        c->iter = 0;
        if (c->rnorm == 0.0) {  // _exact_log (solvers.py:179-181)
            c->exact = 1;
            c->converged = 1;
            c->stop_reason = STOP_RESIDUAL;
            if (c->hist_cap > 0) c->hist[0] = 0.0;
            c->hist_len = 1;
            stop_loop(c);
            return;
        }
        c->rz = tot[2];
    }
};

// q = A p, fused p.q -> alpha (solvers.py:202-206)
struct CgPqFin {
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const {
        const int64_t it = c->iter + 1;
        c->iter = it;
        const double pq = tot[0];
        if (!isfinite(pq) || pq <= kBreakdownRtol * fabs(c->rz)) {
            breakdown(c, it);
            return;
        }
        c->alpha = c->rz / pq;
    }
};

// x += alpha p; r -= alpha q; z = M r; dots r.r, r.z -> criteria, beta (solvers.py:207-222)
template <class V>
struct CgUpdate : SkipNone {
    using value_type = V;
    const V *p, *q, *inv;
    V *x, *r, *z;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[2]) const {
        const auto P = ldp<W>(p, i), Q = ldp<W>(q, i), D = ldp_or_one<W>(inv, i);
        auto X = ldp<W>(x, i), R = ldp<W>(r, i);
        Pk<V, W> Z;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            X.v[w] = axpy_e(alpha, P.v[w], X.v[w]);
            R.v[w] = axpy_e(-alpha, Q.v[w], R.v[w]);
            Z.v[w] = inv ? vmul(R.v[w], D.v[w]) : R.v[w];
            part[0] = addd(part[0], mulp(R.v[w], R.v[w]));
            part[1] = addd(part[1], mulp(R.v[w], Z.v[w]));
        }
        stp<W>(x, i, X);
        stp<W>(r, i, R);
        stp<W>(z, i, Z);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[2]) const {
        const int64_t it = c->iter;
        const double rnorm = sqrt(tot[0]);
        c->rnorm = rnorm;
        record(c, it, rnorm);
        int reason = check_criteria(c, it, rnorm, c->bnorm);
        if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
        if (reason != STOP_NONE) {
            finish_with(c, it, reason);
            return;
        }
        const double rz_new = tot[1];
        if (!isfinite(rz_new) || c->rz == 0.0) {
            breakdown(c, it);
            return;
        }
        c->beta = rz_new / c->rz;
        c->rz = rz_new;
    }
};

// p = z + beta p  (scal(beta, p); axpy(1, z, p))
template <class V>
struct CgDirection : SkipNone {
    using value_type = V;
    const V *z;
    V *p;
    double beta;
    __device__ __forceinline__ void prepare(const Ctl *c) { beta = c->beta; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        const auto Z = ldp<W>(z, i);
        auto P = ldp<W>(p, i);
#pragma unroll
        for (int w = 0; w < W; ++w) P.v[w] = axpy_e(1.0, Z.v[w], scal_e(beta, P.v[w]));
        stp<W>(p, i, P);
    }
};

}  // namespace sb
