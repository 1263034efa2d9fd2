// bicgstab.cuh -- BiCGSTAB's fused elementwise steps and reduction finalisers (recurrence
// in oracle/sbref.cpp), shared by bicgstab.cu and the row-partitioned dist_krylov.cu.
#pragma once
#include <cmath>

#include "solver_common.cuh"

namespace sb {

// ================================================================ BiCGSTAB
struct SkipEarly {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->early != 0; }
    __device__ __forceinline__ void prepare(const Ctl *) {}
};

// p = r (first) or p = r + beta (p - omega v) as axpy(-omega,v,p); scal(beta,p); axpy(1,r,p);
// phat = M p
template <class V>
struct BiDirection : SkipNone {
    using value_type = V;
    const V *r, *v, *inv;
    V *p, *ph;
    double beta, omega;
    bool first;
    __device__ __forceinline__ void prepare(const Ctl *c) {
        beta = c->beta;
        omega = c->omega;
        first = c->iter == 0;
    }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        const auto R = ldp<W>(r, i), D = ldp_or_one<W>(inv, i);
        Pk<V, W> P, PH;
        if (first) {
            P = R;
        } else {
            const auto Vv = ldp<W>(v, i);
            P = ldp<W>(p, i);
#pragma unroll
            for (int w = 0; w < W; ++w)
                P.v[w] = axpy_e(1.0, R.v[w], scal_e(beta, axpy_e(-omega, Vv.v[w], P.v[w])));
        }
        stp<W>(p, i, P);
        if (!ph) return;  // tri: phat comes from the sweeps
#pragma unroll
        for (int w = 0; w < W; ++w) PH.v[w] = inv ? vmul(P.v[w], D.v[w]) : P.v[w];
        stp<W>(ph, i, PH);
    }
};

// s = r - alpha v; shat = M s; ||s|| may stop early (x += alpha phat follows)
template <class V>
struct BiS : SkipNone {
    using value_type = V;
    using part_type = CAcc;
    const V *r, *v, *inv;
    V *s, *sh;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, CAcc (&part)[1]) const {
        const auto R = ldp<W>(r, i), Vv = ldp<W>(v, i), D = ldp_or_one<W>(inv, i);
        Pk<V, W> S, SH;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            S.v[w] = axpy_e(-alpha, Vv.v[w], R.v[w]);
            SH.v[w] = inv ? vmul(S.v[w], D.v[w]) : S.v[w];
            cadd(part[0], mulp(S.v[w], S.v[w]));
        }
        stp<W>(s, i, S);
        if (sh) stp<W>(sh, i, SH);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const {
        const double snorm = sqrt(tot[0]);
        c->snorm = snorm;
        if (c->has_rf && check_criteria(c, c->iter, snorm, c->bnorm) == STOP_RESIDUAL) {
            record(c, c->iter, snorm);
            c->early = 1;
        }
    }
};

// early stop: x += alpha phat, then finish
template <class V>
struct BiEarlyX {
    using value_type = V;
    const V *ph;
    V *x;
    double alpha;
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->early == 0; }
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        const auto PH = ldp<W>(ph, i);
        auto X = ldp<W>(x, i);
#pragma unroll
        for (int w = 0; w < W; ++w) X.v[w] = axpy_e(alpha, PH.v[w], X.v[w]);
        stp<W>(x, i, X);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&)[1]) const {
        finish_with(c, c->iter, STOP_RESIDUAL);
    }
};

// t = A shat with t.t and s.t -> omega
struct BiOmegaFin {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->early != 0; }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[2]) const {
        const double tt = tot[0], ts = tot[1];
        if (!isfinite(tt) || !isfinite(ts) || tt == 0.0) {
            breakdown(c, c->iter);
            return;
        }
        c->omega = ts / tt;
    }
};

// x += alpha phat + omega shat; r = s - omega t; dots r.r, rhat.r (next rho)
template <class V>
struct BiUpdate : SkipEarly {
    using value_type = V;
    using part_type = CAcc;
    const V *ph, *sh, *s, *t, *rh;
    V *x, *r;
    double alpha, omega;
    __device__ __forceinline__ void prepare(const Ctl *c) {
        alpha = c->alpha;
        omega = c->omega;
    }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, CAcc (&part)[2]) const {
        const auto PH = ldp<W>(ph, i), SH = ldp<W>(sh, i), S = ldp<W>(s, i), T = ldp<W>(t, i),
                   RH = ldp<W>(rh, i);
        auto X = ldp<W>(x, i);
        Pk<V, W> R;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            X.v[w] = axpy_e(omega, SH.v[w], axpy_e(alpha, PH.v[w], X.v[w]));
            R.v[w] = axpy_e(-omega, T.v[w], S.v[w]);
            cadd(part[0], mulp(R.v[w], R.v[w]));
            cadd(part[1], mulp(RH.v[w], R.v[w]));
        }
        stp<W>(x, i, X);
        stp<W>(r, i, R);
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
        if (c->omega == 0.0) {
            breakdown(c, it);
            return;
        }
        const double rho = tot[1];
        if (!isfinite(rho) || fabs(rho) <= kBreakdownRtol * c->shadow_norm * rnorm) {
            breakdown(c, it + 1);
            return;
        }
        c->rho_prev = c->rho;
        c->rho = rho;
        c->beta = (rho / c->rho_prev) * (c->alpha / c->omega);
    }
};

// ShadowInit (solver_common.cuh) with compensated dots
template <class V>
struct BiShadowInit : ShadowInit<V> {
    using part_type = CAcc;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, CAcc (&part)[2]) const {
        const auto B = ldp<W>(this->b, i), T = ldp<W>(this->t, i);
        Pk<V, W> R;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-1.0, T.v[w], B.v[w]);
            cadd(part[0], mulp(B.v[w], B.v[w]));
            cadd(part[1], mulp(R.v[w], R.v[w]));
        }
        stp<W>(this->r, i, R);
        stp<W>(this->shadow, i, R);
    }
};

}  // namespace sb
