// gmres.cuh -- GMRES(m)'s fused elementwise steps, Givens / criteria finalisers and the
// cycle-end update (solvers.py:322-399), shared by gmres.cu and dist_krylov.cu.
#pragma once
#include <cmath>

#include "solver_common.cuh"

namespace sb {

// ================================================================ GMRES(m) (solvers.py:322-399)
struct SkipCycleEnd {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->cycle_end != 0; }
    __device__ __forceinline__ void prepare(const Ctl *) {}
};
struct SkipUnlessCycleEnd {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->cycle_end == 0; }
    __device__ __forceinline__ void prepare(const Ctl *) {}
};

// restart: r = b - A x, beta = ||r||; reset the cycle's small dense state
template <class V>
struct GmRestart : SkipNone {
    using value_type = V;
    const V *b, *t;
    V *r;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[1]) const {
        const auto B = ldp<W>(b, i), T = ldp<W>(t, i);
        Pk<V, W> R;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-1.0, T.v[w], B.v[w]);
            part[0] = addd(part[0], mulp(R.v[w], R.v[w]));
        }
        stp<W>(r, i, R);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const {
        const double beta = sqrt(tot[0]);
        if (beta == 0.0) {
            if (c->iter == 0) exact_log(c);
            else finish_with(c, c->iter, STOP_RESIDUAL);
            return;
        }
        const int64_t m = c->dim;
        c->beta_restart = beta;
        for (int64_t i = 0; i <= m; ++i) c->g[i] = 0.0;
        for (int64_t i = 0; i < m; ++i) c->cs[i] = c->sn[i] = 0.0;
        for (int64_t i = 0; i < m * m; ++i) c->R[i] = 0.0;
        c->g[0] = beta;
        c->j = 0;
        c->cycle_end = 0;
        c->finish = 0;
        c->cycle += 1;
    }
};

// v0 = (1 / beta) r  (copy + scal(1.0 / beta))
template <class V>
struct GmFirstBasis : SkipNone {
    using value_type = V;
    const V *r;
    V *v0;
    double inv_beta;
    __device__ __forceinline__ void prepare(const Ctl *c) { inv_beta = 1.0 / c->beta_restart; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        auto R = ldp<W>(r, i);
#pragma unroll
        for (int w = 0; w < W; ++w) R.v[w] = scal_e(inv_beta, R.v[w]);
        stp<W>(v0, i, R);
    }
};

// z = M v_j
template <class V>
struct GmPrecond : SkipCycleEnd {
    using value_type = V;
    const V *vj, *inv;
    V *z;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        auto Z = ldp<W>(vj, i);
        const auto D = ldp<W>(inv, i);
#pragma unroll
        for (int w = 0; w < W; ++w) Z.v[w] = vmul(Z.v[w], D.v[w]);
        stp<W>(z, i, Z);
    }
};

// w = A z with h_0j = v_0.w fused
struct GmH0Fin {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->cycle_end != 0; }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const { c->hcol[0] = tot[0]; }
};

// w = A (M v_j) with the Jacobi product M v_j (np.multiply, precond.py:62) evaluated at
// each gathered column instead of a separate z = M v_j pass: bitwise the same w and
// h_0j, one launch and two vector passes fewer per inner iteration (row-owning formats)
template <class V>
struct EpiGmPrecondGather : EpiSolver<V, 1, GmH0Fin> {
    const V *vj, *inv;
    __device__ __forceinline__ V gather(int64_t c) const { return vmul(__ldg(vj + c), __ldg(inv + c)); }
};

// one MGS step: w -= h_i v_i, then h_{i+1} = v_{i+1}.w (single pass)
template <class V>
struct GmMgsStep : SkipCycleEnd {
    using value_type = V;
    const V *vi, *vnext;
    V *w;
    int i;
    double h;
    __device__ __forceinline__ void prepare(const Ctl *c) { h = c->hcol[i]; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t e, double (&part)[1]) const {
        const auto VI = ldp<W>(vi, e), VN = ldp<W>(vnext, e);
        auto Wv = ldp<W>(w, e);
#pragma unroll
        for (int k = 0; k < W; ++k) {
            Wv.v[k] = axpy_e(-h, VI.v[k], Wv.v[k]);
            part[0] = addd(part[0], mulp(VN.v[k], Wv.v[k]));
        }
        stp<W>(w, e, Wv);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const { c->hcol[i + 1] = tot[0]; }
};

// givens_rotation (solvers.py:138-143)
__device__ __forceinline__ void givens(double a, double b, double &c, double &s, double &r) {
    if (a == 0.0 && b == 0.0) {
        c = 1.0;
        s = 0.0;
        r = 0.0;
        return;
    }
    r = hypot(a, b);
    c = __ddiv_rn(a, r);
    s = __ddiv_rn(b, r);
}

// last MGS step of column j: w -= h_jj v_j, ||w||, then the reference's per-inner-iteration
// scalar work: rotations, estimate |g_{j+1}|, criteria, happy breakdown, cycle end
template <class V>
struct GmMgsLast : SkipCycleEnd {
    using value_type = V;
    const V *vj;
    V *w;
    int j;
    double h;
    __device__ __forceinline__ void prepare(const Ctl *c) { h = c->hcol[j]; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t e, double (&part)[1]) const {
        const auto VJ = ldp<W>(vj, e);
        auto Wv = ldp<W>(w, e);
#pragma unroll
        for (int k = 0; k < W; ++k) {
            Wv.v[k] = axpy_e(-h, VJ.v[k], Wv.v[k]);
            part[0] = addd(part[0], mulp(Wv.v[k], Wv.v[k]));
        }
        stp<W>(w, e, Wv);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const {
        double *hc = c->hcol;
        const double hnorm = sqrt(tot[0]);
        hc[j + 1] = hnorm;
        for (int i = 0; i <= j + 1; ++i)
            if (!isfinite(hc[i])) {
                c->status = ST_NUMERIC;
                c->status_iter = c->iter + 1;
                stop_loop(c);
                return;
            }
        for (int i = 0; i < j; ++i) {
            const double hi = hc[i], hi1 = hc[i + 1];
            hc[i] = __dadd_rn(__dmul_rn(c->cs[i], hi), __dmul_rn(c->sn[i], hi1));
            hc[i + 1] = __dadd_rn(__dmul_rn(-c->sn[i], hi), __dmul_rn(c->cs[i], hi1));
        }
        double cr, sr, rr;
        givens(hc[j], hc[j + 1], cr, sr, rr);
        c->cs[j] = cr;
        c->sn[j] = sr;
        hc[j] = rr;
        const int64_t m = c->dim;
        for (int i = 0; i <= j; ++i) c->R[i * m + j] = hc[i];
        c->g[j + 1] = __dmul_rn(-sr, c->g[j]);
        c->g[j] = __dmul_rn(cr, c->g[j]);
        const double est = fabs(c->g[j + 1]);
        if (!isfinite(est)) {
            c->status = ST_NUMERIC;
            c->status_iter = c->iter + 1;
            stop_loop(c);
            return;
        }
        const int64_t total = c->iter + 1;
        c->iter = total;
        record(c, total, est);
        const int reason = check_criteria(c, total, est, c->bnorm);
        const bool happy = hnorm <= __dmul_rn(1e-30, c->bnorm);
        c->hnorm = hnorm;
        if (reason != STOP_NONE || happy || j + 1 == m) {
            c->cycle_end = 1;
            c->k = j + 1;
            c->finish = reason != STOP_NONE;
            c->stop_reason = reason;
        } else {
            c->j = j + 1;
        }
    }
};

// v_{j+1} = (1 / ||w||) w
template <class V>
struct GmNextBasis : SkipCycleEnd {
    using value_type = V;
    const V *w;
    V *vn;
    double inv_h;
    __device__ __forceinline__ void prepare(const Ctl *c) { inv_h = 1.0 / c->hnorm; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t e, double (&)[1]) const {
        auto Wv = ldp<W>(w, e);
#pragma unroll
        for (int k = 0; k < W; ++k) Wv.v[k] = scal_e(inv_h, Wv.v[k]);
        stp<W>(vn, e, Wv);
    }
};

// _back_substitute (solvers.py:301-308)
struct GmBackSub {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->cycle_end == 0; }
    __device__ __forceinline__ void run(Ctl *c) const {
        const int k = c->k;
        const int64_t m = c->dim;
        for (int i = k - 1; i >= 0; --i) {
            double acc = c->g[i];
            for (int q = i + 1; q < k; ++q) acc = __dsub_rn(acc, __dmul_rn(c->R[i * m + q], c->y[q]));
            c->y[i] = __ddiv_rn(acc, c->R[i * m + i]);
        }
    }
};

// _gmres_update: zacc = sum_i axpy(y_i, v_i, zacc) (sequential, rounded per step);
// x += M zacc; then finish if a criterion fired
template <class V, int MAXK>
struct GmUpdate : SkipUnlessCycleEnd {
    using value_type = V;
    const V *basis;
    size_t vstride;  // elements between consecutive basis vectors
    const V *inv;
    V *x;
    const double *y;
    int k;
    __device__ __forceinline__ void prepare(const Ctl *c) {
        k = c->k;
        y = c->y;
    }
    template <int W>
    __device__ __forceinline__ void elem(int64_t e, double (&)[1]) const {
        Pk<V, W> acc;
#pragma unroll
        for (int w = 0; w < W; ++w) acc.v[w] = (V)0;
        for (int i = 0; i < k; ++i) {
            const auto Vi = ldp<W>(basis + (size_t)i * vstride, e);
            const double yi = y[i];
#pragma unroll
            for (int w = 0; w < W; ++w) acc.v[w] = axpy_e(yi, Vi.v[w], acc.v[w]);
        }
        const auto D = ldp_or_one<W>(inv, e);
        auto X = ldp<W>(x, e);
#pragma unroll
        for (int w = 0; w < W; ++w) X.v[w] = axpy_e(1.0, inv ? vmul(acc.v[w], D.v[w]) : acc.v[w], X.v[w]);
        stp<W>(x, e, X);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&)[1]) const {
        if (c->finish) finish_with(c, c->iter, c->stop_reason);
    }
};

// ILU / IC right preconditioning (_gmres_update with m.apply, solvers.py:311-319): the
// accumulated V_k y goes to `acc`, two triangular sweeps form dx, then x += dx.
template <class V>
struct GmAccum : SkipUnlessCycleEnd {
    using value_type = V;
    const V *basis;
    size_t vstride;
    V *acc_out;
    const double *y;
    int k;
    __device__ __forceinline__ void prepare(const Ctl *c) {
        k = c->k;
        y = c->y;
    }
    template <int W>
    __device__ __forceinline__ void elem(int64_t e, double (&)[1]) const {
        Pk<V, W> acc;
#pragma unroll
        for (int w = 0; w < W; ++w) acc.v[w] = (V)0;
        for (int i = 0; i < k; ++i) {
            const auto Vi = ldp<W>(basis + (size_t)i * vstride, e);
            const double yi = y[i];
#pragma unroll
            for (int w = 0; w < W; ++w) acc.v[w] = axpy_e(yi, Vi.v[w], acc.v[w]);
        }
        stp<W>(acc_out, e, acc);
    }
};

template <class V>
struct GmAddX : SkipUnlessCycleEnd {  // x = axpy(1.0, dx, x); then finish if a criterion fired
    using value_type = V;
    const V *dx;
    V *x;
    template <int W>
    __device__ __forceinline__ void elem(int64_t e, double (&)[1]) const {
        const auto D = ldp<W>(dx, e);
        auto X = ldp<W>(x, e);
#pragma unroll
        for (int w = 0; w < W; ++w) X.v[w] = axpy_e(1.0, D.v[w], X.v[w]);
        stp<W>(x, e, X);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&)[1]) const {
        if (c->finish) finish_with(c, c->iter, c->stop_reason);
    }
};

}  // namespace sb
