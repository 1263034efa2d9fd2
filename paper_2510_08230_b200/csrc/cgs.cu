// cgs.cu -- CGS on the device (solvers.py:231-284) with the residual update fused into the SpMV.
#include <cmath>

#include "solver_common.cuh"
#include "trisolve.cuh"

namespace sb {

// ================================================================ CGS (solvers.py:231-284)
// u = r, p = u (first) | u = r + beta q; p = u + beta (q + beta p) with the reference's
// copy/scal/axpy rounding; phat = M p
template <class V>
struct CgsDirection : SkipNone {
    using value_type = V;
    const V *r, *q, *inv;
    V *u, *p, *ph;
    double beta;
    bool first;
    __device__ __forceinline__ void prepare(const Ctl *c) {
        beta = c->beta;
        first = c->iter == 0;
    }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        const auto R = ldp<W>(r, i), D = ldp_or_one<W>(inv, i);
        Pk<V, W> U, P, PH;
        if (first) {
            U = R;
            P = R;
        } else {
            const auto Q = ldp<W>(q, i);
            P = ldp<W>(p, i);
            const double b2 = __dmul_rn(beta, beta);
#pragma unroll
            for (int w = 0; w < W; ++w) {
                U.v[w] = axpy_e(1.0, R.v[w], scal_e(beta, Q.v[w]));
                P.v[w] = axpy_e(1.0, U.v[w], axpy_e(beta, Q.v[w], scal_e(b2, P.v[w])));
            }
        }
        stp<W>(u, i, U);
        stp<W>(p, i, P);
        if (!ph) return;
#pragma unroll
        for (int w = 0; w < W; ++w) PH.v[w] = inv ? vmul(P.v[w], D.v[w]) : P.v[w];
        stp<W>(ph, i, PH);
    }
};

// q = u - alpha v; uhat = M (u + q); x += alpha uhat
template <class V>
struct CgsQ : SkipNone {
    using value_type = V;
    const V *u, *v, *inv;
    V *q, *uh, *x;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        const auto U = ldp<W>(u, i), Vv = ldp<W>(v, i), D = ldp_or_one<W>(inv, i);
        Pk<V, W> Q, UH;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            Q.v[w] = axpy_e(-alpha, Vv.v[w], U.v[w]);
            const V uq = axpy_e(1.0, Q.v[w], U.v[w]);
            UH.v[w] = inv ? vmul(uq, D.v[w]) : uq;
        }
        stp<W>(q, i, Q);
        stp<W>(uh, i, UH);
        if (!x) return;  // tri path: uh holds u + q, M is applied by the sweeps
        auto X = ldp<W>(x, i);
#pragma unroll
        for (int w = 0; w < W; ++w) X.v[w] = axpy_e(alpha, UH.v[w], X.v[w]);
        stp<W>(x, i, X);
    }
};

// SpMV epilogue: t = A uhat row by row, immediately r -= alpha t with dots r.r and rs.r
template <class V>
struct EpiCgsResidual {
    static constexpr int N = 2;
    V *t, *r;
    const V *rs;
    Ctl *ctl;
    double *partials;
    __device__ __forceinline__ bool skip() const { return loop_done(ctl); }
    __device__ __forceinline__ void row(int64_t i, double acc, double (&part)[N]) const {
        const V ti = (V)acc;
        t[i] = ti;
        const V ri = axpy_e(-ctl->alpha, ti, r[i]);
        r[i] = ri;
        part[0] = addd(part[0], mulp(ri, ri));
        part[1] = addd(part[1], mulp(rs[i], ri));
    }
    __device__ __forceinline__ void finish(double (&part)[N]) const {
        double tot[N];
        if (grid_reduce<N>(part, partials, &ctl->ticket[0], tot) && threadIdx.x == 0) last(ctl, tot);
    }
    __device__ __forceinline__ static void last(Ctl *c, const double (&tot)[2]) {
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
        const double rho = tot[1];
        if (!isfinite(rho) || fabs(rho) <= kBreakdownRtol * c->shadow_norm * rnorm) {
            breakdown(c, it + 1);
            return;
        }
        c->rho_prev = c->rho;
        c->rho = rho;
        c->beta = rho / c->rho_prev;
    }
};

// the same update as a separate pass for row-splitting formats (t already written)
template <class V>
struct CgsResidualPass : SkipNone {
    using value_type = V;
    const V *t, *rs;
    V *r;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[2]) const {
        const auto T = ldp<W>(t, i), RS = ldp<W>(rs, i);
        auto R = ldp<W>(r, i);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-alpha, T.v[w], R.v[w]);
            part[0] = addd(part[0], mulp(R.v[w], R.v[w]));
            part[1] = addd(part[1], mulp(RS.v[w], R.v[w]));
        }
        stp<W>(r, i, R);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[2]) const {
        EpiCgsResidual<V>::last(c, tot);
    }
};

// x += alpha uhat (tri path: uhat came from the sweeps)
template <class V>
struct XAxpyAlpha : SkipNone {
    using value_type = V;
    const V *uh;
    V *x;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        const auto UH = ldp<W>(uh, i);
        auto X = ldp<W>(x, i);
#pragma unroll
        for (int w = 0; w < W; ++w) X.v[w] = axpy_e(alpha, UH.v[w], X.v[w]);
        stp<W>(x, i, X);
    }
};

template <class V, class I>
sb_status tri_precond_check(const sb_tri_precond &m, sb_error *err, cudaStream_t st);

template <class V, class I>
sb_status cgs_solve(const SolveArgs &a) {
    sb_error *err = a.err;
    int64_t n = 0;
    sb_status s = check_solve_args<V>(a, n);
    if (s != SB_OK) return s;
    const int64_t cap = a.log->history_cap;
    SolverWs w = carve_ws(a.ws, SB_SOLVER_CGS, sizeof(V), n, 0, cap);
    V *r = ws_vec<V>(w, 0), *rs = ws_vec<V>(w, 1), *u = ws_vec<V>(w, 2), *p = ws_vec<V>(w, 3),
      *q = ws_vec<V>(w, 4), *v = ws_vec<V>(w, 5), *uh = ws_vec<V>(w, 6), *ph = ws_vec<V>(w, 7),
      *t = ws_vec<V>(w, 8);
    const V *b = (const V *)a.b->data, *inv = (const V *)a.inv;
    V *x = (V *)a.x->data;
    Ctl *ctl = w.ctl;
    double *part = w.partials;
    const sb_matrix M = *a.A;
    const bool fused = matrix_row_owning(M);
    const sb_tri_precond *tri = a.tri;
    if (tri) {
        s = tri_precond_check<V, I>(*tri, err, a.st);
        if (s != SB_OK) return s;
    }
    const TriWs tw = tri ? carve_tri_ws(tri->workspace, n) : TriWs{};
    // z = U^{-1} L^{-1} in through the scratch vector (skipped once the loop is done)
    auto precond = [=](const V *in, V *scratch, V *out, cudaStream_t st) -> cudaError_t {
        cudaError_t e = launch_trsv<V, I>(*tri->l, true, tri->l_unit != 0, in, 1, scratch, 1, tw, ctl,
                                          TRI_SKIP_DONE, st);
        if (e != cudaSuccess) return e;
        return launch_trsv<V, I>(*tri->u, false, false, scratch, 1, out, 1, tw, ctl, TRI_SKIP_DONE, st);
    };
    Ctl h = initial_ctl(*a.crit, w, cap);
    LoopSpec spec;
    spec.key = "cgs" + std::to_string(sizeof(V)) + std::to_string(sizeof(I)) + "|" + matrix_key(M) +
               ptr_key({a.inv, b, x, a.ws, w.vecs, w.hist, w.small});
    if (tri)
        spec.key += "|tri" + std::to_string(tri->l_unit) +
                    ptr_key({tri->l->row_ptrs, tri->l->values, tri->u->row_ptrs, tri->u->values, tri->workspace});
    spec.poll_chunk = 8;
    spec.setup = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(M, x, 1, t, 1, EpiStore<V>{t, 1}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<2>(n, ctl, part, ShadowInit<V>{{}, b, t, r, rs}, st);
        if (e != cudaSuccess) return e;
        // CGS keeps rho_prev = 0 until the first iteration ends (solvers.py:240)
        return cudaSuccess;
    };
    spec.body = [=](cudaStream_t st) -> cudaError_t {
        // solvers.py:261 phat = M p (tri: sweeps p -> t -> phat; t is free until A uhat)
        cudaError_t e = launch_ew<0>(n, ctl, part, CgsDirection<V>{{}, r, q, inv, u, p, tri ? nullptr : ph, 0, false}, st);
        if (e != cudaSuccess) return e;
        if (tri && (e = precond(p, t, ph, st)) != cudaSuccess) return e;
        e = matrix_apply<V, I>(M, ph, 1, v, 1, EpiSolver<V, 1, BiSigmaFin>{v, rs, nullptr, ctl, part, {}}, st);
        if (e != cudaSuccess) return e;
        if (tri) {  // :269-274 q = u - alpha v; uq = u + q (in t); uhat = M uq; x += alpha uhat
            e = launch_ew<0>(n, ctl, part, CgsQ<V>{{}, u, v, nullptr, q, t, nullptr, 0}, st);
            if (e != cudaSuccess) return e;
            if ((e = precond(t, ph, uh, st)) != cudaSuccess) return e;
            e = launch_ew<0>(n, ctl, part, XAxpyAlpha<V>{{}, uh, x, 0}, st);
        } else {
            e = launch_ew<0>(n, ctl, part, CgsQ<V>{{}, u, v, inv, q, uh, x, 0}, st);
        }
        if (e != cudaSuccess) return e;
        if (fused) return matrix_apply<V, I>(M, uh, 1, t, 1, EpiCgsResidual<V>{t, r, rs, ctl, part}, st);
        e = matrix_apply<V, I>(M, uh, 1, t, 1, EpiSolverStore<V, NeverSkip>{t, ctl, {}}, st);
        if (e != cudaSuccess) return e;
        return launch_ew<2>(n, ctl, part, CgsResidualPass<V>{{}, t, rs, r, 0}, st);
    };
    s = run_loop(spec, ctl, h, a.st, err);
    if (s != SB_OK) return s;
    return finish_log(h, a, w);
}

}  // namespace sb

using namespace sb;

extern "C" {

#define SB_DEFS(V, VN, I, IN) \
    sb_status sb_cgs_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,                   \
                                       const sb_dense *b, sb_dense *x, const sb_criteria *crit,    \
                                       void *workspace, sb_log *log, sb_stream_t stream,           \
                                       sb_error *err) {                                            \
        SB_GUARD_BEGIN                                                                             \
        return cgs_solve<V, I>(SolveArgs{a, inv_diag, b, x, crit, 0, workspace, log,               \
                                         as_stream(stream), err});                                 \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_cgs_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,            \
                                           const sb_dense *b, sb_dense *x, const sb_criteria *crit,\
                                           void *workspace, sb_log *log, sb_stream_t stream,       \
                                           sb_error *err) {                                        \
        SB_GUARD_BEGIN                                                                             \
        SolveArgs sa{a, nullptr, b, x, crit, 0, workspace, log, as_stream(stream), err};           \
        sa.tri = m;                                                                                \
        return cgs_solve<V, I>(sa);                                                                \
        SB_GUARD_END                                                                               \
    }

SB_DEFS(float, float, int32_t, i32)
SB_DEFS(float, float, int64_t, i64)
SB_DEFS(double, double, int32_t, i32)
SB_DEFS(double, double, int64_t, i64)

}  // extern "C"
