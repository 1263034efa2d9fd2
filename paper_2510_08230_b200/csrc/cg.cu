// cg.cu -- preconditioned CG on the device (solvers.py:188-224): 3 fused kernels per iteration.
#include <cmath>
#include <atomic>
#include <cstdlib>

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

// ---------------------------------------------------------------- fused-direction CG
// Two kernels per iteration instead of three.  Iteration k's SpMV evaluates the search
// direction p_k = z + beta p_{k-1} (scal then axpy, the reference's exact rounding) on
// the fly at every gathered column, so p_k is never a separate pass: the epilogue
// stores q = A p_k and the row's own p_k (ping-pong buffers: iteration k reads
// buf[(k-1)&1] and writes buf[k&1], so no CTA overwrites a value another CTA still
// gathers), accumulates p_k.q, and applies the PREVIOUS iteration's x += alpha p_{k-1}
// (deferred from the update kernel, which then streams only r, q, M: r -= alpha q,
// z = M r, r.r, r.z).  The x update of the final iteration is applied after the loop
// (cg_xfinal_kernel).  Per iteration: A + 11 V n bytes instead of A + 13 V n, and one
// launch fewer; every value is bitwise what the three-kernel loop computes.
template <class V, bool DeferX>
struct EpiCgFused {
    static constexpr int N = 1;
    static constexpr int kMinThreadsPerSM = 1024;
    V *q, *pnew, *x;
    const V *z, *pold;
    Ctl *ctl;
    double *partials;
    double beta, alpha;
    int first;
    __device__ __forceinline__ bool skip() const { return loop_done(ctl); }
    __device__ __forceinline__ void prepare() {
        // read before any CTA of this launch can finish (the last CTA, which rewrites
        // iter / alpha, starts its finalisation only after every CTA has arrived)
        first = ctl->iter == 0;
        beta = ctl->beta;
        alpha = ctl->alpha;
    }
    __device__ __forceinline__ V gather(int64_t c) const {
        const V zc = __ldg(z + c);
        return first ? zc : axpy_e(1.0, zc, scal_e(beta, __ldg(pold + c)));
    }
    __device__ __forceinline__ void row(int64_t i, double acc, double (&part)[N]) const {
        const V qi = (V)acc;
        q[i] = qi;
        const V pi = gather(i);
        pnew[i] = pi;
        if (DeferX && !first) x[i] = axpy_e(alpha, __ldg(pold + i), x[i]);
        part[0] = addd(part[0], mulp(pi, qi));
    }
    __device__ __forceinline__ void finish(double (&part)[N]) const {
        double tot[N];
        if (grid_reduce<N>(part, partials, &ctl->ticket[0], tot) && threadIdx.x == 0) {
            if (DeferX) ctl->xpend = 0;  // x += alpha_{k-1} p_{k-1} applied by every CTA above
            CgPqFin{}.last(ctl, tot);
        }
    }
};

// r -= alpha q; z = M r; dots r.r, r.z -> criteria, beta (x deferred to the next SpMV)
template <class V>
struct CgUpdateR : SkipNone {
    using value_type = V;
    const V *q, *inv;
    V *r, *z;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[2]) const {
        const auto Q = ldp<W>(q, i), D = ldp_or_one<W>(inv, i);
        auto R = ldp<W>(r, i);
        Pk<V, W> Z;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-alpha, Q.v[w], R.v[w]);
            Z.v[w] = inv ? vmul(R.v[w], D.v[w]) : R.v[w];
            part[0] = addd(part[0], mulp(R.v[w], R.v[w]));
            part[1] = addd(part[1], mulp(R.v[w], Z.v[w]));
        }
        stp<W>(r, i, R);
        stp<W>(z, i, Z);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[2]) const {
        c->xpend = 1;  // this iteration's x += alpha p is owed (next SpMV or cg_xfinal_kernel)
        CgUpdate<V>{}.last(c, tot);
    }
};

// after the loop: the deferred x += alpha_k p_k of the last completed iteration k
template <class V>
__global__ void __launch_bounds__(256) cg_xfinal_kernel(int64_t n, const Ctl *c, const V *p0,
                                                        const V *p1, V *x) {
    if (!c->xpend) return;
    const V *p = (c->iter & 1) ? p1 : p0;
    const double alpha = c->alpha;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = axpy_e(alpha, p[i], x[i]);
}

// fused-direction loop on (default) / off (the three-kernel loop; A/B and parity tests)
// 2 = x update deferred into the next SpMV as well (A + 11 V n)
static std::atomic<int> g_cg_fused{[] {
    const char *e = getenv("SPARSEB200_CG_FUSED");
    return e ? atoi(e) : 1;
}()};
inline bool cg_fused_enabled() { return g_cg_fused.load() != 0; }

template <class V, class I>
sb_status cg_solve(const SolveArgs &a) {
    sb_error *err = a.err;
    int64_t n = 0;
    sb_status s = check_solve_args<V>(a, n);
    if (s != SB_OK) return s;
    const int64_t cap = a.log->history_cap;
    SolverWs w = carve_ws(a.ws, SB_SOLVER_CG, sizeof(V), n, 0, cap);
    V *r = ws_vec<V>(w, 0), *z = ws_vec<V>(w, 1), *p = ws_vec<V>(w, 2), *q = ws_vec<V>(w, 3),
      *t = ws_vec<V>(w, 4);
    const V *b = (const V *)a.b->data, *inv = (const V *)a.inv;
    V *x = (V *)a.x->data;
    Ctl *ctl = w.ctl;
    double *part = w.partials;
    const sb_matrix M = *a.A;
    Ctl h = initial_ctl(*a.crit, w, cap);
    LoopSpec spec;
    spec.key = "cg" + std::to_string(sizeof(V)) + std::to_string(sizeof(I)) + "|" + matrix_key(M) +
               ptr_key({a.inv, b, x, a.ws, w.vecs, w.hist, w.small});
    spec.poll_chunk = 8;
    spec.hot_base = r;  // r, z, p, q, t are contiguous in the workspace
    spec.hot_bytes = 5 * w.vec_bytes;
    const bool fused = cg_fused_enabled() && matrix_row_owning(M);
    spec.setup = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(M, x, 1, t, 1, EpiStore<V>{t, 1}, st);
        if (e != cudaSuccess) return e;
        return launch_ew<3>(n, ctl, part, CgInit<V>{{}, b, t, inv, r, z, fused ? nullptr : p}, st);
    };
    if (fused) {
        // p ping-pongs between p (buf 0) and t (buf 1; free once setup consumed A x0);
        // one body = an odd and an even iteration, so the buffer roles stay fixed
        spec.key += "|fused";
        spec.poll_chunk = 4;
        const bool defer_x = g_cg_fused.load() == 2;
        spec.key += defer_x ? "x" : "";
        spec.body = [=](cudaStream_t st) -> cudaError_t {
            for (int h = 0; h < 2; ++h) {
                V *pold = h == 0 ? p : t, *pnew = h == 0 ? t : p;
                cudaError_t e;
                if (defer_x) {
                    e = matrix_apply<V, I>(
                        M, pold, 1, q, 1, EpiCgFused<V, true>{q, pnew, x, z, pold, ctl, part, 0.0, 0.0, 0}, st);
                    if (e != cudaSuccess) return e;
                    e = launch_ew<2>(n, ctl, part, CgUpdateR<V>{{}, q, inv, r, z, 0.0}, st);
                } else {
                    e = matrix_apply<V, I>(
                        M, pold, 1, q, 1, EpiCgFused<V, false>{q, pnew, x, z, pold, ctl, part, 0.0, 0.0, 0}, st);
                    if (e != cudaSuccess) return e;
                    e = launch_ew<2>(n, ctl, part, CgUpdate<V>{{}, pnew, q, inv, x, r, z, 0.0}, st);
                }
                if (e != cudaSuccess) return e;
            }
            return cudaSuccess;
        };
        if (defer_x)
            spec.finish = [=](cudaStream_t st) -> cudaError_t {
                cg_xfinal_kernel<V><<<solver_grid(), 256, 0, st>>>(n, ctl, p, t, x);
                return cudaGetLastError();
            };
        s = run_loop(spec, ctl, h, a.st, err);
        if (s != SB_OK) return s;
        return finish_log(h, a, w);
    }
    spec.body = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(
            M, p, 1, q, 1, EpiSolver<V, 1, CgPqFin>{q, p, nullptr, ctl, part, CgPqFin{}}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<2>(n, ctl, part, CgUpdate<V>{{}, p, q, inv, x, r, z, 0.0}, st);
        if (e != cudaSuccess) return e;
        return launch_ew<0>(n, ctl, part, CgDirection<V>{{}, z, p, 0.0}, st);
    };
    s = run_loop(spec, ctl, h, a.st, err);
    if (s != SB_OK) return s;
    return finish_log(h, a, w);
}


}  // namespace sb

using namespace sb;

extern "C" {

void sb_set_cg_fused(int mode) { g_cg_fused = mode; }

#define SB_DEFS(V, VN, I, IN) \
    sb_status sb_cg_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,                    \
                                      const sb_dense *b, sb_dense *x, const sb_criteria *crit,     \
                                      void *workspace, sb_log *log, sb_stream_t stream,            \
                                      sb_error *err) {                                             \
        SB_GUARD_BEGIN                                                                             \
        return cg_solve<V, I>(SolveArgs{a, inv_diag, b, x, crit, 0, workspace, log,                \
                                        as_stream(stream), err});                                  \
        SB_GUARD_END                                                                               \
    }

SB_DEFS(float, float, int32_t, i32)
SB_DEFS(float, float, int64_t, i64)
SB_DEFS(double, double, int32_t, i32)
SB_DEFS(double, double, int64_t, i64)

}  // extern "C"
