// solver_common.cuh -- device-resident Krylov solver state and the loop runner.
//
// Every scalar of the reference's host loop (solvers.py:188-399) lives in a device
// control block `Ctl`: the kernels compute dots with fused deterministic grid
// reductions and the LAST block of each reduction evaluates the reference's scalar
// logic (breakdown tests, check_criteria, Givens rotations) in one thread.  The
// host is therefore out of the loop: one iteration (GMRES: one restart cycle) is
// captured once into the body of a CUDA-graph WHILE conditional node, and the
// kernel that decides to stop clears the condition with cudaGraphSetConditional.
// A host-polled fallback (chunks of iterations, done flag read back every chunk)
// exists for environments without conditional nodes.
#pragma once

#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "capi_util.cuh"
#include "spmv_launch.cuh"

namespace sb {

constexpr double kBreakdownRtol = 1e-30;  // solvers.py:46
enum { STOP_NONE = -1, STOP_RESIDUAL = 0, STOP_MAX_ITERS = 1 };
enum { ST_OK = 0, ST_BREAKDOWN = 1, ST_NUMERIC = 2 };

struct Ctl {
    // criteria (solvers.py:52-76 reduced to OR semantics)
    int64_t max_iters;
    int32_t has_rf;
    int32_t pad0;
    double rf;
    // state
    int64_t iter;          // iterations executed (GMRES: total inner iterations)
    int32_t done;          // solve finished (any reason)
    int32_t status;        // ST_*
    int32_t stop_reason;   // STOP_*
    int32_t converged;
    int64_t status_iter;   // BreakdownError.iteration
    int64_t hist_len;
    int64_t hist_cap;
    double *hist;          // device history (one residual per criteria check)
    unsigned long long cond;  // cudaGraphConditionalHandle of the running loop, 0 if polled
    unsigned ticket[4];
    // scalars
    double bnorm, rnorm, rz, alpha, beta, rho, rho_prev, omega, sigma, snorm, shadow_norm;
    int32_t early;         // BiCGSTAB: ||s|| met the residual criterion
    int32_t exact;         // initial guess already exact (_exact_log)
    // GMRES (pointers into the workspace, sized by krylov_dim)
    int64_t dim;
    int32_t j, k, cycle_end, finish;
    double *hcol, *g, *cs, *sn, *y, *R;  // R: dim x dim, row-major
    double hnorm, beta_restart;
    int64_t cycle;
    double dot[24];  // row-partitioned solves: local dot totals, reduced across ranks in place
    unsigned long long tphase[10];  // persistent CG: CTA 0's ns per phase, summed over iterations
    unsigned long long barrier;    // persistent CG: grid-barrier arrivals (0 at every solve start)
};
static_assert(sizeof(Ctl) <= 4096, "control block must fit kCtlBytes");

__device__ __forceinline__ void stop_loop(Ctl *c) {
    c->done = 1;
    if (c->cond) cudaGraphSetConditional((cudaGraphConditionalHandle)c->cond, 0);
}

// Entry test of every loop kernel: a finished solve turns the kernel into a no-op, and
// (inside the graph) clears the WHILE condition -- this also ends a loop whose setup
// finished the solve (exact initial guess) before the graph was launched.  ctl->cond
// is only non-zero while the graph runs, so setup kernels never touch the handle.
__device__ __forceinline__ bool loop_done(const Ctl *c) {
    if (!c->done) return false;
    if (c->cond && blockIdx.x == 0 && threadIdx.x == 0)
        cudaGraphSetConditional((cudaGraphConditionalHandle)c->cond, 0);
    return true;
}

// solvers.check_criteria (solvers.py:121-135): residual wins ties
__device__ __forceinline__ int check_criteria(const Ctl *c, int64_t it, double res, double bnorm) {
    if (c->has_rf) {
        const double thr = bnorm > 0 ? __dmul_rn(c->rf, bnorm) : c->rf;
        if (res <= thr) return STOP_RESIDUAL;
    }
    if (it >= c->max_iters) return STOP_MAX_ITERS;
    return STOP_NONE;
}

__device__ __forceinline__ void record(Ctl *c, int64_t it, double res) {
    if (it - 1 < c->hist_cap) c->hist[it - 1] = res;
    c->hist_len = it;
}

__device__ __forceinline__ void finish_with(Ctl *c, int64_t it, int reason) {
    c->iter = it;
    c->converged = reason == STOP_RESIDUAL;
    c->stop_reason = reason;
    stop_loop(c);
}

__device__ __forceinline__ void breakdown(Ctl *c, int64_t it) {
    c->status = ST_BREAKDOWN;
    c->status_iter = it;
    c->iter = it;
    stop_loop(c);
}

// ---------------------------------------------------------------- elementwise + reduce
// Packs of W consecutive elements moved with one 16-byte (or 8-byte) access; all solver
// vectors are 16-byte aligned (workspace vectors are 256-byte aligned; b / x / inv are
// checked by check_solve_args).
template <class V, int W>
struct Pk {
    V v[W];
};
template <int W, class V>
__device__ __forceinline__ Pk<V, W> ldp(const V *p, int64_t i) {
    Pk<V, W> r;
    if constexpr (W * sizeof(V) == 16) {
        const int4 t = *reinterpret_cast<const int4 *>(p + i);
        memcpy(&r, &t, 16);
    } else if constexpr (W * sizeof(V) == 8) {
        const int2 t = *reinterpret_cast<const int2 *>(p + i);
        memcpy(&r, &t, 8);
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w) r.v[w] = p[i + w];
    }
    return r;
}
template <int W, class V>
__device__ __forceinline__ Pk<V, W> ldp_or_one(const V *p, int64_t i) {  // nullptr -> identity
    if (p) return ldp<W>(p, i);
    Pk<V, W> r;
#pragma unroll
    for (int w = 0; w < W; ++w) r.v[w] = (V)1;
    return r;
}
template <int W, class V>
__device__ __forceinline__ void stp(V *p, int64_t i, const Pk<V, W> &r) {
    if constexpr (W * sizeof(V) == 16) {
        int4 t;
        memcpy(&t, &r, 16);
        *reinterpret_cast<int4 *>(p + i) = t;
    } else if constexpr (W * sizeof(V) == 8) {
        int2 t;
        memcpy(&t, &r, 8);
        *reinterpret_cast<int2 *>(p + i) = t;
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w) p[i + w] = r.v[w];
    }
}

// One grid-stride pass over n rows in packs of W (tail with W = 1) applying
// Op::elem<W>, with N fused fp64 reductions finalised (deterministically) in the last
// block by Op::last.  Fixed grid -> fixed summation order.
inline int solver_grid() { return device_info().sms * 8; }

// partial type of an elementwise op's fused dots: double, or CAcc if the op declares
// `using part_type = CAcc;` (compensated, see common.cuh)
template <class O, class = void>
struct op_part {
    using type = double;
};
template <class O>
struct op_part<O, std::void_t<typename O::part_type>> {
    using type = typename O::part_type;
};

template <int N, int W, class Op>
__global__ void __launch_bounds__(256) ew_kernel(int64_t n, Ctl *ctl, double *partials, Op op) {
    pdl_wait();
    pdl_trigger();
    if (loop_done(ctl) || op.skip(ctl)) return;
    op.prepare(ctl);
    typename op_part<Op>::type part[N > 0 ? N : 1] = {};
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t npk = n / W;
    for (int64_t k = gtid; k < npk; k += stride) op.template elem<W>(k * W, part);
    for (int64_t i = npk * W + gtid; i < n; i += stride) op.template elem<1>(i, part);
    if constexpr (N > 0) {
        double tot[N];
        if (grid_reduce<N>(part, partials, &ctl->ticket[0], tot) && threadIdx.x == 0) op.last(ctl, tot);
    } else {
        (void)part;
    }
}

template <int N, class Op>
cudaError_t launch_ew(int64_t n, Ctl *ctl, double *partials, const Op &op, cudaStream_t st) {
    constexpr int W = 16 / sizeof(typename Op::value_type);
    return launch_pdl(ew_kernel<N, W, Op>, solver_grid(), 256, 0, st, n, ctl, partials, op);
}

// single-thread scalar step (host-free control logic between passes)
template <class Op>
__global__ void scalar_kernel(Ctl *ctl, Op op) {
    if (loop_done(ctl) || op.skip(ctl)) return;
    op.run(ctl);
}

// SpMV epilogue for solvers: y = A b with N fused dots of y against per-row vectors,
// finalised by Fin::last in the last block; skipped when the loop is finished.
template <class V, int NDOT, class Fin>
struct EpiSolver {
    static constexpr int N = NDOT;
    V *y;
    const V *u0, *u1;  // dot partners: part[0] += u0.y (or y.y if u0 == nullptr), part[1] += u1.y
    Ctl *ctl;
    double *partials;
    Fin fin;
    __device__ __forceinline__ bool skip() const { return loop_done(ctl) || fin.skip(ctl); }
    __device__ __forceinline__ void row(int64_t i, double acc, double (&part)[N]) const {
        const V yi = (V)acc;
        y[i] = yi;
        part[0] = addd(part[0], u0 ? mulp(u0[i], yi) : mulp(yi, yi));
        if constexpr (N > 1) part[1] = addd(part[1], mulp(u1[i], yi));
    }
    __device__ __forceinline__ void finish(double (&part)[N]) const {
        double tot[N];
        if (grid_reduce<N>(part, partials, &ctl->ticket[0], tot) && threadIdx.x == 0) fin.last(ctl, tot);
    }
};

// EpiSolver with compensated fused dots
template <class V, int NDOT, class Fin>
struct EpiSolverC {
    static constexpr int N = NDOT;
    using part_type = CAcc;
    V *y;
    const V *u0, *u1;
    Ctl *ctl;
    double *partials;
    Fin fin;
    __device__ __forceinline__ bool skip() const { return loop_done(ctl) || fin.skip(ctl); }
    __device__ __forceinline__ void row(int64_t i, double acc, CAcc (&part)[N]) const {
        const V yi = (V)acc;
        y[i] = yi;
        cadd(part[0], u0 ? mulp(u0[i], yi) : mulp(yi, yi));
        if constexpr (N > 1) cadd(part[1], mulp(u1[i], yi));
    }
    __device__ __forceinline__ void finish(CAcc (&part)[N]) const {
        double tot[N];
        if (grid_reduce<N>(part, partials, &ctl->ticket[0], tot) && threadIdx.x == 0) fin.last(ctl, tot);
    }
};

// SpMV epilogue that only stores (skips when done / when Skip says so)
template <class V, class Skip>
struct EpiSolverStore {
    static constexpr int N = 1;
    V *y;
    Ctl *ctl;
    Skip sk;
    __device__ __forceinline__ bool skip() const { return loop_done(ctl) || sk.skip(ctl); }
    __device__ __forceinline__ void row(int64_t i, double acc, double (&)[N]) const { y[i] = (V)acc; }
    __device__ __forceinline__ void finish(double (&)[N]) const {}
};

struct NeverSkip {
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
};

// ---------------------------------------------------------------- workspace layout
struct SolverWs {
    Ctl *ctl;
    double *partials;  // 3 x kMaxGrid doubles
    double *hist;
    double *small;     // GMRES small dense arrays
    unsigned char *vecs;
    size_t vec_bytes;  // bytes per vector (256-aligned)
};

constexpr int64_t kMaxGrid = 8192;
constexpr size_t kCtlBytes = 4096;

inline size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

inline int solver_num_vectors(int solver, int64_t dim) {
    switch (solver) {
    case SB_SOLVER_CG: return 6;  // r z p q t + q1 (single-sync persistent loop)
    case SB_SOLVER_CGS: return 10;
    case SB_SOLVER_BICGSTAB: return 8;
    default: return (int)dim + 1 + 4;  // basis + r, t, z, w
    }
}

inline size_t gmres_small_bytes(int64_t dim) {
    return a256(sizeof(double) * (size_t)(4 * (dim + 2) + dim + dim * dim));
}

inline size_t solver_ws_bytes(int solver, int vbytes, int64_t n, int64_t dim, int64_t hist_cap) {
    const size_t vb = a256((size_t)vbytes * (size_t)(n > 0 ? n : 1));
    return kCtlBytes + a256(3 * kMaxGrid * sizeof(double)) + a256(sizeof(double) * (size_t)(hist_cap > 0 ? hist_cap : 1)) +
           (solver == SB_SOLVER_GMRES ? gmres_small_bytes(dim) : 0) +
           (size_t)solver_num_vectors(solver, dim) * vb;
}

inline SolverWs carve_ws(void *ws, int solver, int vbytes, int64_t n, int64_t dim, int64_t hist_cap) {
    unsigned char *p = (unsigned char *)ws;
    SolverWs w;
    w.ctl = (Ctl *)p;
    p += kCtlBytes;
    w.partials = (double *)p;
    p += a256(3 * kMaxGrid * sizeof(double));
    w.hist = (double *)p;
    p += a256(sizeof(double) * (size_t)(hist_cap > 0 ? hist_cap : 1));
    w.small = (double *)p;
    if (solver == SB_SOLVER_GMRES) p += gmres_small_bytes(dim);
    w.vecs = p;
    w.vec_bytes = a256((size_t)vbytes * (size_t)(n > 0 ? n : 1));
    return w;
}

template <class V>
inline V *ws_vec(const SolverWs &w, int idx) {
    return (V *)(w.vecs + (size_t)idx * w.vec_bytes);
}

// ---------------------------------------------------------------- loop runner
bool graph_mode_enabled();

struct LoopSpec {
    std::string key;                                   // identifies the captured body
    std::function<cudaError_t(cudaStream_t)> setup;    // enqueued once before the loop
    std::function<cudaError_t(cudaStream_t)> body;     // one loop iteration (or GMRES cycle)
    int poll_chunk;                                    // iterations per host poll (fallback)
    void *hot_base = nullptr;                          // L2-persisting window (work vectors)
    size_t hot_bytes = 0;
    bool local_fallback = false;  // graph build failure polls this loop only (NCCL bodies)
};

// Writes the initial control block (with the loop's conditional handle), enqueues
// setup, then runs body until ctl->done: graph mode launches a cached exec of
// WHILE(body); the fallback enqueues chunks of `poll_chunk` bodies and polls the
// done flag one chunk behind.  Returns after the stream has drained; the final Ctl
// is copied back into `hctl`.
sb_status run_loop(const LoopSpec &spec, Ctl *dctl, Ctl &hctl, cudaStream_t st, sb_error *err);


// ---------------------------------------------------------------- graph-cache keys
std::string ptr_key(std::initializer_list<const void *> ps);
std::string matrix_key(const sb_matrix &M);

// ---------------------------------------------------------------- shared solver pieces
template <class V>
__device__ __forceinline__ V precond_e(const V *inv, int64_t i, V r) {
    return inv ? vmul(r, inv[i]) : r;  // _apply_precond: Jacobi multiply, or identity copy
}

struct SkipNone {
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
    __device__ __forceinline__ void prepare(const Ctl *) {}
};


struct SolveArgs {
    const sb_matrix *A;
    const void *inv;
    const sb_dense *b;
    sb_dense *x;
    const sb_criteria *crit;
    int64_t dim;
    void *ws;
    sb_log *log;
    cudaStream_t st;
    sb_error *err;
    const sb_tri_precond *tri = nullptr;  // ILU / IC factors (CG, GMRES), else Jacobi / none
};

template <class V>
sb_status check_solve_args(const SolveArgs &a, int64_t &n) {
    sb_error *err = a.err;
    if (!a.A || !a.b || !a.x || !a.crit || !a.ws || !a.log)
        return fail(err, SB_ERR_INVALID_ARGUMENT, "solver: null argument");
    const int64_t rows = matrix_rows(*a.A), cols = matrix_cols(*a.A);
    if (rows != cols)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "solver needs a square operator, got %lldx%lld",
                    (long long)rows, (long long)cols);
    if (a.b->rows != rows || a.b->cols != 1 || a.x->rows != rows || a.x->cols != 1)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "expected %lldx1 vectors, got b (%lld, %lld) and x (%lld, %lld)",
                    (long long)rows, (long long)a.b->rows, (long long)a.b->cols, (long long)a.x->rows,
                    (long long)a.x->cols);
    if (a.b->stride != 1 || a.x->stride != 1)
        return fail(err, SB_ERR_UNSUPPORTED, "solver vectors must be contiguous (stride 1)");
    if (a.crit->max_iters < 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "max_iters must be positive");
    if (((uintptr_t)a.b->data | (uintptr_t)a.x->data | (uintptr_t)a.inv) % 16 != 0)
        return fail(err, SB_ERR_UNSUPPORTED, "solver vectors must be 16-byte aligned");
    n = rows;
    return SB_OK;
}

inline Ctl initial_ctl(const sb_criteria &c, const SolverWs &w, int64_t hist_cap) {
    Ctl h;
    std::memset(&h, 0, sizeof(h));
    h.max_iters = c.max_iters;
    h.has_rf = c.has_residual;
    h.rf = c.reduction_factor;
    h.stop_reason = STOP_NONE;
    h.hist = w.hist;
    h.hist_cap = hist_cap;
    return h;
}

inline sb_status finish_log(const Ctl &h, const SolveArgs &a, const SolverWs &w) {
    sb_error *err = a.err;
    sb_log *log = a.log;
    log->iterations = h.exact ? 0 : h.iter;
    log->converged = h.converged;
    log->stop_reason = h.stop_reason < 0 ? 1 : h.stop_reason;
    log->history_len = h.hist_len;
    const int64_t ncopy = std::min<int64_t>(h.hist_len, std::min<int64_t>(log->history_cap, h.hist_cap));
    if (ncopy > 0 && log->history)
        SB_CUDA(cudaMemcpy(log->history, w.hist, sizeof(double) * ncopy, cudaMemcpyDeviceToHost));
    if (h.status == ST_BREAKDOWN) {
        if (err) err->iteration = h.status_iter;
        return fail(err, SB_ERR_BREAKDOWN, "solver breakdown at iteration %lld", (long long)h.status_iter);
    }
    if (h.status == ST_NUMERIC) {
        if (err) err->iteration = h.status_iter;
        return fail(err, SB_ERR_NUMERIC_FAILURE, "non-finite Hessenberg column or residual estimate at inner iteration %lld",
                    (long long)h.status_iter);
    }
    return SB_OK;
}


// ================================================================ shared: b.b (bnorm) + residual
template <class V>
struct NormB : SkipNone {
    using value_type = V;
    const V *b;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[1]) const {
        const auto B = ldp<W>(b, i);
#pragma unroll
        for (int w = 0; w < W; ++w) part[0] = addd(part[0], mulp(B.v[w], B.v[w]));
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const { c->bnorm = sqrt(tot[0]); }
};

__device__ __forceinline__ void exact_log(Ctl *c) {  // solvers.py:179-181
    c->exact = 1;
    c->iter = 0;
    c->converged = 1;
    c->stop_reason = STOP_RESIDUAL;
    if (c->hist_cap > 0) c->hist[0] = 0.0;
    c->hist_len = 1;
    stop_loop(c);
}

// r = b - A x (t holds A x); shadow = r; dots b.b, r.r.  Used by BiCGSTAB and CGS, whose
// first rho = shadow.r equals r.r exactly (same products, same order).
template <class V>
struct ShadowInit : SkipNone {
    using value_type = V;
    const V *b, *t;
    V *r, *shadow;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[2]) const {
        const auto B = ldp<W>(b, i), T = ldp<W>(t, i);
        Pk<V, W> R;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-1.0, T.v[w], B.v[w]);
            part[0] = addd(part[0], mulp(B.v[w], B.v[w]));
            part[1] = addd(part[1], mulp(R.v[w], R.v[w]));
        }
        stp<W>(r, i, R);
        stp<W>(shadow, i, R);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[2]) const {
        c->bnorm = sqrt(tot[0]);
        c->rnorm = sqrt(tot[1]);
        c->iter = 0;
        if (c->rnorm == 0.0) {
            exact_log(c);
            return;
        }
        c->shadow_norm = c->rnorm;
        c->rho = tot[1];
        c->rho_prev = 1.0;
        c->alpha = 1.0;
        c->omega = 1.0;
        // iteration-1 rho test (solvers.py:244-247 style)
        if (!isfinite(c->rho) || fabs(c->rho) <= kBreakdownRtol * c->shadow_norm * c->rnorm) breakdown(c, 1);
    }
};


// v = A phat with sigma = shadow.v -> alpha (BiCGSTAB / CGS; solvers.py:262-266)
struct BiSigmaFin {
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const {
        const int64_t it = c->iter + 1;
        c->iter = it;
        const double sigma = tot[0];
        if (!isfinite(sigma) || fabs(sigma) <= kBreakdownRtol * fabs(c->rho)) {
            breakdown(c, it);
            return;
        }
        c->alpha = c->rho / sigma;
    }
};

}  // namespace sb
