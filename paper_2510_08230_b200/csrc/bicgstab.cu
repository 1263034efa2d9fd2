// bicgstab.cu -- right-preconditioned BiCGSTAB on the device (recurrence in oracle/sbref.cpp).
//
// Every dot of this solver is Neumaier-compensated (CAcc partials, compensated warp / block
// / grid trees): on the 256^3 convection-diffusion system (config #4) the recurrence is
// so sensitive to the summation order that plain fp64 tree dots break down at iteration
// ~170 while near-exact dots follow the exact-arithmetic trajectory and converge (the
// oracle with compensated dots: 1059 iterations).  The dots are streamed
// with the vectors, so the extra flops are free in these bandwidth-bound passes.
#include <cmath>

#include "bicgstab.cuh"
#include "solver_common.cuh"
#include "trisolve.cuh"

namespace sb {

template <class V, class I>
sb_status tri_precond_check(const sb_tri_precond &m, sb_error *err, cudaStream_t st);

template <class V, class I>
sb_status bicgstab_solve(const SolveArgs &a) {
    sb_error *err = a.err;
    int64_t n = 0;
    sb_status s = check_solve_args<V>(a, n);
    if (s != SB_OK) return s;
    const int64_t cap = a.log->history_cap;
    SolverWs w = carve_ws(a.ws, SB_SOLVER_BICGSTAB, sizeof(V), n, 0, cap);
    V *r = ws_vec<V>(w, 0), *rh = ws_vec<V>(w, 1), *p = ws_vec<V>(w, 2), *v = ws_vec<V>(w, 3),
      *sv = ws_vec<V>(w, 4), *ph = ws_vec<V>(w, 5), *sh = ws_vec<V>(w, 6), *t = ws_vec<V>(w, 7);
    const V *b = (const V *)a.b->data, *inv = (const V *)a.inv;
    V *x = (V *)a.x->data;
    Ctl *ctl = w.ctl;
    double *part = w.partials;
    const sb_matrix M = *a.A;
    const sb_tri_precond *tri = a.tri;
    if (tri) {
        s = tri_precond_check<V, I>(*tri, err, a.st);
        if (s != SB_OK) return s;
    }
    const TriWs tw = tri ? carve_tri_ws(tri->workspace, n) : TriWs{};
    // out = U^{-1} L^{-1} in through t (t is free until A shat); skipped once the loop is done
    auto precond = [=](const V *in, V *out, cudaStream_t st) -> cudaError_t {
        cudaError_t e = launch_trsv<V, I>(*tri->l, true, tri->l_unit != 0, in, 1, t, 1, tw, ctl,
                                          TRI_SKIP_DONE, st);
        if (e != cudaSuccess) return e;
        return launch_trsv<V, I>(*tri->u, false, false, t, 1, out, 1, tw, ctl, TRI_SKIP_DONE, st);
    };
    Ctl h = initial_ctl(*a.crit, w, cap);
    LoopSpec spec;
    spec.key = "bicgstab" + std::to_string(sizeof(V)) + std::to_string(sizeof(I)) + "|" +
               matrix_key(M) + ptr_key({a.inv, b, x, a.ws, w.vecs, w.hist, w.small});
    if (tri)
        spec.key += "|tri" + std::to_string(tri->l_unit) +
                    ptr_key({tri->l->row_ptrs, tri->l->values, tri->u->row_ptrs, tri->u->values, tri->workspace});
    spec.poll_chunk = 8;
    spec.setup = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(M, x, 1, t, 1, EpiStore<V>{t, 1}, st);
        if (e != cudaSuccess) return e;
        return launch_ew<2>(n, ctl, part, BiShadowInit<V>{{{}, b, t, r, rh}}, st);
    };
    spec.body = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = launch_ew<0>(n, ctl, part, BiDirection<V>{{}, r, v, inv, p, tri ? nullptr : ph, 0, 0, false}, st);
        if (e != cudaSuccess) return e;
        if (tri && (e = precond(p, ph, st)) != cudaSuccess) return e;
        e = matrix_apply<V, I>(M, ph, 1, v, 1, EpiSolverC<V, 1, BiSigmaFin>{v, rh, nullptr, ctl, part, {}}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<1>(n, ctl, part, BiS<V>{{}, r, v, inv, sv, tri ? nullptr : sh, 0}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<1>(n, ctl, part, BiEarlyX<V>{ph, x, 0}, st);
        if (e != cudaSuccess) return e;
        if (tri && (e = precond(sv, sh, st)) != cudaSuccess) return e;  // after an early stop: skipped
        e = matrix_apply<V, I>(M, sh, 1, t, 1, EpiSolverC<V, 2, BiOmegaFin>{t, nullptr, sv, ctl, part, {}}, st);
        if (e != cudaSuccess) return e;
        return launch_ew<2>(n, ctl, part, BiUpdate<V>{{}, ph, sh, sv, t, rh, x, r, 0, 0}, st);
    };
    s = run_loop(spec, ctl, h, a.st, err);
    if (s != SB_OK) return s;
    return finish_log(h, a, w);
}

}  // namespace sb

using namespace sb;

extern "C" {

#define SB_DEFS(V, VN, I, IN) \
    sb_status sb_bicgstab_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,              \
                                            const sb_dense *b, sb_dense *x,                        \
                                            const sb_criteria *crit, void *workspace, sb_log *log, \
                                            sb_stream_t stream, sb_error *err) {                   \
        SB_GUARD_BEGIN                                                                             \
        return bicgstab_solve<V, I>(SolveArgs{a, inv_diag, b, x, crit, 0, workspace, log,          \
                                              as_stream(stream), err});                            \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_bicgstab_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,       \
                                                const sb_dense *b, sb_dense *x,                    \
                                                const sb_criteria *crit, void *workspace,          \
                                                sb_log *log, sb_stream_t stream, sb_error *err) {  \
        SB_GUARD_BEGIN                                                                             \
        SolveArgs sa{a, nullptr, b, x, crit, 0, workspace, log, as_stream(stream), err};           \
        sa.tri = m;                                                                                \
        return bicgstab_solve<V, I>(sa);                                                           \
        SB_GUARD_END                                                                               \
    }

SB_DEFS(float, float, int32_t, i32)
SB_DEFS(float, float, int64_t, i64)
SB_DEFS(double, double, int32_t, i32)
SB_DEFS(double, double, int64_t, i64)

}  // extern "C"
