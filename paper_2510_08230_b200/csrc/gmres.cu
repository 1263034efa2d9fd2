// gmres.cu -- restarted GMRES(m) on the device (solvers.py:322-399): single-pass MGS with fused
// dots, Givens rotations and criteria in the reductions' last block, one graph per cycle.
#include <cmath>

#include "gmres.cuh"
#include "solver_common.cuh"
#include "trisolve.cuh"

namespace sb {

template <class V, class I>
sb_status gmres_solve(const SolveArgs &a) {
    sb_error *err = a.err;
    int64_t n = 0;
    sb_status s = check_solve_args<V>(a, n);
    if (s != SB_OK) return s;
    const int64_t m = a.dim;
    if (m < 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "krylov_dim must be positive");
    if (m > 4096) return fail(err, SB_ERR_UNSUPPORTED, "krylov_dim > 4096");
    const int64_t cap = a.log->history_cap;
    SolverWs w = carve_ws(a.ws, SB_SOLVER_GMRES, sizeof(V), n, m, cap);
    V *basis = ws_vec<V>(w, 0);
    const size_t vstride = w.vec_bytes / sizeof(V);
    V *r = ws_vec<V>(w, (int)m + 1), *t = ws_vec<V>(w, (int)m + 2), *z = ws_vec<V>(w, (int)m + 3),
      *wv = ws_vec<V>(w, (int)m + 4);
    auto V_ = [=](int64_t i) { return basis + (size_t)i * vstride; };
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
    Ctl h = initial_ctl(*a.crit, w, cap);
    h.dim = m;
    double *sm = w.small;
    h.hcol = sm;
    h.g = sm + (m + 2);
    h.cs = sm + 2 * (m + 2);
    h.sn = sm + 3 * (m + 2);
    h.y = sm + 4 * (m + 2);
    h.R = sm + 4 * (m + 2) + m;
    LoopSpec spec;
    spec.key = "gmres" + std::to_string(sizeof(V)) + std::to_string(sizeof(I)) + "|" + std::to_string(m) +
               "|" + matrix_key(M) + ptr_key({a.inv, b, x, a.ws, w.vecs, w.hist, w.small});
    if (tri)
        spec.key += "|tri" + std::to_string(tri->l_unit) +
                    ptr_key({tri->l->row_ptrs, tri->l->values, tri->u->row_ptrs, tri->u->values, tri->workspace});
    spec.poll_chunk = 1;
    const bool fuse_jacobi = inv && matrix_row_owning(M);
    spec.key += fuse_jacobi ? "|fj" : "";
    spec.setup = [=](cudaStream_t st) -> cudaError_t {
        return launch_ew<1>(n, ctl, part, NormB<V>{{}, b}, st);
    };
    spec.body = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(M, x, 1, t, 1, EpiSolverStore<V, NeverSkip>{t, ctl, {}}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<1>(n, ctl, part, GmRestart<V>{{}, b, t, r}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<0>(n, ctl, part, GmFirstBasis<V>{{}, r, V_(0), 0.0}, st);
        if (e != cudaSuccess) return e;
        for (int64_t j = 0; j < m; ++j) {
            if (inv && fuse_jacobi) {  // w = A (M v_j), Jacobi evaluated in the SpMV gather
                e = matrix_apply<V, I>(M, V_(j), 1, wv, 1,
                                       EpiGmPrecondGather<V>{{wv, V_(0), nullptr, ctl, part, {}}, V_(j), inv}, st);
                if (e != cudaSuccess) return e;
            } else {
                const V *zin = V_(j);
                if (tri) {  // z = U^{-1} L^{-1} v_j (t is free inside a cycle)
                    e = launch_trsv<V, I>(*tri->l, true, tri->l_unit != 0, V_(j), 1, t, 1, tw, ctl,
                                          TRI_SKIP_CYCLE_END, st);
                    if (e != cudaSuccess) return e;
                    e = launch_trsv<V, I>(*tri->u, false, false, t, 1, z, 1, tw, ctl, TRI_SKIP_CYCLE_END, st);
                    if (e != cudaSuccess) return e;
                    zin = z;
                } else if (inv) {
                    e = launch_ew<0>(n, ctl, part, GmPrecond<V>{{}, V_(j), inv, z}, st);
                    if (e != cudaSuccess) return e;
                    zin = z;
                }
                e = matrix_apply<V, I>(M, zin, 1, wv, 1, EpiSolver<V, 1, GmH0Fin>{wv, V_(0), nullptr, ctl, part, {}},
                                       st);
                if (e != cudaSuccess) return e;
            }
            for (int64_t i = 0; i < j; ++i) {
                e = launch_ew<1>(n, ctl, part, GmMgsStep<V>{{}, V_(i), V_(i + 1), wv, (int)i, 0.0}, st);
                if (e != cudaSuccess) return e;
            }
            e = launch_ew<1>(n, ctl, part, GmMgsLast<V>{{}, V_(j), wv, (int)j, 0.0}, st);
            if (e != cudaSuccess) return e;
            if (j + 1 < m) {
                e = launch_ew<0>(n, ctl, part, GmNextBasis<V>{{}, wv, V_(j + 1), 0.0}, st);
                if (e != cudaSuccess) return e;
            }
        }
        scalar_kernel<<<1, 1, 0, st>>>(ctl, GmBackSub{});
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (tri) {  // r (free until the next restart) <- V_k y; dx = M^{-1} r; x += dx
            e = launch_ew<0>(n, ctl, part, GmAccum<V>{{}, basis, vstride, r, nullptr, 0}, st);
            if (e != cudaSuccess) return e;
            e = launch_trsv<V, I>(*tri->l, true, tri->l_unit != 0, r, 1, t, 1, tw, ctl, TRI_SKIP_UNLESS_CYCLE_END, st);
            if (e != cudaSuccess) return e;
            e = launch_trsv<V, I>(*tri->u, false, false, t, 1, z, 1, tw, ctl, TRI_SKIP_UNLESS_CYCLE_END, st);
            if (e != cudaSuccess) return e;
            return launch_ew<1>(n, ctl, part, GmAddX<V>{{}, z, x}, st);
        }
        return launch_ew<1>(n, ctl, part, GmUpdate<V, 0>{{}, basis, vstride, inv, x, nullptr, 0}, st);
    };
    s = run_loop(spec, ctl, h, a.st, err);
    if (s != SB_OK) return s;
    return finish_log(h, a, w);
}

}  // namespace sb

using namespace sb;

extern "C" {

#define SB_DEFS(V, VN, I, IN) \
    sb_status sb_gmres_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,                 \
                                         const sb_dense *b, sb_dense *x, const sb_criteria *crit,  \
                                         int64_t krylov_dim, void *workspace, sb_log *log,         \
                                         sb_stream_t stream, sb_error *err) {                      \
        SB_GUARD_BEGIN                                                                             \
        return gmres_solve<V, I>(SolveArgs{a, inv_diag, b, x, crit, krylov_dim, workspace, log,    \
                                           as_stream(stream), err});                               \
        SB_GUARD_END                                                                               \
    }

#define SB_TRI_DEFS(V, VN, I, IN)                                                                  \
    sb_status sb_gmres_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,           \
                                             const sb_dense *b, sb_dense *x,                        \
                                             const sb_criteria *crit, int64_t krylov_dim,           \
                                             void *workspace, sb_log *log, sb_stream_t stream,      \
                                             sb_error *err) {                                       \
        SB_GUARD_BEGIN                                                                              \
        if (!m || !m->l || !m->u || !m->workspace)                                                  \
            return fail(err, SB_ERR_INVALID_ARGUMENT, "triangular preconditioner: null argument");  \
        SolveArgs sa{a, nullptr, b, x, crit, krylov_dim, workspace, log, as_stream(stream), err};   \
        sa.tri = m;                                                                                 \
        return gmres_solve<V, I>(sa);                                                               \
        SB_GUARD_END                                                                                \
    }
SB_TRI_DEFS(float, float, int32_t, i32)
SB_TRI_DEFS(float, float, int64_t, i64)
SB_TRI_DEFS(double, double, int32_t, i32)
SB_TRI_DEFS(double, double, int64_t, i64)

SB_DEFS(float, float, int32_t, i32)
SB_DEFS(float, float, int64_t, i64)
SB_DEFS(double, double, int32_t, i32)
SB_DEFS(double, double, int64_t, i64)

}  // extern "C"
