// trisolve.cu -- sparse triangular solves, ILU(0) and IC(0) factorizations on the device.
//
// Reference: linop.solve_lower_tri / solve_upper_tri (linop.py:169-198) ->
// _kernels.solve_lower / solve_upper (_kernels.py:91-137); precond.ilu0_factorize
// (precond.py:155-187), _split_lu (:190-202), ic0_factorize (:205-256).  Every row's
// arithmetic follows the reference loop in its order, so the results are bit-exact;
// the parallelism comes from running rows whose dependencies are complete concurrently
// (sync-free: ready flags, rows claimed in order by warps, see trisolve.cuh).
#include <algorithm>

#include "capi_util.cuh"
#include "trisolve.cuh"

namespace sb {

// ---------------------------------------------------------------- pattern split
// counts[i] = entries of row i with col < i (or <= i): the strict lower part of _split_lu
// (or the lower pattern of ic0_factorize)
template <class I>
__global__ void split_count_kernel(int64_t n, const I *__restrict__ rp, const I *__restrict__ ci, int incl_diag,
                                   int64_t *counts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const I *lo = ci + rp[i], *hi = ci + rp[i + 1];
        const I key = (I)(incl_diag ? i + 1 : i);
        counts[i] = (int64_t)(lbound(lo, hi, key) - lo);
    }
}

template <class V, class I>
__global__ void split_scatter_kernel(int64_t n, const I *__restrict__ rp, const I *__restrict__ ci,
                                     const V *__restrict__ val, const I *__restrict__ lp, const I *__restrict__ up,
                                     I *lc, V *lv, I *uc, V *uv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = rp[i], nl = (int64_t)lp[i + 1] - lp[i];
        for (int64_t k = 0; k < nl; ++k) {
            lc[lp[i] + k] = ci[s + k];
            lv[lp[i] + k] = val[s + k];
        }
        const int64_t nu = (int64_t)rp[i + 1] - s - nl;
        for (int64_t k = 0; k < nu; ++k) {
            uc[up[i] + k] = ci[s + nl + k];
            uv[up[i] + k] = val[s + nl + k];
        }
    }
}

// ---------------------------------------------------------------- ILU(0)
// diag_pos[i] = position of (i, i) in row i, -1 if absent
template <class I>
__global__ void diag_pos_kernel(int64_t n, const I *__restrict__ rp, const I *__restrict__ ci, int64_t *dpos) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const I *lo = ci + rp[i], *hi = ci + rp[i + 1];
        const I *p = lbound(lo, hi, (I)i);
        dpos[i] = (p != hi && (int64_t)*p == i) ? (int64_t)(p - ci) : -1;
    }
}

// Row i (one thread, rows claimed in order): for each stored k < i (column order) wait
// for row k, l_ik = a_ik / u_kk, then a_ij -= l_ik * u_kj over row k's upper entries
// present in row i; finally the pivot check.  Value-dtype arithmetic like the reference's
// NumPy scalars.  The first failing row (the one the sequential loop raises at) wins
// through atomicMin; a failing row still publishes its flag so nobody waits forever.
template <class V, class I>
__global__ void __launch_bounds__(256) ilu0_kernel(int64_t n, const I *__restrict__ rp, const I *__restrict__ ci,
                                                   V *vals, const int64_t *__restrict__ dpos, TriWs w) {
    for (;;) {
        const int64_t base = claim_rows(w.counter);
        if (base >= n) return;
        const int64_t i = base + (threadIdx.x & 31);
        if (i < n) {
            const int64_t s = rp[i], e = rp[i + 1];
            unsigned long long fail = ~0ull;
            for (int64_t idx = s; idx < e; ++idx) {
                const int64_t k = ci[idx];
                if (k >= i) break;
                wait_ready(w.ready, k);
                const int64_t dk = dpos[k];
                const V ukk = dk >= 0 ? __ldcg(vals + dk) : (V)0;
                if (ukk == (V)0) {
                    fail = ((unsigned long long)i << 32) | (unsigned long long)k;
                    break;
                }
                const V lik = vdiv(vals[idx], ukk);
                vals[idx] = lik;
                for (int64_t idx2 = dk + 1; idx2 < (int64_t)rp[k + 1]; ++idx2) {
                    const I j = ci[idx2];
                    const I *p = lbound(ci + s, ci + e, j);
                    if (p != ci + e && *p == j) {
                        V &a = vals[p - ci];
                        a = vsub(a, vmul(lik, __ldcg(vals + idx2)));
                    }
                }
            }
            if (fail == ~0ull && (dpos[i] < 0 || vals[dpos[i]] == (V)0))
                fail = ((unsigned long long)i << 32) | (unsigned long long)i;
            if (fail != ~0ull) atomicMin(w.err, fail);
            __threadfence();
            st_release_i32(w.ready + i, 1);
        }
    }
}

// Same rows, arithmetic and order as ilu0_kernel, in the converged-polling form of
// sptrsv_poll_kernel: each lane's cursor walks its row's L part while the pivot rows it
// needs are published, never blocking inside divergent code.
template <class V, class I>
__global__ void __launch_bounds__(256) ilu0_poll_kernel(int64_t n, const I *__restrict__ rp,
                                                        const I *__restrict__ ci, V *vals,
                                                        const int64_t *__restrict__ dpos, TriWs w) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int64_t base = claim_rows(w.counter);
        if (base >= n) return;
        const int64_t i = base + lane;
        bool active = i < n;
        int64_t s = 0, e = 0, idx = 0;
        unsigned long long fail = ~0ull;
        if (active) {
            s = rp[i];
            e = rp[i + 1];
            idx = s;
        }
        unsigned ns = 32;
        for (;;) {
            bool moved = false;
            if (active) {
                bool finished = false;
                for (; idx < e; ++idx) {
                    const int64_t k = ci[idx];
                    if (k >= i) {
                        finished = true;
                        break;
                    }
                    if (ld_acquire_i32(w.ready + k) == 0) break;
                    moved = true;
                    const int64_t dk = dpos[k];
                    const V ukk = dk >= 0 ? __ldcg(vals + dk) : (V)0;
                    if (ukk == (V)0) {
                        fail = ((unsigned long long)i << 32) | (unsigned long long)k;
                        finished = true;
                        break;
                    }
                    const V lik = vdiv(vals[idx], ukk);
                    vals[idx] = lik;
                    for (int64_t idx2 = dk + 1; idx2 < (int64_t)rp[k + 1]; ++idx2) {
                        const I j = ci[idx2];
                        const I *q = lbound(ci + s, ci + e, j);
                        if (q != ci + e && *q == j) {
                            V &a = vals[q - ci];
                            a = vsub(a, vmul(lik, __ldcg(vals + idx2)));
                        }
                    }
                }
                if (idx == e) finished = true;
                if (finished) {
                    if (fail == ~0ull && (dpos[i] < 0 || vals[dpos[i]] == (V)0))
                        fail = ((unsigned long long)i << 32) | (unsigned long long)i;
                    if (fail != ~0ull) atomicMin(w.err, fail);
                    __threadfence();
                    st_release_i32(w.ready + i, 1);
                    active = false;
                    moved = true;
                }
            }
            if (!__any_sync(0xffffffffu, active)) break;
            if (__any_sync(0xffffffffu, moved)) {
                ns = 32;
            } else {
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
            }
        }
    }
}

// ---------------------------------------------------------------- IC(0)
// Lower pattern (cols <= i, diagonal last) of A, computed in fp64 like the reference's
// Python floats (lv scratch), cast to the value dtype per row.
template <class V, class I>
__global__ void __launch_bounds__(256) ic0_kernel(int64_t n, const I *__restrict__ lp, const I *__restrict__ lc,
                                                  const V *__restrict__ la, double *lv, V *out, TriWs w) {
    for (;;) {
        const int64_t base = claim_rows(w.counter);
        if (base >= n) return;
        const int64_t i = base + (threadIdx.x & 31);
        if (i < n) {
            const int64_t si = lp[i], ei = lp[i + 1];
            unsigned long long fail = ~0ull;
            for (int64_t pos = si; pos < ei && fail == ~0ull; ++pos) {
                const int64_t j = lc[pos];
                if (j < i) wait_ready(w.ready, j);
                double s = (double)la[pos];
                const int64_t sj = lp[j], ej = lp[j + 1];
                int64_t pi = si, pj = sj;
                while (pi < ei && pj < ej) {
                    const int64_t c1 = lc[pi], c2 = lc[pj];
                    if (c1 >= j || c2 >= j) break;
                    if (c1 == c2) {
                        s = __dsub_rn(s, __dmul_rn(lv[pi], j == i ? lv[pj] : __ldcg(lv + pj)));
                        ++pi;
                        ++pj;
                    } else if (c1 < c2) {
                        ++pi;
                    } else {
                        ++pj;
                    }
                }
                if (j == i) {
                    if (s <= 0.0) fail = ((unsigned long long)i << 32) | (unsigned long long)i;
                    else lv[pos] = __dsqrt_rn(s);
                } else {
                    const double ljj = ej > sj ? __ldcg(lv + ej - 1) : 0.0;
                    if (ej == sj || (int64_t)lc[ej - 1] != j || ljj == 0.0)
                        fail = ((unsigned long long)i << 32) | (unsigned long long)j;
                    else lv[pos] = __ddiv_rn(s, ljj);
                }
            }
            if (fail == ~0ull && (ei == si || (int64_t)lc[ei - 1] != i))
                fail = ((unsigned long long)i << 32) | (unsigned long long)i;
            if (fail != ~0ull) atomicMin(w.err, fail);
            for (int64_t pos = si; pos < ei; ++pos) out[pos] = (V)lv[pos];
            __threadfence();
            st_release_i32(w.ready + i, 1);
        }
    }
}

// IC(0) in the converged-polling form (same rows, arithmetic and order as ic0_kernel):
// each lane's cursor walks its row while the rows it needs are published.
template <class V, class I>
__global__ void __launch_bounds__(256) ic0_poll_kernel(int64_t n, const I *__restrict__ lp,
                                                       const I *__restrict__ lc, const V *__restrict__ la,
                                                       double *lv, V *out, TriWs w) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int64_t base = claim_rows(w.counter);
        if (base >= n) return;
        const int64_t i = base + lane;
        bool active = i < n;
        int64_t si = 0, ei = 0, pos = 0;
        unsigned long long fail = ~0ull;
        if (active) {
            si = lp[i];
            ei = lp[i + 1];
            pos = si;
        }
        unsigned ns = 32;
        for (;;) {
            bool moved = false;
            if (active) {
                for (; pos < ei && fail == ~0ull; ++pos) {
                    const int64_t j = lc[pos];
                    if (j < i && ld_acquire_i32(w.ready + j) == 0) break;
                    moved = true;
                    double sacc = (double)la[pos];
                    const int64_t sj = lp[j], ej = lp[j + 1];
                    int64_t pi = si, pj = sj;
                    while (pi < ei && pj < ej) {
                        const int64_t c1 = lc[pi], c2 = lc[pj];
                        if (c1 >= j || c2 >= j) break;
                        if (c1 == c2) {
                            sacc = __dsub_rn(sacc, __dmul_rn(lv[pi], j == i ? lv[pj] : __ldcg(lv + pj)));
                            ++pi;
                            ++pj;
                        } else if (c1 < c2) {
                            ++pi;
                        } else {
                            ++pj;
                        }
                    }
                    if (j == i) {
                        if (sacc <= 0.0) fail = ((unsigned long long)i << 32) | (unsigned long long)i;
                        else lv[pos] = __dsqrt_rn(sacc);
                    } else {
                        const double ljj = ej > sj ? __ldcg(lv + ej - 1) : 0.0;
                        if (ej == sj || (int64_t)lc[ej - 1] != j || ljj == 0.0)
                            fail = ((unsigned long long)i << 32) | (unsigned long long)j;
                        else lv[pos] = __ddiv_rn(sacc, ljj);
                    }
                }
                if (pos >= ei || fail != ~0ull) {
                    if (fail == ~0ull && (ei == si || (int64_t)lc[ei - 1] != i))
                        fail = ((unsigned long long)i << 32) | (unsigned long long)i;
                    if (fail != ~0ull) atomicMin(w.err, fail);
                    for (int64_t q = si; q < ei; ++q) out[q] = (V)lv[q];
                    __threadfence();
                    st_release_i32(w.ready + i, 1);
                    active = false;
                    moved = true;
                }
            }
            if (!__any_sync(0xffffffffu, active)) break;
            if (__any_sync(0xffffffffu, moved)) {
                ns = 32;
            } else {
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
            }
        }
    }
}

inline int sweep_grid(int64_t n) { return (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)device_info().sms * 8); }

inline sb_status read_err(const TriWs &w, cudaStream_t st, unsigned long long &key, sb_error *err) {
    SB_CUDA(cudaMemcpyAsync(&key, w.err, sizeof(key), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    return SB_OK;
}

inline sb_status reset_ws(const TriWs &w, int64_t n, cudaStream_t st, sb_error *err) {
    SB_CUDA(cudaMemsetAsync(w.ready, 0, sizeof(int) * (size_t)(n > 0 ? n : 1), st));
    SB_CUDA(cudaMemsetAsync(w.counter, 0, sizeof(unsigned long long), st));
    SB_CUDA(cudaMemsetAsync(w.err, 0xff, sizeof(unsigned long long), st));
    return SB_OK;
}

template <class V, class I>
sb_status trisolve(const sb_csr *T, int lower, int unit, const sb_dense *b, sb_dense *x, void *ws, cudaStream_t st,
                   sb_error *err) {
    if (!T || !b || !x || !ws) return fail(err, SB_ERR_INVALID_ARGUMENT, "trisolve: null argument");
    if (T->rows != T->cols)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "triangular solve needs a square matrix, got %lldx%lld",
                    (long long)T->rows, (long long)T->cols);
    if (b->rows != T->rows || x->rows != T->rows || b->cols != x->cols)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "apply shape mismatch");
    const TriWs w = carve_tri_ws(ws, T->rows);
    sb_status s = tri_factor_check<V, I>(*T, lower != 0, unit != 0, w, st, err);
    if (s != SB_OK) return s;
    for (int64_t j = 0; j < b->cols; ++j)
        SB_CUDA((launch_trsv<V, I>(*T, lower != 0, unit != 0, (const V *)b->data + j, b->stride, (V *)x->data + j,
                                   x->stride, w, nullptr, TRI_SKIP_NONE, st)));
    return SB_OK;
}

template <class V, class I>
sb_status ilu0(const sb_csr *A, void *vals_out, void *ws, void *dpos_ws, cudaStream_t st, sb_error *err) {
    if (!A || !vals_out || !ws || !dpos_ws) return fail(err, SB_ERR_INVALID_ARGUMENT, "ilu0: null argument");
    if (A->rows != A->cols)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "ILU(0) needs a square matrix, got %lldx%lld",
                    (long long)A->rows, (long long)A->cols);
    const int64_t n = A->rows;
    if (n == 0) return SB_OK;
    const TriWs w = carve_tri_ws(ws, n);
    sb_status s = reset_ws(w, n, st, err);
    if (s != SB_OK) return s;
    SB_CUDA(cudaMemcpyAsync(vals_out, A->values, sizeof(V) * (size_t)A->nnz, cudaMemcpyDeviceToDevice, st));
    int64_t *dpos = (int64_t *)dpos_ws;
    diag_pos_kernel<I><<<sweep_grid(n), 256, 0, st>>>(n, (const I *)A->row_ptrs, (const I *)A->col_idxs, dpos);
    SB_CUDA(cudaGetLastError());
    // converged polling (default; 128^3: 23.65 -> 22.6 ms) or the blocking-spin sweep
    // (SPARSEB200_ILU_POLL=0)
    static const bool poll = !getenv("SPARSEB200_ILU_POLL") || atoi(getenv("SPARSEB200_ILU_POLL")) != 0;
    if (poll)
        ilu0_poll_kernel<V, I><<<sweep_grid(n), 256, 0, st>>>(n, (const I *)A->row_ptrs, (const I *)A->col_idxs,
                                                              (V *)vals_out, dpos, w);
    else
        ilu0_kernel<V, I><<<sweep_grid(n), 256, 0, st>>>(n, (const I *)A->row_ptrs, (const I *)A->col_idxs,
                                                         (V *)vals_out, dpos, w);
    SB_CUDA(cudaGetLastError());
    unsigned long long key;
    s = read_err(w, st, key, err);
    if (s != SB_OK) return s;
    if (key == ~0ull) return SB_OK;
    const int64_t row = (int64_t)(key & 0xffffffffull);
    if (err) err->row = row;
    return fail(err, SB_ERR_ZERO_PIVOT, "zero pivot at row %lld", (long long)row);
}

template <class V, class I>
sb_status ic0(int64_t n, const void *lp, const void *lc, const void *la, void *out, void *ws, void *scratch,
              cudaStream_t st, sb_error *err) {
    if (n == 0) return SB_OK;
    if (!lp || !lc || !la || !out || !ws || !scratch) return fail(err, SB_ERR_INVALID_ARGUMENT, "ic0: null argument");
    const TriWs w = carve_tri_ws(ws, n);
    sb_status s = reset_ws(w, n, st, err);
    if (s != SB_OK) return s;
    // converged polling (default; 128^3: 16.1 -> 15.8 ms) or the blocking spin (SPARSEB200_ILU_POLL=0)
    static const bool poll = !getenv("SPARSEB200_ILU_POLL") || atoi(getenv("SPARSEB200_ILU_POLL")) != 0;
    if (poll)
        ic0_poll_kernel<V, I><<<sweep_grid(n), 256, 0, st>>>(n, (const I *)lp, (const I *)lc, (const V *)la,
                                                             (double *)scratch, (V *)out, w);
    else
        ic0_kernel<V, I><<<sweep_grid(n), 256, 0, st>>>(n, (const I *)lp, (const I *)lc, (const V *)la,
                                                        (double *)scratch, (V *)out, w);
    SB_CUDA(cudaGetLastError());
    unsigned long long key;
    s = read_err(w, st, key, err);
    if (s != SB_OK) return s;
    if (key == ~0ull) return SB_OK;
    const int64_t row = (int64_t)(key & 0xffffffffull);
    if (err) err->row = row;
    return fail(err, SB_ERR_INDEFINITE_PIVOT, "non-positive or missing pivot at row %lld", (long long)row);
}

}  // namespace sb

using namespace sb;

extern "C" {

size_t sb_tri_workspace_bytes(int64_t n) { return tri_ws_bytes(n); }

#define SB_TRI_I(I, IN)                                                                             \
    sb_status sb_csr_split_count_##IN(int64_t n, const void *rp, const void *ci, int32_t incl_diag,  \
                                      int64_t *counts, sb_stream_t stream, sb_error *err) {          \
        SB_GUARD_BEGIN                                                                               \
        if (n == 0) return SB_OK;                                                                    \
        split_count_kernel<I><<<sweep_grid(n), 256, 0, as_stream(stream)>>>(                         \
            n, (const I *)rp, (const I *)ci, incl_diag, counts);                                     \
        SB_CUDA(cudaGetLastError());                                                                 \
        return SB_OK;                                                                                \
        SB_GUARD_END                                                                                 \
    }

#define SB_TRI_VI(V, VN, I, IN)                                                                     \
    sb_status sb_csr_split_scatter_##VN##_##IN(int64_t n, const void *rp, const void *ci,            \
                                               const void *val, const void *lp, const void *up,      \
                                               void *lc, void *lv, void *uc, void *uv,               \
                                               sb_stream_t stream, sb_error *err) {                  \
        SB_GUARD_BEGIN                                                                               \
        if (n == 0) return SB_OK;                                                                    \
        split_scatter_kernel<V, I><<<sweep_grid(n), 256, 0, as_stream(stream)>>>(                    \
            n, (const I *)rp, (const I *)ci, (const V *)val, (const I *)lp, (const I *)up, (I *)lc,   \
            (V *)lv, (I *)uc, (V *)uv);                                                              \
        SB_CUDA(cudaGetLastError());                                                                 \
        return SB_OK;                                                                                \
        SB_GUARD_END                                                                                 \
    }                                                                                                \
    sb_status sb_csr_trisolve_##VN##_##IN(const sb_csr *t, int32_t lower, int32_t unit_diag,         \
                                          const sb_dense *b, sb_dense *x, void *workspace,           \
                                          sb_stream_t stream, sb_error *err) {                       \
        SB_GUARD_BEGIN                                                                               \
        return trisolve<V, I>(t, lower, unit_diag, b, x, workspace, as_stream(stream), err);         \
        SB_GUARD_END                                                                                 \
    }                                                                                                \
    sb_status sb_csr_tri_check_##VN##_##IN(const sb_csr *t, int32_t lower, int32_t unit_diag,        \
                                           void *workspace, sb_stream_t stream, sb_error *err) {     \
        SB_GUARD_BEGIN                                                                               \
        if (!t || !workspace) return fail(err, SB_ERR_INVALID_ARGUMENT, "tri_check: null argument"); \
        return tri_factor_check<V, I>(*t, lower != 0, unit_diag != 0,                                \
                                      carve_tri_ws(workspace, t->rows), as_stream(stream), err);     \
        SB_GUARD_END                                                                                 \
    }                                                                                                \
    sb_status sb_ilu0_##VN##_##IN(const sb_csr *a, void *values_out, void *workspace,                \
                                  void *diag_workspace, sb_stream_t stream, sb_error *err) {         \
        SB_GUARD_BEGIN                                                                               \
        return ilu0<V, I>(a, values_out, workspace, diag_workspace, as_stream(stream), err);         \
        SB_GUARD_END                                                                                 \
    }                                                                                                \
    sb_status sb_ic0_##VN##_##IN(int64_t n, const void *lp, const void *lc, const void *la,          \
                                 void *values_out, void *workspace, void *scratch,                   \
                                 sb_stream_t stream, sb_error *err) {                                \
        SB_GUARD_BEGIN                                                                               \
        return ic0<V, I>(n, lp, lc, la, values_out, workspace, scratch, as_stream(stream), err);     \
        SB_GUARD_END                                                                                 \
    }

SB_TRI_I(int32_t, i32)
SB_TRI_I(int64_t, i64)
SB_TRI_VI(float, float, int32_t, i32)
SB_TRI_VI(float, float, int64_t, i64)
SB_TRI_VI(double, double, int32_t, i32)
SB_TRI_VI(double, double, int64_t, i64)

}  // extern "C"
