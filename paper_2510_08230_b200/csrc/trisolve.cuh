// trisolve.cuh -- sync-free sparse triangular solves on the device, shared by the
// standalone entry points (trisolve.cu) and the ILU / IC preconditioned solver loops.
//
// Reference: _kernels.solve_lower / solve_upper (_kernels.py:91-137) via
// linop.solve_lower_tri / solve_upper_tri (linop.py:169-198): one sequential sweep;
// acc = b[i] + 0.0 in fp64, acc -= values[k] * x[j] in stored order (the product in the
// value dtype), x[i] = acc (unit diagonal) or acc / diag, cast on store.
//
// B200 shape: one thread per row, rows claimed in solve order by warps through an
// atomic counter (so every row a thread waits on belongs to an already running warp:
// no deadlock whatever the scheduling), a per-row ready flag published with a release
// store after x[i] and awaited with acquire loads.  Rows whose dependencies are done
// proceed immediately, so the sweep runs at the matrix's dependency-level parallelism
// without an analysis phase or one launch per level.  Each row's arithmetic is the
// reference's, in the reference's order -> bit-exact results.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "capi_util.cuh"
#include "solver_common.cuh"

namespace sb {

// workspace of one triangular sweep: ready flags (n int32) + claim counter
struct TriWs {
    int *ready;
    unsigned long long *counter;
    unsigned long long *err;  // first failing row key (factorizations / checks)
};

inline size_t tri_ws_bytes(int64_t n) { return a256(sizeof(int) * (size_t)(n > 0 ? n : 1)) + 256; }

inline TriWs carve_tri_ws(void *ws, int64_t n) {
    unsigned char *p = (unsigned char *)ws;
    TriWs w;
    w.ready = (int *)p;
    p += a256(sizeof(int) * (size_t)(n > 0 ? n : 1));
    w.counter = (unsigned long long *)p;
    w.err = (unsigned long long *)(p + 64);
    return w;
}

__device__ __forceinline__ int ld_acquire_i32(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_i32(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Value-as-flag publication (sptrsv_poll_kernel<..., VF = true>): x is pre-filled with a
// signalling-NaN sentinel that floating-point arithmetic never produces (any NaN result
// is a quiet NaN), the solved value is published with a release store and consumed with
// one acquire load -- one L2 round trip per dependency instead of flag + value.
template <class V>
struct TriSentinel;
template <>
struct TriSentinel<double> {
    static constexpr unsigned long long bits = 0x7FF4A5A5A5A5A5A5ull;
};
template <>
struct TriSentinel<float> {
    static constexpr unsigned bits = 0x7FA5A5A5u;
};
__device__ __forceinline__ bool ld_acquire_val(const double *p, double &v) {
    unsigned long long u;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(u) : "l"(p) : "memory");
    v = __longlong_as_double((long long)u);
    return u != TriSentinel<double>::bits;
}
__device__ __forceinline__ bool ld_acquire_val(const float *p, float &v) {
    unsigned u;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(u) : "l"(p) : "memory");
    v = __uint_as_float(u);
    return u != TriSentinel<float>::bits;
}
__device__ __forceinline__ void st_release_val(double *p, double v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v))
                 : "memory");
}
__device__ __forceinline__ void st_release_val(float *p, float v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(__float_as_uint(v)) : "memory");
}
// Spin with a short back-off: hundreds of thousands of waiting threads issuing
// back-to-back acquire loads would flood L2 and slow the very stores they wait for
// (128^3 IC-CG: 1283 -> 1055 ms).  A level-sorted sweep order was also measured: it
// scatters every warp's rows over the matrix and was slower (lower sweep 4.7 -> 5.3 ms).
__device__ __forceinline__ void wait_ready(const int *ready, int64_t j) {
    unsigned ns = 32;
    while (ld_acquire_i32(ready + j) == 0) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

// Claims the next 32 * k rows (in solve order) for the calling warp; all lanes return
// the same base.  Must be called by the full warp.
__device__ __forceinline__ int64_t claim_rows(unsigned long long *counter, unsigned k = 1) {
    unsigned long long base = 0;
    if ((threadIdx.x & 31) == 0) base = atomicAdd(counter, 32ull * k);
    return (int64_t)__shfl_sync(0xffffffffu, base, 0);
}

// solver-loop skip rule (ctl may be null for standalone sweeps)
enum { TRI_SKIP_NONE = 0, TRI_SKIP_DONE = 1, TRI_SKIP_CYCLE_END = 2, TRI_SKIP_UNLESS_CYCLE_END = 3 };
__device__ __forceinline__ bool tri_skip(const Ctl *c, int mode) {
    if (!c || mode == TRI_SKIP_NONE) return false;
    if (loop_done(c)) return true;
    if (mode == TRI_SKIP_CYCLE_END) return c->cycle_end != 0;
    if (mode == TRI_SKIP_UNLESS_CYCLE_END) return c->cycle_end == 0;
    return false;
}

template <class V>
__global__ void tri_sentinel_fill_kernel(int64_t n, V *x, int64_t ldx, const Ctl *ctl, int skip_mode) {
    if (tri_skip(ctl, skip_mode)) return;  // a skipped sweep leaves x untouched
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if constexpr (sizeof(V) == 8)
            reinterpret_cast<unsigned long long *>(x)[i * ldx] = TriSentinel<double>::bits;
        else
            reinterpret_cast<unsigned *>(x)[i * ldx] = TriSentinel<float>::bits;
    }
}

// x = T^{-1} b for a triangular CSR T whose structure was validated (tri_check_kernel).
// A warp claims RPT * 32 rows; lane l solves rows base + 32 u + l for u = 0 .. RPT-1 in
// order.  Still deadlock-free: the lowest unsolved row has every dependency solved, and
// its lane has finished all of its earlier rows, so it is the row that lane is on.  More
// rows per claim = more of the sweep resident at once: the sweep is a pipeline whose
// throughput is (rows in flight) / (hops per row's dependency chain).
template <class V, class I, bool LOWER, int RPT = 1>
__global__ void __launch_bounds__(256) sptrsv_kernel(int64_t n, const I *__restrict__ rp,
                                                     const I *__restrict__ ci, const V *__restrict__ val,
                                                     const V *b, int64_t ldb, V *x, int64_t ldx, int unit,
                                                     TriWs w, const Ctl *ctl, int skip_mode) {
    if (tri_skip(ctl, skip_mode)) return;
    for (;;) {
        const int64_t base = claim_rows(w.counter, RPT);
        if (base >= n) return;
#pragma unroll 1
        for (int u = 0; u < RPT; ++u) {
        const int64_t t = base + 32 * u + (threadIdx.x & 31);
        if (t < n) {
            const int64_t i = LOWER ? t : n - 1 - t;
            double acc = (double)b[i * ldb] + 0.0;
            double diag = 1.0;
            for (int64_t k = rp[i]; k < (int64_t)rp[i + 1]; ++k) {
                const int64_t j = ci[k];
                if (LOWER ? j < i : j > i) {
                    wait_ready(w.ready, j);
                    acc = __dsub_rn(acc, mulp(val[k], __ldcg(x + j * ldx)));
                } else if (j == i) {
                    diag = (double)val[k];
                }
            }
            x[i * ldx] = (LOWER && unit) ? (V)acc : (V)__ddiv_rn(acc, diag);
            st_release_i32(w.ready + i, 1);
        }
        }
    }
}

// Converged-polling variant: a warp claims RPT * 32 rows; every lane keeps a cursor into
// each of its rows and, each round, consumes entries while their dependencies are ready
// (never blocking inside divergent code, so no reliance on independent-thread scheduling
// between lanes of one warp), publishes finished rows and moves on; a round in which no
// lane of the warp progressed ends with a short sleep.  Same per-row arithmetic and order.
template <class V, class I, bool LOWER, int RPT, bool VF = false>
__global__ void __launch_bounds__(256) sptrsv_poll_kernel(int64_t n, const I *__restrict__ rp,
                                                          const I *__restrict__ ci, const V *__restrict__ val,
                                                          const V *b, int64_t ldb, V *x, int64_t ldx, int unit,
                                                          TriWs w, const Ctl *ctl, int skip_mode) {
    if (tri_skip(ctl, skip_mode)) return;
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int64_t base = claim_rows(w.counter, RPT);
        if (base >= n) return;
        // RPT independent row slots per lane (rows base + 32 u + lane), each advanced
        // whenever its dependencies are ready: a later row of the claim never waits for an
        // earlier one of the same lane (claims straddling grid lines would otherwise hold
        // low-level rows behind high-level ones)
        int64_t i[RPT], k[RPT], ke[RPT];
        double acc[RPT], diag[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int64_t t = base + 32 * u + lane;
            k[u] = ke[u] = 0;
            i[u] = -1;
            acc[u] = 0.0;
            diag[u] = 1.0;
            if (t < n) {
                i[u] = LOWER ? t : n - 1 - t;
                k[u] = rp[i[u]];
                ke[u] = rp[i[u] + 1];
                acc[u] = (double)b[i[u] * ldb] + 0.0;
            }
        }
        unsigned ns = 32;
        for (;;) {
            bool moved = false, busy = false;
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
                if (i[u] < 0) continue;
                for (; k[u] < ke[u]; ++k[u]) {
                    const int64_t j = ci[k[u]];
                    if (LOWER ? j < i[u] : j > i[u]) {
                        V xj;
                        if constexpr (VF) {
                            if (!ld_acquire_val(x + j * ldx, xj)) break;
                        } else {
                            if (ld_acquire_i32(w.ready + j) == 0) break;
                            xj = __ldcg(x + j * ldx);
                        }
                        acc[u] = __dsub_rn(acc[u], mulp(val[k[u]], xj));
                    } else if (j == i[u]) {
                        diag[u] = (double)val[k[u]];
                    }
                    moved = true;
                }
                if (k[u] == ke[u]) {
                    const V xi = (LOWER && unit) ? (V)acc[u] : (V)__ddiv_rn(acc[u], diag[u]);
                    if constexpr (VF) {
                        st_release_val(x + i[u] * ldx, xi);
                    } else {
                        x[i[u] * ldx] = xi;
                        st_release_i32(w.ready + i[u], 1);
                    }
                    i[u] = -1;
                    moved = true;
                } else {
                    busy = true;
                }
            }
            if (!__any_sync(0xffffffffu, busy)) break;
            if (__any_sync(0xffffffffu, moved)) {
                ns = 32;
            } else {
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
            }
        }
    }
}

// Structure / diagonal check in solve order (the reference stops at the first failing
// row): key = position * 4 + kind, kind 1 = entry on the wrong side, 2 = missing or
// zero diagonal (non-unit).  atomicMin keeps the first failing row.
template <class V, class I>
__global__ void __launch_bounds__(256) tri_check_kernel(int64_t n, const I *__restrict__ rp,
                                                        const I *__restrict__ ci, const V *__restrict__ val,
                                                        int lower, int unit, unsigned long long *err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int kind = 0;
        bool has_diag = false;
        double diag = 0.0;
        for (int64_t k = rp[i]; k < (int64_t)rp[i + 1]; ++k) {
            const int64_t j = ci[k];
            if (lower ? j > i : j < i) {
                kind = 1;
                break;
            }
            if (j == i) {
                has_diag = true;
                diag = (double)val[k];
            }
        }
        if (kind == 0 && !(lower && unit) && (!has_diag || diag == 0.0)) kind = 2;
        if (kind) {
            const unsigned long long pos = lower ? (unsigned long long)i : (unsigned long long)(n - 1 - i);
            atomicMin(err, pos * 4ull + (unsigned long long)kind);
        }
    }
}

template <class V, class I>
cudaError_t launch_trsv(const sb_csr &T, bool lower, bool unit, const V *b, int64_t ldb, V *x, int64_t ldx,
                        const TriWs &w, const Ctl *ctl, int skip_mode, cudaStream_t st) {
    const int64_t n = T.rows;
    if (n == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(w.counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    // Default: the converged-polling kernel, one row per lane (tools/precond_bench.py, IC-CG
    // ms, blocking-spin -> polling: 64^3 98 -> 84, 96^3 341 -> 284, 128^3 1058 -> 867;
    // ILU-GMRES conv-diff 64^3 137 -> 118).  SPARSEB200_TRSV_MODE=0 selects the blocking
    // spin kernel; SPARSEB200_TRSV_RPT = 2 / 4 rows per lane.  Measured: processing a lane's
    // rows strictly in order is fast where claims align with grid lines (128^3 IC-CG 430 ms
    // at 4 rows) and ~10x slower where they straddle them (96^3: low-level rows held behind
    // high-level ones); independent slots (the kernel above) are robust but poll more per
    // round and gain nothing (128^3 796 / 814 / 866 ms at 1 / 2 / 4 rows; issuing the slots'
    // readiness loads together per round: 864 / 1027 ms), so 1 row per lane.  The back-off
    // cap (256 ns) is flat: 32-512 ns give 3.03-3.12 ms per lower sweep.
    static const int rpt = getenv("SPARSEB200_TRSV_RPT") ? atoi(getenv("SPARSEB200_TRSV_RPT")) : 1;
    // Mode 2 (default): polling with the value as its own flag (IC-CG 128^3 866 -> 804 ms,
    // 96^3 282 -> 261, 64^3 84 -> 78; ILU-GMRES 64^3 118 -> 109); 1: polling with separate
    // ready flags (also used when x overlaps b); 0: blocking spin.
    static const int mode = getenv("SPARSEB200_TRSV_MODE") ? atoi(getenv("SPARSEB200_TRSV_MODE")) : 2;
    const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)device_info().sms * 8);
    // value-as-flag needs x disjoint from b (the sentinel fill would clobber b)
    const char *xb = (const char *)x, *bb = (const char *)b;
    const size_t span = (size_t)((n - 1) * ldx + 1) * sizeof(V);
    const size_t bspan = (size_t)((n - 1) * ldb + 1) * sizeof(V);
    const bool disjoint = xb + span <= bb || bb + bspan <= xb;
    const bool vf = mode == 2 && disjoint;
    if (!vf) {
        e = cudaMemsetAsync(w.ready, 0, sizeof(int) * (size_t)n, st);
        if (e != cudaSuccess) return e;
    } else {
        tri_sentinel_fill_kernel<V><<<(int)std::min<int64_t>(ceil_div(n, 256), (int64_t)device_info().sms * 16), 256, 0, st>>>(
            n, x, ldx, ctl, skip_mode);
    }
    auto go = [&](auto lower_c, auto rpt_c) {
        if (vf)
            sptrsv_poll_kernel<V, I, decltype(lower_c)::value, decltype(rpt_c)::value, true><<<grid, 256, 0, st>>>(
                n, (const I *)T.row_ptrs, (const I *)T.col_idxs, (const V *)T.values, b, ldb, x, ldx,
                (lower && unit) ? 1 : 0, w, ctl, skip_mode);
        else if (mode >= 1)
            sptrsv_poll_kernel<V, I, decltype(lower_c)::value, decltype(rpt_c)::value><<<grid, 256, 0, st>>>(
                n, (const I *)T.row_ptrs, (const I *)T.col_idxs, (const V *)T.values, b, ldb, x, ldx,
                (lower && unit) ? 1 : 0, w, ctl, skip_mode);
        else
            sptrsv_kernel<V, I, decltype(lower_c)::value, decltype(rpt_c)::value><<<grid, 256, 0, st>>>(
                n, (const I *)T.row_ptrs, (const I *)T.col_idxs, (const V *)T.values, b, ldb, x, ldx,
                (lower && unit) ? 1 : 0, w, ctl, skip_mode);
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    using R1 = std::integral_constant<int, 1>;
    using R2 = std::integral_constant<int, 2>;
    using R4 = std::integral_constant<int, 4>;
    using R8 = std::integral_constant<int, 8>;
    if (lower) {
        if (rpt == 8) go(T_{}, R8{});
        else if (rpt == 4) go(T_{}, R4{});
        else if (rpt == 2) go(T_{}, R2{});
        else go(T_{}, R1{});
    } else {
        if (rpt == 8) go(F_{}, R8{});
        else if (rpt == 4) go(F_{}, R4{});
        else if (rpt == 2) go(F_{}, R2{});
        else go(F_{}, R1{});
    }
    return cudaGetLastError();
}

// Structure / diagonal check of one factor in solve order, synchronous: returns
// SB_ERR_NOT_TRIANGULAR / SB_ERR_SINGULAR_TRIANGLE with the reference's row.
template <class V, class I>
sb_status tri_factor_check(const sb_csr &T, bool lower, bool unit, const TriWs &w, cudaStream_t st, sb_error *err) {
    const int64_t n = T.rows;
    if (n == 0) return SB_OK;
    SB_CUDA(cudaMemsetAsync(w.err, 0xff, sizeof(unsigned long long), st));
    const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)device_info().sms * 8);
    tri_check_kernel<V, I><<<grid, 256, 0, st>>>(n, (const I *)T.row_ptrs, (const I *)T.col_idxs,
                                                 (const V *)T.values, lower ? 1 : 0, unit ? 1 : 0, w.err);
    SB_CUDA(cudaGetLastError());
    unsigned long long key = 0;
    SB_CUDA(cudaMemcpyAsync(&key, w.err, sizeof(key), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    if (key == ~0ull) return SB_OK;
    const int64_t pos = (int64_t)(key >> 2), row = lower ? pos : n - 1 - pos;
    if (err) err->row = row;
    if ((key & 3) == 1)
        return fail(err, SB_ERR_NOT_TRIANGULAR, "entry %s the diagonal in row %lld", lower ? "above" : "below",
                    (long long)row);
    return fail(err, SB_ERR_SINGULAR_TRIANGLE, "zero or missing diagonal in row %lld", (long long)row);
}

template <class V, class I>
sb_status tri_precond_check(const sb_tri_precond &m, sb_error *err, cudaStream_t st) {
    const int64_t n = m.l->rows;
    if (m.l->rows != m.l->cols || m.u->rows != m.u->cols || m.u->rows != n)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "triangular factors must be square and of one size");
    const TriWs w = carve_tri_ws(m.workspace, n);
    sb_status s = tri_factor_check<V, I>(*m.l, true, m.l_unit != 0, w, st, err);
    if (s != SB_OK) return s;
    return tri_factor_check<V, I>(*m.u, false, false, w, st, err);
}

}  // namespace sb
