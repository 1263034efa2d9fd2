// spmv.cuh -- sm_100a SpMV kernels for CSR / COO / ELL / SELL-P / Hybrid.
//
// Reference semantics: linop.spmv_csr / spmv_coo (linop.py:102-159) ->
// _kernels.spmv_csr_rows / spmv_coo_entries (_kernels.py:62-88): x[i] is the fp64
// sum of the row's products, written with one rounding to the value type; rows with
// no entries write 0.
//
// Kernels that own whole rows (strict, stream, vector, ELL, SELL-P) take an
// epilogue `Epi` that receives (row, fp64 sum): the plain store, or a solver
// epilogue that also accumulates a fused dot product (e.g. CG's p.Ap) and finalises
// it with a deterministic grid reduction.  Row-splitting kernels (merge-path CSR,
// segmented COO) write x and are followed by a carry fix-up pass.
//
// Row-accumulation order:
//   strict / stream / ELL / SELL-P: sequential in stored order -> bitwise equal to
//     the reference for every value type (the stream kernel is the production path
//     for regular matrices such as the Poisson configs);
//   vector / merge / COO: per-lane or per-thread sequential partials combined by a
//     fixed tree -> deterministic, within the 1e-12 / 1e-5 scale tolerance.
#pragma once

#include <type_traits>
#include <utility>

#include "common.cuh"

namespace sb {

// ============================================================ epilogues
// Optional epilogue hooks, detected at compile time:
//   prepare()   per-launch setup in every CTA (e.g. scalars read from a solver's
//               control block once, not per row);
//   gather(off) the gathered operand computed on the fly instead of loaded from b
//               (CG's search direction p = z + beta p, fused into the SpMV that
//               consumes it).  Only the row-owning kernels (strict / stream / vector /
//               ELL / SELL-P) honour it; the launchers reject it for the others.
template <class E, class = void>
struct epi_has_gather : std::false_type {};
template <class E>
struct epi_has_gather<E, std::void_t<decltype(std::declval<const E &>().gather(int64_t(0)))>>
    : std::true_type {};
template <class E, class = void>
struct epi_has_prepare : std::false_type {};
template <class E>
struct epi_has_prepare<E, std::void_t<decltype(std::declval<E &>().prepare())>> : std::true_type {};

// Epilogues that gather through a hook carry more live registers; such an epilogue may
// ask the TMA-staged kernels for a minimum residency (kMinThreadsPerSM / R CTAs per SM)
// so the register allocator keeps four 256-row CTAs resident.
template <class E, class = void>
struct epi_min_threads : std::integral_constant<int, 0> {};
template <class E>
struct epi_min_threads<E, std::void_t<decltype(E::kMinThreadsPerSM)>>
    : std::integral_constant<int, E::kMinThreadsPerSM> {};
template <class Epi>
constexpr int epi_min_ctas(int R) {
    return epi_min_threads<Epi>::value / R;  // 0 = unspecified (the compiler's own heuristic)
}

// partial-sum type of an epilogue's fused dots: double, or CAcc (compensated) when the
// epilogue declares `using part_type = CAcc;`
template <class E, class = void>
struct epi_part {
    using type = double;
};
template <class E>
struct epi_part<E, std::void_t<typename E::part_type>> {
    using type = typename E::part_type;
};
template <class E>
using epi_part_t = typename epi_part<E>::type;

template <class Epi, class V>
__device__ __forceinline__ V gather_b(const Epi &e, const V *__restrict__ b, int64_t off) {
    if constexpr (epi_has_gather<Epi>::value) return e.gather(off);
    else return __ldg(b + off);
}
// column offset into b: unit stride (the common single-vector case) as its own
// instantiation, so the gather is one wide multiply-add instead of a 64-bit multiply
template <bool U1>
__device__ __forceinline__ int64_t bidx(int64_t c, int64_t ldb) {
    if constexpr (U1) return c;
    else return c * ldb;
}
template <class Epi>
__device__ __forceinline__ void epi_prepare(Epi &e) {
    if constexpr (epi_has_prepare<Epi>::value) e.prepare();
}

template <class V>
struct EpiStore {
    static constexpr int N = 1;  // no reduction; N=1 only sizes the (unused) partial array
    V *x;
    int64_t ldx;
    __device__ __forceinline__ bool skip() const { return false; }
    __device__ __forceinline__ void row(int64_t i, double acc, double (&)[N]) const {
        x[i * ldx] = (V)acc;
    }
    __device__ __forceinline__ void finish(double (&)[N]) const {}
};

// ============================================================ CSR: strict (device oracle)
// One thread per row straight from global memory: the reference loop verbatim.
template <class V, class I, class Epi>
__global__ void __launch_bounds__(256) csr_strict_kernel(int64_t rows, const I *__restrict__ rp,
                                                         const I *__restrict__ ci,
                                                         const V *__restrict__ val,
                                                         const V *__restrict__ b, int64_t ldb,
                                                         Epi epi) {
    if (epi.skip()) return;
    epi_prepare(epi);
    epi_part_t<Epi> part[Epi::N] = {};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int64_t k = rp[i]; k < (int64_t)rp[i + 1]; ++k)
            acc = addd(acc, mulp(val[k], gather_b(epi, b, (int64_t)ci[k] * ldb)));
        epi.row(i, acc, part);
    }
    epi.finish(part);
}

// ============================================================ CSR: stream (TMA-staged)
// Persistent CTAs walk fixed blocks of R rows.  For each block one elected thread
// issues 1-D TMA bulk copies (cp.async.bulk, completion on an mbarrier) of the
// block's row_ptrs slice and its contiguous value / column ranges into a two-stage
// shared-memory ring, prefetching block k+1 while block k is consumed.  Each thread
// then reduces one row sequentially from shared memory (gathering b through L1/L2),
// which reproduces the reference's accumulation order exactly.
template <class V, class I>
struct StreamLayout {
    static constexpr int VV = 16 / sizeof(V);
    static constexpr int VI = 16 / sizeof(I);
    int cap_v, cap_c, cap_r;  // elements per stage
    __host__ __device__ StreamLayout(int R, int nnz_cap) {
        // + 8: the row-tail reads of the stream kernel run up to 7 entries past a row's end
        cap_v = (nnz_cap + 2 * VV + 8 + 3) & ~3;
        cap_c = (nnz_cap + 2 * VI + 8 + 3) & ~3;
        cap_r = (R + 1 + 2 * VI + 3) & ~3;
    }
    __host__ __device__ size_t stage_bytes() const {
        size_t b = (size_t)cap_v * sizeof(V);
        b = (b + 15) & ~size_t(15);
        b += (size_t)cap_c * sizeof(I);
        b = (b + 15) & ~size_t(15);
        b += (size_t)cap_r * sizeof(I);
        return (b + 15) & ~size_t(15);
    }
    __host__ __device__ size_t off_c() const { return ((size_t)cap_v * sizeof(V) + 15) & ~size_t(15); }
    __host__ __device__ size_t off_r() const {
        return (off_c() + (size_t)cap_c * sizeof(I) + 15) & ~size_t(15);
    }
};

struct StreamMeta {
    int64_t r0, r1, av, ac, ar;  // block rows [r0, r1); smem bases (global element index of slot 0)
};

template <class T>
__device__ __forceinline__ uint32_t stage_range(const T *g, int64_t lo, int64_t hi, int64_t len,
                                                T *s, int64_t &base) {
    // copy g[lo, hi) (hi <= len) into s, starting at the 16-byte aligned element `base`;
    // returns the bulk bytes issued (the unaligned tail beyond len's last full vector is
    // copied with scalar loads).
    constexpr int VE = 16 / sizeof(T);
    base = lo & ~(int64_t)(VE - 1);
    const int64_t full_end = len & ~(int64_t)(VE - 1);
    int64_t bulk_end = (hi + VE - 1) & ~(int64_t)(VE - 1);
    if (bulk_end > full_end) bulk_end = full_end;
    if (bulk_end < base) bulk_end = base;
    for (int64_t e = bulk_end; e < hi; ++e) s[e - base] = g[e];
    return (uint32_t)((bulk_end - base) * (int64_t)sizeof(T));
}

template <class V, class I, int R, class Epi, int NS = 2>
__global__ void __launch_bounds__(R, epi_min_ctas<Epi>(R)) csr_stream_kernel(int64_t rows, int64_t nnz,
                                                       const I *__restrict__ rp,
                                                       const I *__restrict__ ci,
                                                       const V *__restrict__ val,
                                                       const V *__restrict__ b, int64_t ldb,
                                                       int nnz_cap, Epi epi) {
    extern __shared__ __align__(128) unsigned char smem[];
    static_assert(NS >= 2 && NS <= 4, "stages");
    __shared__ __align__(8) uint64_t bar[NS];
    __shared__ StreamMeta meta[NS];
    const StreamLayout<V, I> L(R, nnz_cap);
    const size_t sb = L.stage_bytes();
    const int tid = threadIdx.x;
    const int64_t nblk = (rows + R - 1) / R;
    const uint64_t pol = policy_evict_first();

    if (tid == 0) {
        for (int q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    __syncthreads();

    // the row-pointer bounds of a block are loaded one block before its issue (thread 0
    // would otherwise start every block one L2 round trip behind the other threads)
    auto bounds = [&](int64_t blk, int64_t &k0, int64_t &k1) {
        const int64_t r0 = blk * R, r1 = r0 + R < rows ? r0 + R : rows;
        k0 = rp[r0];
        k1 = rp[r1];
    };
    auto issue = [&](int64_t blk, int s, int64_t k0, int64_t k1) {  // thread 0 only
        unsigned char *st = smem + s * sb;
        V *sv = reinterpret_cast<V *>(st);
        I *sc = reinterpret_cast<I *>(st + L.off_c());
        I *sr = reinterpret_cast<I *>(st + L.off_r());
        const int64_t r0 = blk * R, r1 = r0 + R < rows ? r0 + R : rows;
        StreamMeta m;
        m.r0 = r0;
        m.r1 = r1;
        uint32_t bv = stage_range(val, k0, k1, nnz, sv, m.av);
        uint32_t bc = stage_range(ci, k0, k1, nnz, sc, m.ac);
        uint32_t br = stage_range(rp, r0, r1 + 1, rows + 1, sr, m.ar);
        meta[s] = m;
        mbar_arrive_expect_tx(&bar[s], bv + bc + br);
        if (bv) bulk_g2s(sv, val + m.av, bv, &bar[s], pol);
        if (bc) bulk_g2s(sc, ci + m.ac, bc, &bar[s], pol);
        if (br) bulk_g2s(sr, rp + m.ar, br, &bar[s], pol);
    };

    // the first block's matrix ranges are immutable: their TMA copies are issued before
    // waiting on the predecessor kernel (programmatic dependent launch)
    int64_t blk = blockIdx.x;
    int64_t nk0 = 0, nk1 = 0;  // bounds of the next block to issue (thread 0)
    if (tid == 0) {
        for (int q = 0; q < NS - 1; ++q)
            if (blk + (int64_t)q * gridDim.x < nblk) {
                bounds(blk + (int64_t)q * gridDim.x, nk0, nk1);
                issue(blk + (int64_t)q * gridDim.x, q, nk0, nk1);
            }
        if (blk + (int64_t)(NS - 1) * gridDim.x < nblk) bounds(blk + (int64_t)(NS - 1) * gridDim.x, nk0, nk1);
    }
    pdl_wait();
    pdl_trigger();
    if (epi.skip()) {
        if (tid == 0)  // no bulk copy outlives the CTA
            for (int q = 0; q < NS - 1; ++q)
                if (blk + (int64_t)q * gridDim.x < nblk) mbar_wait(&bar[q], 0);
        return;
    }
    epi_prepare(epi);
    const bool unit = ldb == 1;
    epi_part_t<Epi> part[Epi::N] = {};
    for (int it = 0; blk < nblk; blk += gridDim.x, ++it) {
        const int s = it % NS;
        const uint32_t parity = (it / NS) & 1;
        if (tid == 0 && blk + (int64_t)(NS - 1) * gridDim.x < nblk) {
            const int64_t bi = blk + (int64_t)(NS - 1) * gridDim.x;
            issue(bi, (it + NS - 1) % NS, nk0, nk1);
            if (bi + gridDim.x < nblk) bounds(bi + gridDim.x, nk0, nk1);
        }
        mbar_wait(&bar[s], parity);
        const unsigned char *st = smem + s * sb;
        const V *sv = reinterpret_cast<const V *>(st);
        const I *sc = reinterpret_cast<const I *>(st + L.off_c());
        const I *sr = reinterpret_cast<const I *>(st + L.off_r());
        const StreamMeta m = meta[s];
        const int64_t i = m.r0 + tid;
        if (i < m.r1) {
            // 32-bit stage offsets of the row (the stage holds < 2^31 entries); the column
            // gathers of a unit-stride b are one wide multiply-add each (the strided form
            // is a separate instantiation, so the loop carries no 64-bit multiply)
            const int64_t kb = sr[i - m.ar], ke = sr[i + 1 - m.ar];
            const int ov = (int)(kb - m.av), oc = (int)(kb - m.ac), cnt = (int)(ke - kb);
            auto rowsum = [&](auto unit_tag) -> double {
                constexpr bool U1 = decltype(unit_tag)::value;
                auto off = [&](int64_t c) -> int64_t {
                    if constexpr (U1) return c;
                    else return c * ldb;
                };
                double acc = 0.0;
                int t = 0;
                for (; t + 8 <= cnt; t += 8) {
                    V vv[8], bb[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        vv[j] = sv[ov + t + j];
                        bb[j] = gather_b(epi, b, off((int64_t)sc[oc + t + j]));
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc = addd(acc, mulp(vv[j], bb[j]));
                }
                if (t < cnt) {
                    // branch-free tail: lanes past the row end gather the row's last column
                    // again (an L1 hit) and are masked at the ordered adds, so every gather
                    // of the row is in flight before the first add (a gather hook that
                    // computes on the loaded values would otherwise serialise one latency
                    // per entry).  The stage reads run past the row end at fixed offsets
                    // from one base (StreamLayout's + 8 slack): no per-entry index clamp or
                    // address arithmetic (fp32 128^3: ~39 -> fewer instructions per entry)
                    const V *pv = sv + ov + t;
                    const I *pc = sc + oc + t;
                    const int rem = cnt - t;
                    const int64_t clast = (int64_t)pc[rem - 1];
                    V vv[8], bb[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        vv[j] = pv[j];
                        const int64_t c = j < rem ? (int64_t)pc[j] : clast;
                        bb[j] = gather_b(epi, b, off(c));
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < rem) acc = addd(acc, mulp(vv[j], bb[j]));
                }
                return acc;
            };
            const double acc = unit ? rowsum(std::true_type{}) : rowsum(std::false_type{});
            epi.row(i, acc, part);
        }
        __syncthreads();  // stage s fully consumed before it is re-issued
    }
    epi.finish(part);
}

// ============================================================ CSR: stream SpMM (multi-RHS)
// x[:, 0:K] = A b[:, 0:K] (b, x row-major with leading dimensions ldb, ldx): the stream
// kernel's TMA-staged row blocks with K accumulators per thread, so the matrix streams
// once for K right-hand sides (linop.py:115 applies column by column; each column's sum
// keeps the same sequential order -> bitwise equal to K single-vector SpMVs).
template <class V, class I, int R, int K>
__global__ void __launch_bounds__(R) csr_stream_spmm_kernel(int64_t rows, int64_t nnz, const I *__restrict__ rp,
                                                            const I *__restrict__ ci, const V *__restrict__ val,
                                                            const V *__restrict__ b, int64_t ldb, V *x,
                                                            int64_t ldx, int nnz_cap) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ StreamMeta meta[2];
    const StreamLayout<V, I> L(R, nnz_cap);
    const size_t sb = L.stage_bytes();
    const int tid = threadIdx.x;
    const int64_t nblk = (rows + R - 1) / R;
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int64_t blk, int s) {
        unsigned char *st = smem + s * sb;
        V *sv = reinterpret_cast<V *>(st);
        I *sc = reinterpret_cast<I *>(st + L.off_c());
        I *sr = reinterpret_cast<I *>(st + L.off_r());
        const int64_t r0 = blk * R, r1 = r0 + R < rows ? r0 + R : rows;
        const int64_t k0 = rp[r0], k1 = rp[r1];
        StreamMeta m;
        m.r0 = r0;
        m.r1 = r1;
        uint32_t bv = stage_range(val, k0, k1, nnz, sv, m.av);
        uint32_t bc = stage_range(ci, k0, k1, nnz, sc, m.ac);
        uint32_t br = stage_range(rp, r0, r1 + 1, rows + 1, sr, m.ar);
        meta[s] = m;
        mbar_arrive_expect_tx(&bar[s], bv + bc + br);
        if (bv) bulk_g2s(sv, val + m.av, bv, &bar[s], pol);
        if (bc) bulk_g2s(sc, ci + m.ac, bc, &bar[s], pol);
        if (br) bulk_g2s(sr, rp + m.ar, br, &bar[s], pol);
    };
    int64_t blk = blockIdx.x;
    if (tid == 0 && blk < nblk) issue(blk, 0);
    for (int it = 0; blk < nblk; blk += gridDim.x, ++it) {
        const int s = it & 1;
        if (tid == 0 && blk + gridDim.x < nblk) issue(blk + gridDim.x, s ^ 1);
        mbar_wait(&bar[s], (it >> 1) & 1);
        const unsigned char *st = smem + s * sb;
        const V *sv = reinterpret_cast<const V *>(st);
        const I *sc = reinterpret_cast<const I *>(st + L.off_c());
        const I *sr = reinterpret_cast<const I *>(st + L.off_r());
        const StreamMeta m = meta[s];
        const int64_t i = m.r0 + tid;
        if (i < m.r1) {
            const int64_t kb = sr[i - m.ar], ke = sr[i + 1 - m.ar];
            double acc[K];
#pragma unroll
            for (int j = 0; j < K; ++j) acc[j] = 0.0;
            for (int64_t k = kb; k < ke; k += 4) {
                V vv[4], bb[4][K];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t kk = k + u < ke ? k + u : ke - 1;
                    vv[u] = sv[kk - m.av];
                    const V *bp = b + (int64_t)sc[kk - m.ac] * ldb;
#pragma unroll
                    for (int j = 0; j < K; ++j) bb[u][j] = __ldg(bp + j);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (k + u < ke)
#pragma unroll
                        for (int j = 0; j < K; ++j) acc[j] = addd(acc[j], mulp(vv[u], bb[u][j]));
            }
#pragma unroll
            for (int j = 0; j < K; ++j) x[i * ldx + j] = (V)acc[j];
        }
        __syncthreads();
    }
}

// ============================================================ CSR: vector (sub-warp per row)
// S lanes per row (S in 2..32 chosen from the mean row length), strided partials,
// fixed shuffle tree.
template <class V, class I, int S, class Epi>
__global__ void __launch_bounds__(256) csr_vector_kernel(int64_t rows, const I *__restrict__ rp,
                                                         const I *__restrict__ ci,
                                                         const V *__restrict__ val,
                                                         const V *__restrict__ b, int64_t ldb,
                                                         Epi epi) {
    if (epi.skip()) return;
    epi_prepare(epi);
    epi_part_t<Epi> part[Epi::N] = {};
    const int lane = threadIdx.x % S;
    const int64_t group = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / S;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / S;
    const int64_t trips = (rows + ngroups - 1) / ngroups;  // uniform trip count keeps shuffles converged
    for (int64_t t = 0; t < trips; ++t) {
        const int64_t i = group + t * ngroups;
        double acc = 0.0;
        if (i < rows) {
            const int64_t kb = rp[i], ke = rp[i + 1];
            int64_t k = kb + lane;
            for (; k + 3 * S < ke; k += 4 * S) {  // four independent gathers in flight
                I c[4];
                V v[4], g[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    c[u] = ld_stream(ci + k + u * S);
                    v[u] = ld_stream(val + k + u * S);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) g[u] = gather_b(epi, b, (int64_t)c[u] * ldb);
#pragma unroll
                for (int u = 0; u < 4; ++u) acc = addd(acc, mulp(v[u], g[u]));
            }
            for (; k < ke; k += S)
                acc = addd(acc, mulp(ld_stream(val + k), gather_b(epi, b, (int64_t)ld_stream(ci + k) * ldb)));
        }
#pragma unroll
        for (int o = S / 2; o > 0; o >>= 1) acc = addd(acc, __shfl_down_sync(0xffffffffu, acc, o, S));
        if (lane == 0 && i < rows) epi.row(i, acc, part);
    }
    epi.finish(part);
}

// ============================================================ reduce-by-key block scan
// Inclusive scan of (key, value) pairs in thread order with
//   (k1, v1) (+) (k2, v2) = (k2, k1 == k2 ? v1 + v2 : v2)
// (keys are non-decreasing across threads).  Returns the inclusive pair in
// (key, val) and the exclusive pair (the previous thread's inclusive pair) in
// (ex_key, ex_val).  Fixed combination tree -> deterministic.
template <int NT>
__device__ __forceinline__ void scan_by_key(int64_t &key, double &val, int64_t &ex_key,
                                            double &ex_val) {
    static_assert(NT % 32 == 0 && NT <= 1024, "block size");
    __shared__ int64_t s_k[NT / 32];
    __shared__ double s_v[NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t k2 = __shfl_up_sync(0xffffffffu, key, o);
        const double v2 = __shfl_up_sync(0xffffffffu, val, o);
        if (lane >= o && k2 == key) val = addd(v2, val);
    }
    if (lane == 31) {
        s_k[warp] = key;
        s_v[warp] = val;
    }
    __syncthreads();
    if (warp == 0) {
        int64_t wk = lane < NT / 32 ? s_k[lane] : INT64_MAX;
        double wv = lane < NT / 32 ? s_v[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t k2 = __shfl_up_sync(0xffffffffu, wk, o);
            const double v2 = __shfl_up_sync(0xffffffffu, wv, o);
            if (lane >= o && k2 == wk) wv = addd(v2, wv);
        }
        if (lane < NT / 32) {
            s_k[lane] = wk;
            s_v[lane] = wv;
        }
    }
    __syncthreads();
    const int64_t pk = warp > 0 ? s_k[warp - 1] : INT64_MIN;
    const double pv = warp > 0 ? s_v[warp - 1] : 0.0;
    // keys are non-decreasing, so an equal key in the previous warps' aggregate means this
    // thread's run started there (and its in-warp aggregate covers lanes 0..lane)
    if (pk == key) val = addd(pv, val);
    int64_t ek = __shfl_up_sync(0xffffffffu, key, 1);
    double ev = __shfl_up_sync(0xffffffffu, val, 1);
    if (lane == 0) {
        ek = pk;
        ev = pv;
    }
    ex_key = ek;
    ex_val = ev;
    __syncthreads();  // s_k / s_v reusable by the next call
}

// Products of a tile's nonzeros into shared memory with every load of a thread issued
// before any is used: IPT coalesced (col, val) pairs, then IPT independent gathers of b
// (the random gathers of irregular matrices are latency-bound without this MLP).
template <class V, class I, int NT, int IPT>
__device__ __forceinline__ void stage_products(const I *__restrict__ ci, const V *__restrict__ val,
                                               int64_t count, const V *__restrict__ b, int64_t ldb,
                                               double *s_prod) {
    I cc[IPT];
    V vv[IPT], bb[IPT];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const int64_t j = threadIdx.x + (int64_t)u * NT;
        if (j < count) {
            cc[u] = ld_stream(ci + j);
            vv[u] = ld_stream(val + j);
        }
    }
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const int64_t j = threadIdx.x + (int64_t)u * NT;
        if (j < count) bb[u] = __ldg(b + (int64_t)cc[u] * ldb);
    }
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const int64_t j = threadIdx.x + (int64_t)u * NT;
        if (j < count) s_prod[j] = mulp(vv[u], bb[u]);
    }
}

// ============================================================ CSR: merge-path
// Load-balanced: every tile owns exactly NT*IPT merge items (row ends + nonzeros),
// so a CTA's work is independent of the row-length distribution.  Tile start
// coordinates come from the plan (merge_path_partition_kernel).  Products are
// staged in shared memory, each thread walks IPT items sequentially, partial rows
// are joined by a block reduce-by-key scan, and a tile's unfinished last row is
// handed to the carry fix-up kernel.
template <class I>
__device__ __forceinline__ int64_t merge_search(int64_t diag, const I *a, int64_t a_len, int64_t b0,
                                                int64_t b_len) {
    // CUB-style MergePathSearch of list a (row ends) against b = b0, b0+1, ...:
    // the number of a-items consumed after `diag` merge steps.
    int64_t lo = diag - b_len > 0 ? diag - b_len : 0;
    int64_t hi = diag < a_len ? diag : a_len;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)a[mid] <= b0 + diag - mid - 1) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <class I>
__global__ void merge_path_partition_kernel(int64_t rows, int64_t nnz, const I *__restrict__ rp,
                                            int64_t items_per_tile, int64_t num_tiles,
                                            int64_t *tile_rows, int64_t *tile_nnz) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t > num_tiles) return;
    int64_t diag = t * items_per_tile;
    if (diag > rows + nnz) diag = rows + nnz;
    const int64_t x = merge_search(diag, rp + 1, rows, 0, nnz);
    tile_rows[t] = x;
    tile_nnz[t] = diag - x;
}

template <class V, class I, int NT, int IPT>
__global__ void __launch_bounds__(NT) csr_merge_kernel(int64_t rows, const I *__restrict__ rp,
                                                       const I *__restrict__ ci,
                                                       const V *__restrict__ val,
                                                       const V *__restrict__ b, int64_t ldb, V *x,
                                                       int64_t ldx, const int64_t *tile_rows,
                                                       const int64_t *tile_nnz, int64_t num_tiles,
                                                       int64_t *carry_rows, double *carry_vals) {
    constexpr int TILE = NT * IPT;
    __shared__ I s_end[TILE + 1];
    __shared__ double s_prod[TILE];
    __shared__ double s_out[TILE];
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int64_t row_s = tile_rows[tile], k_s = tile_nnz[tile];
        const int64_t row_e = tile_rows[tile + 1], k_e = tile_nnz[tile + 1];
        const int64_t nA = row_e - row_s, nB = k_e - k_s;
        const int64_t nload = (row_e + 1 < rows ? row_e + 1 : rows) - row_s;  // ends of rows row_s..row_e
        for (int64_t j = threadIdx.x; j < nload; j += NT) s_end[j] = rp[row_s + j + 1];
        stage_products<V, I, NT, IPT>(ci + k_s, val + k_s, nB, b, ldb, s_prod);
        __syncthreads();
        const int64_t total = nA + nB;
        const int64_t d0 = (int64_t)threadIdx.x * IPT;
        int64_t r = nA;
        bool emitted = false;
        int64_t first_row = -1;
        double acc = 0.0;
        if (d0 < total) {
            r = merge_search(d0, s_end, nA, k_s, nB);
            int64_t k = k_s + d0 - r;
            for (int it = 0; it < IPT && d0 + it < total; ++it) {
                if (r < nload && k < (int64_t)s_end[r]) {
                    acc = addd(acc, s_prod[k - k_s]);
                    ++k;
                } else {
                    s_out[r] = acc;
                    if (!emitted) {
                        emitted = true;
                        first_row = r;
                    }
                    acc = 0.0;
                    ++r;
                }
            }
        }
        int64_t key = r, ex_key;
        double cv = acc, ex_val;
        scan_by_key<NT>(key, cv, ex_key, ex_val);
        if (emitted && ex_key == first_row) s_out[first_row] = addd(ex_val, s_out[first_row]);
        __syncthreads();
        for (int64_t j = threadIdx.x; j < nA; j += NT) x[(row_s + j) * ldx] = (V)s_out[j];
        if (threadIdx.x == NT - 1) {
            // inclusive total over the tile = this tile's partial of row row_e (idle threads
            // carry key nA, so the scan propagates it to the last thread)
            const int64_t consumed = nA > 0 ? k_e - (int64_t)s_end[nA - 1] : nB;
            const bool carry = row_e < rows && consumed > 0;
            carry_rows[tile] = carry ? row_e : -1;
            carry_vals[tile] = carry ? cv : 0.0;
        }
        __syncthreads();
    }
}

// ============================================================ CSR: nnz tiles
// Tile t = nonzeros [t C, (t+1) C): exactly C nonzeros per tile whatever the row lengths.
// One elected thread TMA-copies the row pointers of the rows starting in the tile
// (first_row[t] .. first_row[t+1], known one tile ahead) -- and, in the staged variant,
// the tile's values and columns -- into a two-stage shared ring, the next tile
// prefetched.  All threads then form the tile's products with every gather of a thread
// in flight at once (random gathers are bound by the L1/L2 sector rate, ~270 G/s on
// B200, tools/micro/gather_bench.cu); the default "direct" variant reads values and
// columns with coalesced streaming loads instead of staging them, which halves the
// shared footprint (more CTAs, more gathers in flight per SM).  Products go to shared
// memory (an fp32 product is exact in fp32).  Rows starting in the tile are reduced
// from shared memory: segments of <= 32 products by one thread in stored order (a row
// wholly inside the tile is then bitwise the reference's sum), longer ones by a warp
// (lane-strided partials, fixed shuffle tree).  A row crossing tile boundaries is not
// written by any tile: its owner emits a "trail" record (row, first-segment sum) and
// every later tile it reaches a "lead" record; tile_carry_fixup_kernel sums each row's
// records in nnz order.  Deterministic, no atomics on values.
struct TileMeta {
    int64_t r0, r1;      // rows starting in the tile
    int64_t dv, dc, dr;  // stage slot of the first value / column / row pointer
    int32_t staged_rp;   // row pointers r0 .. r1 staged (else read from global)
};

template <class V, class I, int C, int RCAP, bool DIRECT = false>
struct TileLayout;
template <class V, class I, int C, int RCAP>
struct TileLayout<V, I, C, RCAP, true> {  // stages hold the row pointers only
    static constexpr int VI = 16 / sizeof(I);
    static constexpr size_t OFF_C = 0, OFF_R = 0;
    static constexpr size_t STAGE = ((size_t)(RCAP + 1 + 2 * VI) * sizeof(I) + 15) & ~size_t(15);
    static constexpr size_t SMEM = 2 * STAGE + (size_t)C * sizeof(V);  // + one product buffer
};
template <class V, class I, int C, int RCAP>
struct TileLayout<V, I, C, RCAP, false> {
    static constexpr int VV = 16 / sizeof(V), VI = 16 / sizeof(I);
    static constexpr size_t OFF_C = ((size_t)(C + 2 * VV) * sizeof(V) + 15) & ~size_t(15);
    static constexpr size_t OFF_R = (OFF_C + (size_t)(C + 2 * VI) * sizeof(I) + 15) & ~size_t(15);
    static constexpr size_t STAGE = (OFF_R + (size_t)(RCAP + 1 + 2 * VI) * sizeof(I) + 15) & ~size_t(15);
    static constexpr size_t SMEM = 2 * STAGE;
};

// Per tile: wait for the stage, products (barrier), owned rows by threads with long
// segments queued (barrier), queued segments by warps, record slots (barrier).
struct TileJob {
    int32_t rel;     // owned-row index relative to first_row[t], or -1 for the lead segment
    int32_t kb, ke;  // product range in the tile
};

// fp32 direct tiles are capped to 32 registers for 8 CTAs per SM (350 -> 333 us on config
// #3); the same cap makes fp64 slower (381 -> 745 us), which keeps the compiler's choice
template <class V, class I, int NT, int C, int RCAP, bool DIRECT = false, int PF = 0, bool U1 = false>
__global__ void __launch_bounds__(NT, (DIRECT && sizeof(V) == 4) ? 2048 / NT : 0) csr_tile_kernel(int64_t rows, int64_t nnz, const I *__restrict__ rp,
                                                       const I *__restrict__ ci, const V *__restrict__ val,
                                                       const V *__restrict__ b, int64_t ldb, V *x, int64_t ldx,
                                                       const int64_t *__restrict__ first_row, int64_t ntiles,
                                                       int64_t *crow, double *cval) {
    using L = TileLayout<V, I, C, RCAP, DIRECT>;
    constexpr int MAXJ = C / 33 + 4;
    constexpr int PER = C / NT;
    static_assert(C % NT == 0, "tile size");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ TileMeta s_meta[2];
    __shared__ TileJob s_jobs[MAXJ];
    __shared__ int s_njobs;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int64_t t, int64_t r0, int64_t r1, int s) {  // thread 0
        unsigned char *st = smem + s * L::STAGE;
        V *sv = reinterpret_cast<V *>(st);
        I *sc = reinterpret_cast<I *>(st + L::OFF_C);
        I *sr = reinterpret_cast<I *>(st + L::OFF_R);
        const int64_t k0 = t * C, k1 = k0 + C < nnz ? k0 + C : nnz;
        int64_t bv0 = k0, bc0 = k0, br0 = 0;
        // DIRECT: values / columns are read by the product phase with coalesced streaming
        // loads (no stage for them: more CTAs per SM); only the row pointers are staged
        const uint32_t bv = DIRECT ? 0u : stage_range(val, k0, k1, nnz, sv, bv0);
        const uint32_t bc = DIRECT ? 0u : stage_range(ci, k0, k1, nnz, sc, bc0);
        const bool srp = RCAP > 0 && r1 - r0 <= RCAP;
        const uint32_t br = srp ? stage_range(rp, r0, r1 + 1, rows + 1, sr, br0) : 0;
        s_meta[s] = TileMeta{r0, r1, k0 - bv0, k0 - bc0, r0 - br0, srp};
        mbar_arrive_expect_tx(&bar[s], bv + bc + br);
        if (bv) bulk_g2s(sv, val + bv0, bv, &bar[s], pol);
        if (bc) bulk_g2s(sc, ci + bc0, bc, &bar[s], pol);
        if (br) bulk_g2s(sr, rp + br0, br, &bar[s], pol);
    };
    int64_t t = blockIdx.x;
    int64_t nr0 = 0, nr1 = 0;
    if (tid == 0 && t < ntiles) {
        issue(t, first_row[t], first_row[t + 1], 0);
        if (t + gridDim.x < ntiles) {
            nr0 = first_row[t + gridDim.x];
            nr1 = first_row[t + gridDim.x + 1];
        }
    }
    for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
        const int s = it & 1;
        if (tid == 0) {
            s_njobs = 0;
            const int64_t tn = t + gridDim.x;
            if (tn < ntiles) {
                issue(tn, nr0, nr1, s ^ 1);
                if (tn + gridDim.x < ntiles) {
                    nr0 = first_row[tn + gridDim.x];
                    nr1 = first_row[tn + gridDim.x + 1];
                }
            }
        }
        if (DIRECT && PF > 0 && tid == 32) {  // values / columns of the tile PF rounds ahead into L2
            const int64_t tp = t + (int64_t)PF * gridDim.x;
            if (tp < ntiles) {
                const int64_t a = tp * C, e = a + C < nnz ? a + C : nnz;
                l2_prefetch_range(val + a, val + e);
                l2_prefetch_range(ci + a, ci + e);
            }
        }
        mbar_wait(&bar[s], (it >> 1) & 1);
        unsigned char *st = smem + s * L::STAGE;
        const TileMeta m = s_meta[s];
        // DIRECT: one product buffer after the two row-pointer stages
        V *sv = DIRECT ? reinterpret_cast<V *>(smem + 2 * L::STAGE) : reinterpret_cast<V *>(st) + m.dv;
        const I *sc = reinterpret_cast<const I *>(st + L::OFF_C) + m.dc;
        const I *sr = reinterpret_cast<const I *>(st + L::OFF_R) + m.dr;
        const int64_t k0 = t * C, k1 = k0 + C < nnz ? k0 + C : nnz;
        const int cnt = (int)(k1 - k0);
        if constexpr (DIRECT) {
            I cc[PER];
            V vv[PER], bb[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = tid + u * NT;
                const int jj = j < cnt ? j : cnt - 1;
                cc[u] = ld_stream(ci + k0 + jj);
                vv[u] = ld_stream(val + k0 + jj);
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) bb[u] = __ldg(b + bidx<U1>((int64_t)cc[u], ldb));
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = tid + u * NT;
                if (j < cnt) sv[j] = (V)mulp(vv[u], bb[u]);
            }
        } else {
            V bb[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = tid + u * NT;
                bb[u] = __ldg(b + bidx<U1>((int64_t)sc[j < cnt ? j : cnt - 1], ldb));
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = tid + u * NT;
                if (j < cnt) sv[j] = (V)mulp(sv[j], bb[u]);
            }
        }
        __syncthreads();
        const int64_t r0 = m.r0, r1 = m.r1;
        auto rpa = [&](int64_t i) -> int64_t {
            if (i >= rows) return nnz;
            return m.staged_rp ? (int64_t)sr[i - r0] : (int64_t)__ldg(rp + i);
        };
        const int64_t lead_end = rpa(r0);
        const bool has_lead = lead_end > k0;
        if (tid == 0 && has_lead) {
            const int e = (int)((lead_end < k1 ? lead_end : k1) - k0);
            s_jobs[atomicAdd(&s_njobs, 1)] = TileJob{-1, 0, e};
        }
        for (int64_t i = r0 + tid; i < r1; i += NT) {
            const int64_t a = rpa(i), e = rpa(i + 1);
            const int kb = (int)(a - k0), ke = (int)((e < k1 ? e : k1) - k0);
            if (ke - kb > 32) {
                s_jobs[atomicAdd(&s_njobs, 1)] = TileJob{(int)(i - r0), kb, ke};
            } else {
                double acc = 0.0;
                for (int k = kb; k < ke; ++k) acc = addd(acc, (double)sv[k]);
                if (e <= k1) {
                    x[i * ldx] = (V)acc;
                } else {
                    crow[2 * t + 1] = i;
                    cval[2 * t + 1] = acc;
                }
            }
        }
        __syncthreads();
        const int nj = s_njobs;
        for (int q = warp; q < nj; q += NT / 32) {
            const TileJob J = s_jobs[q];
            double acc = 0.0;
            for (int k = J.kb + lane; k < J.ke; k += 32) acc = addd(acc, (double)sv[k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc = addd(acc, __shfl_down_sync(0xffffffffu, acc, o));
            if (lane == 0) {
                if (J.rel < 0) {
                    crow[2 * t] = r0 - 1;
                    cval[2 * t] = acc;
                } else {
                    const int64_t i = r0 + J.rel;
                    if (k0 + J.ke < rpa(i + 1)) {
                        crow[2 * t + 1] = i;
                        cval[2 * t + 1] = acc;
                    } else {
                        x[i * ldx] = (V)acc;
                    }
                }
            }
        }
        if (tid == 0) {
            if (!has_lead) crow[2 * t] = -1;
            if (!(r1 > r0 && rpa(r1) > k1)) crow[2 * t + 1] = -1;
        }
        __syncthreads();
    }
}

// first_row[t] = first row starting at or after nonzero t*C (rows for t*C beyond every
// row start)
template <class I>
__global__ void tile_partition_kernel(int64_t rows, const I *__restrict__ rp, int64_t C, int64_t ntiles,
                                      int64_t *first_row) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    if (t == ntiles) {  // trailing empty rows (start == nnz) belong to the last tile
        first_row[t] = rows;
        return;
    }
    const int64_t key = t * C;
    int64_t lo = 0, hi = rows;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)rp[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    first_row[t] = lo;
}

// Records in nnz order: [lead_0, trail_0, lead_1, trail_1, ...].  A row crossing tiles
// a..b has trail_a, lead_{a+1}, ..., lead_b with only empty trail slots between them; the
// first record of each run sums the run in order and writes the row.
template <class V>
__global__ void tile_carry_fixup_kernel(int64_t nrec, const int64_t *crow, const double *cval, V *x,
                                        int64_t ldx) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nrec) return;
    const int64_t r = crow[k];
    if (r < 0) return;
    if (k > 0 && (crow[k - 1] == r || (crow[k - 1] < 0 && k > 1 && crow[k - 2] == r))) return;
    double s = cval[k];
    for (int64_t u = k + 1; u < nrec; ++u) {
        if (crow[u] == r) s = addd(s, cval[u]);
        else if (crow[u] < 0 && (u & 1) && u + 1 < nrec && crow[u + 1] == r) continue;
        else break;
    }
    x[r * ldx] = (V)s;
}

// Deterministic carry fix-up: runs of equal carry rows are summed in tile order and
// added once to the row's value (written by the tile that finished the row).
template <class V>
__global__ void carry_fixup_kernel(int64_t num_tiles, const int64_t *carry_rows,
                                   const double *carry_vals, V *x, int64_t ldx) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= num_tiles) return;
    const int64_t r = carry_rows[t];
    if (r < 0 || (t > 0 && carry_rows[t - 1] == r)) return;
    double s = carry_vals[t];
    for (int64_t u = t + 1; u < num_tiles && carry_rows[u] == r; ++u) s = addd(s, carry_vals[u]);
    x[r * ldx] = (V)addd((double)x[r * ldx], s);
}

// ============================================================ COO: segmented reduction
// Tiles of NT*IPT consecutive (sorted) entries.  Each thread reduces IPT entries by
// row key; a block reduce-by-key scan joins runs crossing threads; runs finished in
// the tile are written; a run continuing into the next tile is carried to the
// fix-up kernel.  With accumulate == false the tile also zeroes the empty rows it
// owns (gaps between its keys, plus the leading / trailing gaps in the first / last
// tile), replacing the reference's separate zero pass (linop.py:155).  With
// accumulate == true results are added into x (the Hybrid format's COO tail).
template <class V, class I, int NT, int IPT>
__global__ void __launch_bounds__(NT) coo_kernel(int64_t rows, int64_t nnz, const I *__restrict__ ri,
                                                 const I *__restrict__ ci, const V *__restrict__ val,
                                                 const V *__restrict__ b, int64_t ldb, V *x,
                                                 int64_t ldx, int64_t num_tiles, int64_t *carry_rows,
                                                 double *carry_vals, bool accumulate) {
    constexpr int TILE = NT * IPT;
    __shared__ double s_prod[TILE];
    __shared__ int64_t s_key[TILE + 1];
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int64_t e0 = tile * TILE;
        const int64_t e1 = e0 + TILE < nnz ? e0 + TILE : nnz;
        const int64_t ne = e1 - e0;
        for (int64_t j = threadIdx.x; j < ne; j += NT) s_key[j] = (int64_t)ld_stream(ri + e0 + j);
        stage_products<V, I, NT, IPT>(ci + e0, val + e0, ne, b, ldb, s_prod);
        if (threadIdx.x == 0) s_key[ne] = e1 < nnz ? (int64_t)ri[e1] : INT64_MAX;
        __syncthreads();
        if (!accumulate) {
            const int64_t prev = e0 == 0 ? -1 : (int64_t)ri[e0 - 1];
            for (int64_t j = threadIdx.x; j < ne; j += NT) {
                const int64_t lo = (j == 0 ? prev : s_key[j - 1]) + 1, hi = s_key[j];
                for (int64_t g = lo; g < hi; ++g) x[g * ldx] = (V)0;
            }
            if (tile == num_tiles - 1 && threadIdx.x == 0)
                for (int64_t g = s_key[ne - 1] + 1; g < rows; ++g) x[g * ldx] = (V)0;
        }
        // pass 1: this thread's trailing run (carry-out)
        const int64_t j0 = (int64_t)threadIdx.x * IPT;
        const int64_t j1 = j0 + IPT < ne ? j0 + IPT : ne;
        const bool active = j0 < ne;
        int64_t key = active ? s_key[j0] : INT64_MAX;
        double acc = 0.0;
        for (int64_t j = j0; j < j1; ++j) {
            if (s_key[j] != key) {
                key = s_key[j];
                acc = 0.0;
            }
            acc = addd(acc, s_prod[j]);
        }
        int64_t ex_key;
        double cv = acc, ex_val;
        scan_by_key<NT>(key, cv, ex_key, ex_val);
        // pass 2: emit runs that finish inside this thread's range
        if (active) {
            int64_t k2 = s_key[j0];
            double a2 = ex_key == k2 ? ex_val : 0.0;
            for (int64_t j = j0; j < j1; ++j) {
                if (s_key[j] != k2) {
                    x[k2 * ldx] = accumulate ? (V)addd((double)x[k2 * ldx], a2) : (V)a2;
                    k2 = s_key[j];
                    a2 = 0.0;
                }
                a2 = addd(a2, s_prod[j]);
            }
            if (s_key[j1] != k2) x[k2 * ldx] = accumulate ? (V)addd((double)x[k2 * ldx], a2) : (V)a2;
            if (j1 == ne) {
                // last active thread: its inclusive pair is the tile's trailing run
                const bool carry = s_key[ne] == k2;
                carry_rows[tile] = carry ? k2 : -1;
                carry_vals[tile] = carry ? cv : 0.0;
            }
        }
        __syncthreads();
    }
}

// ============================================================ COO: warp segmented reduction
// Every warp owns chunks of CHUNK consecutive (sorted) entries.  Per step each lane
// loads K entries (entry base + k*32 + lane: coalesced), issues the K gathers, then for
// each k the warp runs an inclusive shuffle scan by row key (5 steps, fixed order); a
// lane whose successor holds another key closes its run and writes it, the open run at
// lane 31 is carried in registers to the next group.  The run still open at the end of a
// chunk is written by the chunk that finishes the row, its partial goes to the carry
// fix-up (deterministic, no atomics).  Empty rows between keys are zeroed by the lane
// that sees the gap (accumulate == false).  No shared memory, no block barriers.
template <class V, class I, int K>
__global__ void __launch_bounds__(256) coo_warp_kernel(int64_t rows, int64_t nnz,
                                                       const I *__restrict__ ri,
                                                       const I *__restrict__ ci,
                                                       const V *__restrict__ val,
                                                       const V *__restrict__ b, int64_t ldb, V *x,
                                                       int64_t ldx, int64_t chunk, int64_t nchunks,
                                                       int64_t *carry_rows, double *carry_vals,
                                                       bool accumulate) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int64_t NONE = INT64_MAX;
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const int64_t e0 = c * chunk;
        const int64_t e1 = e0 + chunk < nnz ? e0 + chunk : nnz;
        int64_t ckey = e0 == 0 ? -1 : (int64_t)ri[e0 - 1];  // key before the first entry
        double cval = 0.0;
        bool open = false;  // (ckey, cval) is a run opened inside this chunk
        for (int64_t base = e0; base < e1; base += 32 * K) {
            int64_t key[K];
            V vv[K], gg[K];
            I cc[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int64_t e = base + k * 32 + lane;
                if (e < e1) {
                    key[k] = (int64_t)ld_stream(ri + e);
                    cc[k] = ld_stream(ci + e);
                    vv[k] = ld_stream(val + e);
                } else {
                    key[k] = NONE;
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (key[k] != NONE) gg[k] = __ldg(b + (int64_t)cc[k] * ldb);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int64_t kk = key[k];
                double v = kk != NONE ? mulp(vv[k], gg[k]) : 0.0;
                if (!accumulate) {  // zero the empty rows between the previous key and this one
                    int64_t prev = __shfl_up_sync(0xffffffffu, kk, 1);
                    if (lane == 0) prev = ckey;
                    if (kk != NONE)
                        for (int64_t g = prev + 1; g < kk; ++g) x[g * ldx] = (V)0;
                }
                // the run carried from the previous group ends where this group starts a new row
                const int64_t k0 = __shfl_sync(0xffffffffu, kk, 0);
                if (open && k0 != ckey) {
                    if (lane == 0) x[ckey * ldx] = accumulate ? (V)addd((double)x[ckey * ldx], cval) : (V)cval;
                    open = false;
                }
                if (lane == 0 && open && kk == ckey) v = addd(cval, v);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int64_t k2 = __shfl_up_sync(0xffffffffu, kk, o);
                    const double v2 = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o && k2 == kk) v = addd(v2, v);
                }
                const int64_t next = __shfl_down_sync(0xffffffffu, kk, 1);
                if (lane < 31 && kk != NONE && next != kk)
                    x[kk * ldx] = accumulate ? (V)addd((double)x[kk * ldx], v) : (V)v;
                const int64_t k31 = __shfl_sync(0xffffffffu, kk, 31);
                const double v31 = __shfl_sync(0xffffffffu, v, 31);
                if (k31 != NONE) {  // lane 31's run stays open into the next group
                    ckey = k31;
                    cval = v31;
                    open = true;
                } else {  // past the chunk end: every run closed at its last valid lane
                    open = false;
                }
            }
        }
        // the run open at the end of the chunk: finished here, or carried to the next chunk
        if (lane == 0) {
            const int64_t after = e1 < nnz ? (int64_t)ri[e1] : NONE;
            const bool carry = open && after == ckey;
            if (open && !carry) x[ckey * ldx] = accumulate ? (V)addd((double)x[ckey * ldx], cval) : (V)cval;
            carry_rows[c] = carry ? ckey : -1;
            carry_vals[c] = carry ? cval : 0.0;
            if (!accumulate && c == nchunks - 1 && e1 == nnz) {
                const int64_t last = (int64_t)ri[nnz - 1];
                for (int64_t g = last + 1; g < rows; ++g) x[g * ldx] = (V)0;
            }
        }
    }
}

// ============================================================ padded layouts (ELL / SELL-P)
// One column of RPT consecutive rows: 16-byte value vector and 8/16-byte index vector.
template <class V, class I, int RPT>
__device__ __forceinline__ void load_column(const V *__restrict__ val, const I *__restrict__ col,
                                            int64_t base, V (&vv)[RPT], I (&cc)[RPT]) {
    if constexpr (RPT * sizeof(V) == 16) {
        int4 raw = __ldcs(reinterpret_cast<const int4 *>(val + base));
        memcpy(vv, &raw, 16);
    } else if constexpr (RPT * sizeof(V) == 8) {
        int2 raw = __ldcs(reinterpret_cast<const int2 *>(val + base));
        memcpy(vv, &raw, 8);
    } else {
#pragma unroll
        for (int r = 0; r < RPT; ++r) vv[r] = __ldcs(val + base + r);
    }
    if constexpr (RPT * sizeof(I) == 16) {
        int4 raw = __ldcs(reinterpret_cast<const int4 *>(col + base));
        memcpy(cc, &raw, 16);
    } else if constexpr (RPT * sizeof(I) == 8) {
        int2 raw = __ldcs(reinterpret_cast<const int2 *>(col + base));
        memcpy(cc, &raw, 8);
    } else {
#pragma unroll
        for (int r = 0; r < RPT; ++r) cc[r] = __ldcs(col + base + r);
    }
}

// Accumulate `len` padded columns (column k at base0 + k*kstride) for RPT rows, four
// columns per step with all loads and gathers issued before the ordered adds (padding
// col = -1 is skipped, so each row's sum keeps the CSR order exactly).
template <class V, class I, int RPT, class Epi, bool U1>
__device__ __forceinline__ void padded_rows(const Epi &epi, const V *__restrict__ val, const I *__restrict__ col,
                                            const V *__restrict__ b, int64_t ldb, int64_t base0,
                                            int64_t kstride, int64_t len, double (&acc)[RPT]) {
    int64_t k = 0;
    for (; k + 4 <= len; k += 4) {
        V vv[4][RPT], gg[4][RPT];
        I cc[4][RPT];
#pragma unroll
        for (int u = 0; u < 4; ++u) load_column<V, I, RPT>(val, col, base0 + (k + u) * kstride, vv[u], cc[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                if constexpr (epi_has_gather<Epi>::value)  // branch-free: padding gathers col 0
                    gg[u][r] = gather_b(epi, b, bidx<U1>((int64_t)(cc[u][r] >= 0 ? cc[u][r] : 0), ldb));
                else  // predicated plain loads: heavily padded slices issue no pad gathers
                    gg[u][r] = cc[u][r] >= 0 ? __ldg(b + bidx<U1>((int64_t)cc[u][r], ldb)) : (V)0;
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                if (cc[u][r] >= 0) acc[r] = addd(acc[r], mulp(vv[u][r], gg[u][r]));
    }
    if (RPT * sizeof(V) == 16 && sizeof(V) == 4) {  // fp32, four rows per thread: the one-column loop measured faster
        for (; k < len; ++k) {
            V vv[RPT];
            I cc[RPT];
            load_column<V, I, RPT>(val, col, base0 + k * kstride, vv, cc);
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                if (cc[r] >= 0) acc[r] = addd(acc[r], mulp(vv[r], gather_b(epi, b, bidx<U1>((int64_t)cc[r], ldb))));
        }
    } else if (k < len) {
        // the last 1-3 columns as one more four-column step (columns past len skipped by a
        // uniform predicate, their indices set to padding): every load and gather of the
        // tail is in flight before the first add, instead of one dependent load -> gather
        // -> add round per column (128^3 has 7 columns = 4 + 3: fp64 ELL 37.8 -> 34.2 us,
        // Hybrid 37.9 -> 34.0; fp32 measured slower with it, 29.6 -> 30.1)
        V vv[4][RPT], gg[4][RPT];
        I cc[4][RPT];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (k + u < len) {
                load_column<V, I, RPT>(val, col, base0 + (k + u) * kstride, vv[u], cc[u]);
            } else {
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    vv[u][r] = V(0);
                    cc[u][r] = (I)-1;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                if constexpr (epi_has_gather<Epi>::value)
                    gg[u][r] = gather_b(epi, b, bidx<U1>((int64_t)(cc[u][r] >= 0 ? cc[u][r] : 0), ldb));
                else
                    gg[u][r] = cc[u][r] >= 0 ? __ldg(b + bidx<U1>((int64_t)cc[u][r], ldb)) : (V)0;
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                if (cc[u][r] >= 0) acc[r] = addd(acc[r], mulp(vv[u][r], gg[u][r]));
    }
}

// ============================================================ ELL (column-major)
// RPT consecutive rows per thread with 16-byte vector loads of values (and 8/16-byte
// loads of column indices); per-row order is the stored order -> bitwise = reference.
template <class V, class I, int RPT, class Epi, bool U1>
__global__ void __launch_bounds__(256) ell_kernel(int64_t rows, int64_t width, int64_t stride,
                                                  const I *__restrict__ col, const V *__restrict__ val,
                                                  const V *__restrict__ b, int64_t ldb, Epi epi) {
    if (epi.skip()) return;
    epi_prepare(epi);
    epi_part_t<Epi> part[Epi::N] = {};
    const int64_t groups = (rows + RPT - 1) / RPT;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = g * RPT;
        double acc[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r) acc[r] = 0.0;
        padded_rows<V, I, RPT, Epi, U1>(epi, val, col, b, ldb, i0, stride, width, acc);
#pragma unroll
        for (int r = 0; r < RPT; ++r)
            if (i0 + r < rows) epi.row(i0 + r, acc[r], part);
    }
    epi.finish(part);
}

// ============================================================ SELL-P
// Slices of S rows; entry k of row i (slice s) at (slice_sets[s] + k)*S + i%S.
// RPT consecutive rows of one slice per thread (S % RPT == 0), vector loads.
template <class V, class I, int RPT, class Epi, bool U1>
__global__ void __launch_bounds__(256) sellp_kernel(int64_t rows, int64_t S,
                                                    const I *__restrict__ slice_lengths,
                                                    const I *__restrict__ slice_sets,
                                                    const I *__restrict__ col,
                                                    const V *__restrict__ val,
                                                    const V *__restrict__ b, int64_t ldb, Epi epi,
                                                    const I *__restrict__ perm) {
    if (epi.skip()) return;
    epi_prepare(epi);
    epi_part_t<Epi> part[Epi::N] = {};
    const int64_t nslices = (rows + S - 1) / S;
    const int64_t groups = nslices * (S / RPT);
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = g * RPT;
        const int64_t s = i0 / S, l0 = i0 % S;
        const int64_t len = slice_lengths[s];
        const int64_t off = (int64_t)slice_sets[s] * S + l0;
        double acc[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r) acc[r] = 0.0;
        padded_rows<V, I, RPT, Epi, U1>(epi, val, col, b, ldb, off, S, len, acc);
#pragma unroll
        for (int r = 0; r < RPT; ++r)
            if (i0 + r < rows) epi.row(perm ? (int64_t)perm[i0 + r] : i0 + r, acc[r], part);
    }
    epi.finish(part);
}

// ============================================================ SELL-P: TMA-staged slice blocks
// A block of SPB = 128 / S consecutive slices is one contiguous range of the value and
// column arrays ((slice_sets[s0] .. slice_sets[s0 + SPB]) * S entries), so it is staged
// exactly like a CSR stream block: one elected thread issues cp.async.bulk copies into a
// two-stage shared-memory ring (mbarrier completion), the next block is prefetched
// while this one is reduced, and thread t reduces row t of the block sequentially
// (column-major within the slice) -> bit-exact with the reference's row order.
struct SellpBlockMeta {
    int64_t s0;              // first slice of the block
    int64_t dv, dc;          // stage slot of the block's first entry (values / columns)
    int32_t len[4], off[4];  // per slice: length, first entry relative to the block start
};

// fp64: min-blocks hint 1 lets the compiler take 56 registers instead of 40 (fewer CTAs
// per SM, more of each thread's loads in flight): 128^3 SELL-P(64) 34.5 -> 32.7 us (0.96);
// fp32 measured slower with it (25.8 -> 26.3) and with a 32-register cap (27.5)
template <class V, class I, int S, class Epi, bool U1>
__global__ void __launch_bounds__(128, sizeof(V) == 8 ? 1 : 0) sellp_block_kernel(int64_t rows, int64_t nslices,
                                                           const I *__restrict__ sl,
                                                           const I *__restrict__ ss,
                                                           const I *__restrict__ col,
                                                           const V *__restrict__ val,
                                                           const V *__restrict__ b, int64_t ldb,
                                                           int cap_entries, Epi epi,
                                                           const I *__restrict__ perm) {
    constexpr int SPB = 128 / S;
    static_assert(SPB >= 1 && SPB <= 4, "slice size 32, 64 or 128");
    if (epi.skip()) return;
    epi_prepare(epi);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ SellpBlockMeta meta[2];
    constexpr int VV = 16 / sizeof(V), VI = 16 / sizeof(I);
    const size_t cap_v = (size_t)cap_entries + 2 * VV, cap_c = (size_t)cap_entries + 2 * VI;
    const size_t off_c = (cap_v * sizeof(V) + 15) & ~size_t(15);
    const size_t stage_bytes = (off_c + cap_c * sizeof(I) + 15) & ~size_t(15);
    const int tid = threadIdx.x;
    const int64_t nblk = (nslices + SPB - 1) / SPB;
    const int64_t total = (int64_t)ss[nslices] * S;
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int64_t blk, int st) {  // thread 0 only
        unsigned char *p = smem + st * stage_bytes;
        V *sv = reinterpret_cast<V *>(p);
        I *sc = reinterpret_cast<I *>(p + off_c);
        const int64_t s0 = blk * SPB, s1 = s0 + SPB < nslices ? s0 + SPB : nslices;
        const int64_t lo = (int64_t)ss[s0] * S, hi = (int64_t)ss[s1] * S;
        SellpBlockMeta m;
        m.s0 = s0;
        int64_t bv_base = 0, bc_base = 0;
        const uint32_t bv = stage_range(val, lo, hi, total, sv, bv_base);
        const uint32_t bc = stage_range(col, lo, hi, total, sc, bc_base);
        m.dv = lo - bv_base;
        m.dc = lo - bc_base;
        for (int j = 0; j < SPB; ++j) {
            const int64_t s = s0 + j;
            m.len[j] = s < s1 ? (int32_t)sl[s] : 0;
            m.off[j] = s < s1 ? (int32_t)((int64_t)ss[s] * S - lo) : 0;
        }
        meta[st] = m;
        mbar_arrive_expect_tx(&bar[st], bv + bc);
        if (bv) bulk_g2s(sv, val + bv_base, bv, &bar[st], pol);
        if (bc) bulk_g2s(sc, col + bc_base, bc, &bar[st], pol);
    };
    epi_part_t<Epi> part[Epi::N] = {};
    int64_t blk = blockIdx.x;
    if (tid == 0 && blk < nblk) issue(blk, 0);
    for (int it = 0; blk < nblk; blk += gridDim.x, ++it) {
        const int st = it & 1;
        const uint32_t parity = (it >> 1) & 1;
        if (tid == 0 && blk + gridDim.x < nblk) issue(blk + gridDim.x, st ^ 1);
        mbar_wait(&bar[st], parity);
        const unsigned char *p = smem + st * stage_bytes;
        const V *sv = reinterpret_cast<const V *>(p);
        const I *sc = reinterpret_cast<const I *>(p + off_c);
        const SellpBlockMeta m = meta[st];
        const int j = tid / S, l = tid % S;
        const int64_t i = (m.s0 + j) * S + l;
        if (j < SPB && i < rows) {
            // 32-bit stage offsets (a stage holds < 2^31 entries)
            const int len = m.len[j];
            const int ov = (int)(m.dv + m.off[j] + l), oc = (int)(m.dc + m.off[j] + l);
            double acc = 0.0;
            int k = 0;
            for (; k + 8 <= len; k += 8) {
                V vv[8], bb[8];
                I cc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    vv[u] = sv[ov + (k + u) * S];
                    cc[u] = sc[oc + (k + u) * S];
                    if constexpr (epi_has_gather<Epi>::value)  // padding: col 0, masked below
                        bb[u] = gather_b(epi, b, bidx<U1>((int64_t)(cc[u] >= 0 ? cc[u] : 0), ldb));
                    else
                        bb[u] = cc[u] >= 0 ? __ldg(b + bidx<U1>((int64_t)cc[u], ldb)) : (V)0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (cc[u] >= 0) acc = addd(acc, mulp(vv[u], bb[u]));
            }
            if (k < len) {
                V vv[8], bb[8];
                I cc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {  // branch-free tail (see csr_stream_kernel)
                    const bool on = k + u < len;
                    if constexpr (sizeof(V) == 4) {
                        // fp32: predicated stage reads at fixed offsets from one base (no
                        // clamped index; 128^3 SELL-P(64) 29.5 -> 26.4 us; fp64 measured
                        // slower with it, 34.7 -> 35.5, and keeps the clamped index)
                        vv[u] = on ? sv[ov + (k + u) * S] : V(0);
                        cc[u] = on ? sc[oc + (k + u) * S] : (I)-1;
                    } else {
                        const int e = (on ? k + u : len - 1) * S;
                        vv[u] = sv[ov + e];
                        cc[u] = on ? sc[oc + e] : (I)-1;
                    }
                    bb[u] = gather_b(epi, b, bidx<U1>((int64_t)(cc[u] >= 0 ? cc[u] : 0), ldb));
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (cc[u] >= 0) acc = addd(acc, mulp(vv[u], bb[u]));
            }
            epi.row(perm ? (int64_t)perm[i] : i, acc, part);
        }
        __syncthreads();
    }
    epi.finish(part);
}

// ============================================================ SELL-P: TMA-staged chunks
// Blocks whose stored entries exceed the stage (long slices) use this variant.  A block
// of SPB = 128 / S consecutive slices is one contiguous range of the value and column
// arrays ((slice_sets[s0] .. slice_sets[s0 + SPB]) * S entries).  It is streamed
// through a two-stage shared-memory ring in chunks of at most cap_entries entries (a
// multiple of S, i.e. whole columns): one elected thread issues the cp.async.bulk copies
// of the next chunk (mbarrier completion) while the current one is reduced.  Thread t
// owns row t of the block and accumulates its columns chunk by chunk in stored
// (column-major) order -> bit-exact with the reference's row sum.  Chunking keeps long
// slices (power-law rows: a 64-row slice of 11,668 columns) streaming instead of
// falling back to the direct kernel.
struct SellpMeta {
    int64_t s0;              // first slice of the block
    int64_t lo;              // block's first entry (global)
    int64_t clo, chi;        // this chunk's entries [clo, chi) (global)
    int64_t bv, bc;          // global entry index held by stage slot 0 (values / columns)
    int32_t len[4], off[4];  // per slice: length, first entry relative to lo
    int32_t last;            // last chunk of the block: emit the rows
};

template <class V, class I, int S, class Epi, bool U1>
__global__ void __launch_bounds__(128) sellp_chunk_kernel(int64_t rows, int64_t nslices,
                                                           const I *__restrict__ sl,
                                                           const I *__restrict__ ss,
                                                           const I *__restrict__ col,
                                                           const V *__restrict__ val,
                                                           const V *__restrict__ b, int64_t ldb,
                                                           int cap_entries, Epi epi,
                                                           const I *__restrict__ perm) {
    constexpr int SPB = 128 / S;
    static_assert(SPB >= 1 && SPB <= 4, "slice size 32, 64 or 128");
    if (epi.skip()) return;
    epi_prepare(epi);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ SellpMeta meta[2];
    constexpr int VV = 16 / sizeof(V), VI = 16 / sizeof(I);
    const size_t cap_v = (size_t)cap_entries + 2 * VV, cap_c = (size_t)cap_entries + 2 * VI;
    const size_t off_c = (cap_v * sizeof(V) + 15) & ~size_t(15);
    const size_t stage_bytes = (off_c + cap_c * sizeof(I) + 15) & ~size_t(15);
    const int64_t chunk = (int64_t)(cap_entries / S) * S;  // whole columns per chunk
    const int tid = threadIdx.x;
    const int64_t nblk = (nslices + SPB - 1) / SPB;
    const int64_t total = (int64_t)ss[nslices] * S;
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // thread 0: stage chunk [clo, min(clo + chunk, hi)) of block blk; returns true if it
    // was the block's last chunk, else sets clo to the next chunk's start
    auto issue = [&](int64_t blk, int64_t &clo, int st) -> bool {
        unsigned char *p = smem + st * stage_bytes;
        V *sv = reinterpret_cast<V *>(p);
        I *sc = reinterpret_cast<I *>(p + off_c);
        const int64_t s0 = blk * SPB, s1 = s0 + SPB < nslices ? s0 + SPB : nslices;
        const int64_t lo = (int64_t)ss[s0] * S, hi = (int64_t)ss[s1] * S;
        if (clo < lo) clo = lo;
        const int64_t chi = clo + chunk < hi ? clo + chunk : hi;
        SellpMeta m;
        m.s0 = s0;
        m.lo = lo;
        m.clo = clo;
        m.chi = chi;
        m.last = chi == hi;
        const uint32_t bv = stage_range(val, clo, chi, total, sv, m.bv);
        const uint32_t bc = stage_range(col, clo, chi, total, sc, m.bc);
        for (int j = 0; j < SPB; ++j) {
            const int64_t s = s0 + j;
            m.len[j] = s < s1 ? (int32_t)sl[s] : 0;
            m.off[j] = s < s1 ? (int32_t)((int64_t)ss[s] * S - lo) : 0;
        }
        meta[st] = m;
        mbar_arrive_expect_tx(&bar[st], bv + bc);
        if (bv) bulk_g2s(sv, val + m.bv, bv, &bar[st], pol);
        if (bc) bulk_g2s(sc, col + m.bc, bc, &bar[st], pol);
        clo = chi;
        return chi == hi;
    };
    epi_part_t<Epi> part[Epi::N] = {};
    int64_t blk = blockIdx.x;
    // the next work item to issue: (nblk_i, nclo); chunks of a block in order, then the
    // CTA's next block
    int64_t nb = blk, nclo = -1;
    if (tid == 0 && blk < nblk && issue(blk, nclo, 0)) {
        nb = blk + gridDim.x;
        nclo = -1;
    }
    double acc = 0.0;
    for (int it = 0; blk < nblk; ++it) {
        const int st = it & 1;
        const uint32_t parity = (it >> 1) & 1;
        if (tid == 0 && nb < nblk && issue(nb, nclo, st ^ 1)) {  // prefetch the next chunk
            nb += gridDim.x;
            nclo = -1;
        }
        mbar_wait(&bar[st], parity);
        const unsigned char *p = smem + st * stage_bytes;
        const V *sv = reinterpret_cast<const V *>(p);
        const I *sc = reinterpret_cast<const I *>(p + off_c);
        const SellpMeta &m = meta[st];  // read in place (no local copy of the arrays)
        const int j = tid / S, l = tid % S;
        const int64_t i = (m.s0 + j) * S + l;
        const bool last = m.last;
        if (j < SPB && i < rows) {
            const int len = m.len[j];
            const int64_t lo = m.lo, off = m.off[j];
            // columns of slice j inside this chunk (chunk bounds are whole columns)
            const int64_t rel0 = m.clo - lo - off, rel1 = m.chi - lo - off;
            int k = rel0 > 0 ? (int)(rel0 / S) : 0;
            const int kend = rel1 <= 0 ? 0 : (int)(rel1 / S < len ? rel1 / S : len);
            const int64_t ov = lo + off + l - m.bv, oc = lo + off + l - m.bc;  // stage slots of k = 0
            for (; k < kend; k += 8) {
                V vv[8], bb[8];
                I cc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {  // branch-free tail (see csr_stream_kernel)
                    const bool on = k + u < kend;
                    if constexpr (sizeof(V) == 4) {  // fp32: predicated reads at fixed offsets
                        vv[u] = on ? sv[ov + (int64_t)(k + u) * S] : V(0);
                        cc[u] = on ? sc[oc + (int64_t)(k + u) * S] : (I)-1;
                    } else {
                        const int kk = on ? k + u : kend - 1;
                        vv[u] = sv[ov + (int64_t)kk * S];
                        cc[u] = on ? sc[oc + (int64_t)kk * S] : (I)-1;
                    }
                    if constexpr (epi_has_gather<Epi>::value)  // padding: col 0, masked below
                        bb[u] = gather_b(epi, b, bidx<U1>((int64_t)(cc[u] >= 0 ? cc[u] : 0), ldb));
                    else
                        bb[u] = cc[u] >= 0 ? __ldg(b + bidx<U1>((int64_t)cc[u], ldb)) : (V)0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (cc[u] >= 0) acc = addd(acc, mulp(vv[u], bb[u]));
            }
            if (last) {
                epi.row(perm ? (int64_t)perm[i] : i, acc, part);
                acc = 0.0;
            }
        }
        if (last) blk += gridDim.x;
        __syncthreads();  // stage st consumed before it is re-issued
    }
    epi.finish(part);
}

// ------------------------------------------------------------ SELL-P: split pieces
// Load balance for blocks far larger than the average (power-law rows, SELL-C-sigma
// windows that gather the longest rows): every block's entry range [lo, hi) is cut into
// pieces of at most `pe` entries (whole chunks), a piece is one work item of a grid-stride
// loop, and the chunks of a piece stream through the same TMA ring as sellp_chunk_kernel.
// A block of one piece stores its rows directly (bit-exact, the stored order); a split
// block's pieces leave one partial sum per row in `carry` (slot = piece index), and
// sellp_piece_fixup_kernel adds them in piece order.  Plan (int64, built by the
// frontend): pstart[nblk + 1] (first piece of each block), pblock[npieces] (block of each
// piece), split[nsplit] (blocks of more than one piece).
template <class V, class I, int S, bool U1>
__global__ void __launch_bounds__(128) sellp_piece_kernel(int64_t rows, int64_t nslices,
                                                           const I *__restrict__ sl,
                                                           const I *__restrict__ ss,
                                                           const I *__restrict__ col,
                                                           const V *__restrict__ val,
                                                           const V *__restrict__ b, int64_t ldb,
                                                           int cap_entries, const int64_t *__restrict__ plan,
                                                           int64_t npieces, int64_t pe, double *carry,
                                                           V *x, int64_t ldx, const I *__restrict__ perm) {
    constexpr int SPB = 128 / S;
    static_assert(SPB >= 1 && SPB <= 4, "slice size 32, 64 or 128");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ SellpMeta meta[2];
    __shared__ int32_t split_of[2];  // the staged chunk's piece belongs to a split block
    constexpr int VV = 16 / sizeof(V), VI = 16 / sizeof(I);
    const size_t cap_v = (size_t)cap_entries + 2 * VV, cap_c = (size_t)cap_entries + 2 * VI;
    const size_t off_c = (cap_v * sizeof(V) + 15) & ~size_t(15);
    const size_t stage_bytes = (off_c + cap_c * sizeof(I) + 15) & ~size_t(15);
    const int64_t chunk = (int64_t)(cap_entries / S) * S;
    const int tid = threadIdx.x;
    const int64_t nblk = (nslices + SPB - 1) / SPB;
    const int64_t total = (int64_t)ss[nslices] * S;
    const int64_t *pstart = plan, *pblock = plan + nblk + 1;
    const uint64_t pol = policy_evict_first();
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // thread 0: stage chunk [clo, min(clo + chunk, piece end)) of piece pc; true if it
    // was the piece's last chunk, else clo advances to the next chunk
    auto issue = [&](int64_t pc, int64_t &clo, int st) -> bool {
        unsigned char *p = smem + st * stage_bytes;
        V *sv = reinterpret_cast<V *>(p);
        I *sc = reinterpret_cast<I *>(p + off_c);
        const int64_t blk = pblock[pc], q = pc - pstart[blk];
        const int64_t s0 = blk * SPB, s1 = s0 + SPB < nslices ? s0 + SPB : nslices;
        const int64_t lo = (int64_t)ss[s0] * S, hi = (int64_t)ss[s1] * S;
        const int64_t plo = lo + q * pe, phi = plo + pe < hi ? plo + pe : hi;
        if (clo < plo) clo = plo;
        const int64_t chi = clo + chunk < phi ? clo + chunk : phi;
        SellpMeta m;
        m.s0 = s0;
        m.lo = lo;
        m.clo = clo;
        m.chi = chi;
        m.last = chi == phi;
        const uint32_t bv = stage_range(val, clo, chi, total, sv, m.bv);
        const uint32_t bc = stage_range(col, clo, chi, total, sc, m.bc);
        for (int j = 0; j < SPB; ++j) {
            const int64_t s = s0 + j;
            m.len[j] = s < s1 ? (int32_t)sl[s] : 0;
            m.off[j] = s < s1 ? (int32_t)((int64_t)ss[s] * S - lo) : 0;
        }
        meta[st] = m;
        split_of[st] = pstart[blk + 1] - pstart[blk] > 1;
        mbar_arrive_expect_tx(&bar[st], bv + bc);
        if (bv) bulk_g2s(sv, val + m.bv, bv, &bar[st], pol);
        if (bc) bulk_g2s(sc, col + m.bc, bc, &bar[st], pol);
        clo = chi;
        return chi == phi;
    };
    int64_t pc = blockIdx.x;
    int64_t npc = pc, nclo = -1;
    if (tid == 0 && pc < npieces && issue(pc, nclo, 0)) {
        npc = pc + gridDim.x;
        nclo = -1;
    }
    double acc = 0.0;
    for (int it = 0; pc < npieces; ++it) {
        const int st = it & 1;
        const uint32_t parity = (it >> 1) & 1;
        if (tid == 0 && npc < npieces && issue(npc, nclo, st ^ 1)) {
            npc += gridDim.x;
            nclo = -1;
        }
        mbar_wait(&bar[st], parity);
        const unsigned char *p = smem + st * stage_bytes;
        const V *sv = reinterpret_cast<const V *>(p);
        const I *sc = reinterpret_cast<const I *>(p + off_c);
        const SellpMeta &m = meta[st];
        const int j = tid / S, l = tid % S;
        const int64_t i = (m.s0 + j) * S + l;
        const bool last = m.last;
        if (j < SPB && i < rows) {
            const int len = m.len[j];
            const int64_t lo = m.lo, off = m.off[j];
            const int64_t rel0 = m.clo - lo - off, rel1 = m.chi - lo - off;
            int k = rel0 > 0 ? (int)(rel0 / S) : 0;
            const int kend = rel1 <= 0 ? 0 : (int)(rel1 / S < len ? rel1 / S : len);
            const int64_t ov = lo + off + l - m.bv, oc = lo + off + l - m.bc;
            for (; k < kend; k += 8) {
                V vv[8], bb[8];
                I cc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int kk = k + u < kend ? k + u : kend - 1;
                    vv[u] = sv[ov + (int64_t)kk * S];
                    cc[u] = k + u < kend ? sc[oc + (int64_t)kk * S] : (I)-1;
                    bb[u] = cc[u] >= 0 ? __ldg(b + bidx<U1>((int64_t)cc[u], ldb)) : (V)0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (cc[u] >= 0) acc = addd(acc, mulp(vv[u], bb[u]));
            }
        }
        if (last) {
            if (split_of[st])
                carry[pc * 128 + tid] = acc;  // every thread: rows past the end stay unread
            else if (j < SPB && i < rows)
                x[(perm ? (int64_t)perm[i] : i) * ldx] = (V)acc;
            acc = 0.0;
            pc += gridDim.x;
        }
        __syncthreads();  // stage st consumed before it is re-issued
    }
}

// rows of split blocks: the pieces' partial sums in piece order
template <class V, class I, int S>
__global__ void __launch_bounds__(128) sellp_piece_fixup_kernel(int64_t rows, int64_t nslices, const int64_t *__restrict__ plan,
                                                                 int64_t npieces, int64_t nsplit, const double *__restrict__ carry,
                                                                 V *x, int64_t ldx, const I *__restrict__ perm) {
    constexpr int SPB = 128 / S;
    const int64_t nblk = (nslices + SPB - 1) / SPB;
    const int64_t *pstart = plan, *split = plan + nblk + 1 + npieces;
    for (int64_t q = blockIdx.x; q < nsplit; q += gridDim.x) {
        const int64_t blk = split[q];
        const int64_t i = blk * 128 + threadIdx.x;  // = (blk SPB + j) S + l
        if (i >= rows) continue;
        double acc = 0.0;
        for (int64_t pc = pstart[blk]; pc < pstart[blk + 1]; ++pc) acc = addd(acc, carry[pc * 128 + threadIdx.x]);
        x[(perm ? (int64_t)perm[i] : i) * ldx] = (V)acc;
    }
}

// Row-owned epilogue applied after a row-splitting SpMV (merge / COO / Hybrid):
// re-reads x and feeds it to the epilogue (so fused dots work for every format).
template <class V, class Epi>
__global__ void __launch_bounds__(256) epilogue_pass_kernel(int64_t rows, const V *x, int64_t ldx,
                                                            Epi epi) {
    if (epi.skip()) return;
    epi_prepare(epi);
    epi_part_t<Epi> part[Epi::N] = {};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x)
        epi.row(i, (double)x[i * ldx], part);
    epi.finish(part);
}

}  // namespace sb
