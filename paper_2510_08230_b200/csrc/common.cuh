// common.cuh -- shared device helpers for the sm_100a SpMV / Krylov library.
//
// Numerics contract (mirrors the reference):
//   * every accumulation is fp64; for fp32 buffers each product is rounded to
//     fp32 first (numba float32*float32 -> float32, _kernels.py:62-68);
//   * no FMA contraction anywhere (explicit __dmul_rn/__dadd_rn, and the whole
//     library is compiled with --fmad=false);
//   * every reduction is deterministic: fixed per-thread order, fixed tree, and
//     a last-block-done finalisation that sums per-block partials in index
//     order (no floating-point atomics).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <utility>

namespace sb {

constexpr int kWarp = 32;

// ------------------------------------------------------------------ element ops
__device__ __forceinline__ double mulp(float a, float b) { return (double)__fmul_rn(a, b); }
__device__ __forceinline__ double mulp(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double addd(double a, double b) { return __dadd_rn(a, b); }

// _kernels.axpy_rows: y = alpha*x + y, alpha fp64, computed in fp64, rounded once on store.
template <class V>
__device__ __forceinline__ V axpy_e(double alpha, V x, V y) {
    return (V)__dadd_rn(__dmul_rn(alpha, (double)x), (double)y);
}
// _kernels.scal_rows: x = alpha*x
template <class V>
__device__ __forceinline__ V scal_e(double alpha, V x) {
    return (V)__dmul_rn(alpha, (double)x);
}
// Jacobi apply (np.multiply in the value dtype, precond.py:62)
__device__ __forceinline__ float vmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double vmul(double a, double b) { return __dmul_rn(a, b); }
// value-dtype scalar ops of the factorizations (NumPy scalar semantics, precond.py:155-187)
__device__ __forceinline__ float vdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double vdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float vsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double vsub(double a, double b) { return __dsub_rn(a, b); }

// first position in [lo, hi) (sorted) whose value is >= key
template <class T>
__host__ __device__ __forceinline__ const T *lbound(const T *lo, const T *hi, T key) {
    while (lo < hi) {
        const T *mid = lo + (hi - lo) / 2;
        if (*mid < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ------------------------------------------------------------------ cache-policy loads
// Matrix streams are read exactly once per SpMV: evict-first in L2, no L1 allocation,
// so the Krylov vectors (a few x 16.8 MB at 128^3) stay L2-resident across kernels.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int4 ld_stream16(const void *ptr, uint64_t pol) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr), "l"(pol));
    return r;
}
// plain (L1-cached) loads / stores carrying an L2 eviction-priority policy
__device__ __forceinline__ double ld_hint(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ float ld_hint(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ void st_hint(double *p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float *p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_unchanged() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <class T>
__device__ __forceinline__ T ld_stream(const T *ptr) {
    return __ldcs(ptr);  // streaming (evict-first) scalar load
}
__device__ __forceinline__ int ld_stream(const int *ptr) { return __ldcs(ptr); }

// ------------------------------------------------------------------ TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}
// 1-D TMA bulk copy global -> shared; completion is signalled on `bar` as tx bytes.
// L2 prefetch hint of the 16-byte aligned part of [lo, hi) (cp.async.bulk.prefetch)
__device__ __forceinline__ void l2_prefetch_range(const void *lo, const void *hi) {
    const uintptr_t a = ((uintptr_t)lo + 15) & ~(uintptr_t)15, e = (uintptr_t)hi & ~(uintptr_t)15;
    if (e > a) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

// the same without an L2 eviction hint (vectors that are re-read soon)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels launched with launch_pdl() may start while their predecessor on the stream is
// still draining: everything before pdl_wait() must touch only data no predecessor
// writes (matrix streams, shared-memory setup); pdl_wait() returns once the predecessor
// grid has completed and its writes are visible.  pdl_trigger() lets the successor's
// CTAs be scheduled as SM resources free up.  Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ deterministic reductions
template <int N>
struct Vec {
    double v[N];
};

// Warp tree (fixed order) then one value per warp through shared memory.
template <int N>
__device__ __forceinline__ void block_reduce(double (&v)[N], double (*scratch)[N]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] = addd(v[k], __shfl_down_sync(0xffffffffu, v[k], o));
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < N; ++k) scratch[warp][k] = v[k];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = lane < nw ? scratch[lane][k] : 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[k] = addd(v[k], __shfl_down_sync(0xffffffffu, v[k], o));
    }
}

// Grid-wide deterministic sum: every block publishes its partials; the last block to
// arrive sums them in block-index order and returns true (in all its threads) with the
// totals in `tot`.  `ticket` is self-resetting.  partials layout: [N][gridDim.x].
template <int N>
__device__ __forceinline__ bool grid_reduce(double (&v)[N], double *partials, unsigned *ticket,
                                            double (&tot)[N]) {
    __shared__ double scratch[32][N];
    __shared__ bool s_last;
    __shared__ double s_tot[N];
    block_reduce<N>(v, scratch);
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) partials[k * G + blockIdx.x] = v[k];
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == (unsigned)G - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    double a[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        a[k] = 0.0;
        for (int i = threadIdx.x; i < G; i += blockDim.x) a[k] = addd(a[k], __ldcg(partials + k * G + i));
    }
    block_reduce<N>(a, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) s_tot[k] = a[k];
        *ticket = 0u;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) tot[k] = s_tot[k];
    return true;
}

// ------------------------------------------------------------------ compensated sums
// Neumaier-compensated partial (s + c): used where a recurrence is sensitive enough to
// the summation order of its dots that only near-exact dots follow the exact-arithmetic
// trajectory (BiCGSTAB on config #4).  Deterministic like the plain path.
struct CAcc {
    double s, c;
};
__device__ __forceinline__ void cadd(CAcc &a, double v) {
    const double t = __dadd_rn(a.s, v);
    const double e = fabs(a.s) >= fabs(v) ? __dadd_rn(__dsub_rn(a.s, t), v) : __dadd_rn(__dsub_rn(v, t), a.s);
    a.c = __dadd_rn(a.c, e);
    a.s = t;
}
__device__ __forceinline__ void cmerge(CAcc &a, const CAcc &b) {
    cadd(a, b.s);
    a.c = __dadd_rn(a.c, b.c);
}
__device__ __forceinline__ double cvalue(const CAcc &a) { return __dadd_rn(a.s, a.c); }

template <int N>
__device__ __forceinline__ void block_reduce_c(CAcc (&v)[N], CAcc (*scratch)[N]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            CAcc b;
            b.s = __shfl_down_sync(0xffffffffu, v[k].s, o);
            b.c = __shfl_down_sync(0xffffffffu, v[k].c, o);
            cmerge(v[k], b);
        }
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < N; ++k) scratch[warp][k] = v[k];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = lane < nw ? scratch[lane][k] : CAcc{0.0, 0.0};
#pragma unroll
        for (int k = 0; k < N; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                CAcc b;
                b.s = __shfl_down_sync(0xffffffffu, v[k].s, o);
                b.c = __shfl_down_sync(0xffffffffu, v[k].c, o);
                cmerge(v[k], b);
            }
    }
}

// grid_reduce with compensated partials: partials layout [2N][gridDim.x] (s then c)
template <int N>
__device__ __forceinline__ bool grid_reduce(CAcc (&v)[N], double *partials, unsigned *ticket, double (&tot)[N]) {
    __shared__ CAcc scratch[32][N];
    __shared__ bool s_last;
    __shared__ double s_tot[N];
    block_reduce_c<N>(v, scratch);
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            partials[(2 * k) * G + blockIdx.x] = v[k].s;
            partials[(2 * k + 1) * G + blockIdx.x] = v[k].c;
        }
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == (unsigned)G - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    CAcc a[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        a[k] = CAcc{0.0, 0.0};
        for (int i = threadIdx.x; i < G; i += blockDim.x)
            cmerge(a[k], CAcc{__ldcg(partials + (2 * k) * G + i), __ldcg(partials + (2 * k + 1) * G + i)});
    }
    block_reduce_c<N>(a, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) s_tot[k] = cvalue(a[k]);
        *ticket = 0u;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) tot[k] = s_tot[k];
    return true;
}

// ------------------------------------------------------------------ launch geometry
struct DeviceInfo {
    int sms = 148;
    int max_smem_optin = 227 * 1024;
};
DeviceInfo &device_info();

// Opt a kernel into 200 KB of dynamic shared memory on the CURRENT device.  The
// attribute is per (function, device), so the memo is keyed on both (a process that
// drives a second GPU configures it there too); thread-safe, cheap after the first call.
void ensure_max_smem(const void *fn);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace sb
