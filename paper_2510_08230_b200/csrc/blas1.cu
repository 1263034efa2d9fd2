#include <set>
// blas1.cu -- BLAS-1 on dense device vectors/matrices and the library-level entry points.
//
// Reference: core.dot / norm2 / axpy / scal / copy_into (core.py:358-401) over
// _kernels.dot_range / axpy_rows / scal_rows / copy_rows (_kernels.py:23-49), and
// JacobiPreconditioner.apply (precond.py:57-63).
#include <mutex>
#include <vector>

#include "capi_util.cuh"
#include "spmv_launch.cuh"

namespace sb {

void ensure_max_smem(const void *fn) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert({fn, dev}).second) {
        int optin = 0;  // B200: 227 KB per block
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
            optin < 200 * 1024)
            optin = 200 * 1024;
        cudaFuncAttributes fa{};  // the opt-in limit covers static + dynamic shared memory
        const size_t stat = cudaFuncGetAttributes(&fa, fn) == cudaSuccess ? fa.sharedSizeBytes : 4096;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)stat);
        cudaGetLastError();
    }
}

DeviceInfo &device_info() {
    static DeviceInfo infos[64];
    static bool init[64] = {};
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (!init[dev]) {
        cudaDeviceGetAttribute(&infos[dev].sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&infos[dev].max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (infos[dev].sms <= 0) infos[dev].sms = 148;
        init[dev] = true;
    }
    return infos[dev];
}

// ---------------------------------------------------------------- kernels
// element (t) of a rows x cols dense matrix with row stride ld
__device__ __forceinline__ int64_t didx(int64_t t, int64_t cols, int64_t ld) {
    return cols == 1 ? t * ld : (t / cols) * ld + t % cols;
}

template <class V>
__global__ void __launch_bounds__(256) dot_kernel(int64_t n, const V *x, int64_t ldx, const V *y,
                                                  int64_t ldy, double *partials, unsigned *ticket,
                                                  double *out) {
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[0] = addd(v[0], mulp(x[i * ldx], y[i * ldy]));
    double tot[1];
    if (grid_reduce<1>(v, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
}

template <class V>
__global__ void __launch_bounds__(256) axpy_kernel(int64_t rows, int64_t cols, double alpha,
                                                   const V *x, int64_t ldx, V *y, int64_t ldy) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t iy = didx(t, cols, ldy);
        y[iy] = axpy_e(alpha, x[didx(t, cols, ldx)], y[iy]);
    }
}

template <class V>
__global__ void __launch_bounds__(256) scal_kernel(int64_t rows, int64_t cols, double alpha, V *x,
                                                   int64_t ldx) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = didx(t, cols, ldx);
        x[i] = scal_e(alpha, x[i]);
    }
}

template <class V>
__global__ void __launch_bounds__(256) copy_kernel(int64_t rows, int64_t cols, const V *x,
                                                   int64_t ldx, V *y, int64_t ldy) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
         t += (int64_t)gridDim.x * blockDim.x)
        y[didx(t, cols, ldy)] = x[didx(t, cols, ldx)];
}

template <class V>
__global__ void __launch_bounds__(256) jacobi_apply_kernel(int64_t rows, int64_t cols,
                                                           const V *inv, const V *b, int64_t ldb,
                                                           V *x, int64_t ldx) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
         t += (int64_t)gridDim.x * blockDim.x)
        x[didx(t, cols, ldx)] = vmul(b[didx(t, cols, ldb)], inv[t / cols]);
}

// ---------------------------------------------------------------- host helpers
template <class V>
sb_status do_dot(const sb_dense *x, const sb_dense *y, double *out, void *ws, cudaStream_t st,
                 sb_error *err) {
    if (!x || !y || !out || !ws) return fail(err, SB_ERR_INVALID_ARGUMENT, "dot: null argument");
    if (x->cols != 1 || y->cols != 1)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "expected a column vector, got (%lld, %lld)",
                    (long long)x->rows, (long long)x->cols);
    if (x->rows != y->rows)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "shape mismatch: (%lld, 1) vs (%lld, 1)",
                    (long long)x->rows, (long long)y->rows);
    unsigned char *w = (unsigned char *)ws;
    unsigned *ticket = (unsigned *)w;
    double *dres = (double *)(w + 64);
    double *partials = (double *)(w + kReduceHeader);
    const int grid = elem_grid(x->rows);
    dot_kernel<V><<<grid, 256, 0, st>>>(x->rows, (const V *)x->data, x->stride, (const V *)y->data,
                                        y->stride, partials, ticket, dres);
    SB_CUDA(cudaGetLastError());
    if (x->rows == 0) {
        *out = 0.0;
        return SB_OK;
    }
    SB_CUDA(cudaMemcpyAsync(out, dres, sizeof(double), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    return SB_OK;
}

template <class V>
sb_status check_same(const sb_dense *x, const sb_dense *y, sb_error *err) {
    if (!x || !y) return fail(err, SB_ERR_INVALID_ARGUMENT, "null dense argument");
    if (x->rows != y->rows || x->cols != y->cols)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "shape mismatch: (%lld, %lld) vs (%lld, %lld)",
                    (long long)x->rows, (long long)x->cols, (long long)y->rows, (long long)y->cols);
    return SB_OK;
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_version(void) { return 1; }

const char *sb_status_string(int code) {
    switch (code) {
    case SB_OK: return "ok";
    case SB_ERR_INVALID_ARGUMENT: return "invalid-argument";
    case SB_ERR_DIMENSION_MISMATCH: return "dimension-mismatch";
    case SB_ERR_PRECISION_MISMATCH: return "precision-mismatch";
    case SB_ERR_UNSUPPORTED: return "unsupported-feature";
    case SB_ERR_INDEX_BOUNDS: return "index-bounds";
    case SB_ERR_BREAKDOWN: return "breakdown";
    case SB_ERR_NUMERIC_FAILURE: return "numeric-failure";
    case SB_ERR_SINGULAR_DIAGONAL: return "singular-diagonal";
    case SB_ERR_CUDA: return "cuda-error";
    case SB_ERR_NCCL: return "nccl-error";
    default: return "unknown";
    }
}

size_t sb_reduce_workspace_bytes(void) { return kReduceBytes; }

#define SB_BLAS1_DEFS(V, VN)                                                                       \
    sb_status sb_dot_##VN(const sb_dense *x, const sb_dense *y, double *out, void *workspace,      \
                          sb_stream_t stream, sb_error *err) {                                     \
        SB_GUARD_BEGIN                                                                             \
        return do_dot<V>(x, y, out, workspace, as_stream(stream), err);                            \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_norm2_##VN(const sb_dense *x, double *out, void *workspace, sb_stream_t stream,   \
                            sb_error *err) {                                                       \
        SB_GUARD_BEGIN                                                                             \
        double d = 0.0;                                                                            \
        sb_status s = do_dot<V>(x, x, &d, workspace, as_stream(stream), err);                      \
        if (s != SB_OK) return s;                                                                  \
        *out = sqrt(d);                                                                            \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_axpy_##VN(double alpha, const sb_dense *x, sb_dense *y, sb_stream_t stream,       \
                           sb_error *err) {                                                        \
        SB_GUARD_BEGIN                                                                             \
        sb_status s = check_same<V>(x, y, err);                                                    \
        if (s != SB_OK) return s;                                                                  \
        if (x->rows * x->cols == 0) return SB_OK;                                                  \
        axpy_kernel<V><<<elem_grid(x->rows * x->cols), 256, 0, as_stream(stream)>>>(               \
            x->rows, x->cols, alpha, (const V *)x->data, x->stride, (V *)y->data, y->stride);      \
        SB_CUDA(cudaGetLastError());                                                               \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_scal_##VN(double alpha, sb_dense *x, sb_stream_t stream, sb_error *err) {         \
        SB_GUARD_BEGIN                                                                             \
        if (!x) return fail(err, SB_ERR_INVALID_ARGUMENT, "scal: null x");                         \
        if (x->rows * x->cols == 0) return SB_OK;                                                  \
        scal_kernel<V><<<elem_grid(x->rows * x->cols), 256, 0, as_stream(stream)>>>(               \
            x->rows, x->cols, alpha, (V *)x->data, x->stride);                                     \
        SB_CUDA(cudaGetLastError());                                                               \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_copy_##VN(const sb_dense *src, sb_dense *dst, sb_stream_t stream, sb_error *err) { \
        SB_GUARD_BEGIN                                                                             \
        sb_status s = check_same<V>(src, dst, err);                                                \
        if (s != SB_OK) return s;                                                                  \
        if (src->rows * src->cols == 0) return SB_OK;                                              \
        copy_kernel<V><<<elem_grid(src->rows * src->cols), 256, 0, as_stream(stream)>>>(           \
            src->rows, src->cols, (const V *)src->data, src->stride, (V *)dst->data, dst->stride); \
        SB_CUDA(cudaGetLastError());                                                               \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_fill_##VN(sb_dense *x, double value, sb_stream_t stream, sb_error *err) {         \
        SB_GUARD_BEGIN                                                                             \
        if (!x) return fail(err, SB_ERR_INVALID_ARGUMENT, "fill: null x");                         \
        SB_CUDA(launch_fill<V>(x->rows, x->cols, (V *)x->data, x->stride, (V)value,                \
                               as_stream(stream)));                                                \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_jacobi_apply_##VN(const void *inv_diag, const sb_dense *b, sb_dense *x,           \
                                   sb_stream_t stream, sb_error *err) {                            \
        SB_GUARD_BEGIN                                                                             \
        sb_status s = check_same<V>(b, x, err);                                                    \
        if (s != SB_OK) return s;                                                                  \
        if (b->rows * b->cols == 0) return SB_OK;                                                  \
        jacobi_apply_kernel<V><<<elem_grid(b->rows * b->cols), 256, 0, as_stream(stream)>>>(       \
            b->rows, b->cols, (const V *)inv_diag, (const V *)b->data, b->stride, (V *)x->data,    \
            x->stride);                                                                            \
        SB_CUDA(cudaGetLastError());                                                               \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }

SB_BLAS1_DEFS(float, float)
SB_BLAS1_DEFS(double, double)

}  // extern "C"
