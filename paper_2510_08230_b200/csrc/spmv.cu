// spmv.cu -- SpMV entry points (every format x value x index), CSR row statistics and
// kernel selection, and LinOp.apply_advanced.
//
// Reference: linop.spmv_csr (linop.py:102-121), spmv_coo (linop.py:137-159),
// apply_advanced (linop.py:81-99); the binding seats bindings.csr_spmv_* /
// coo_spmv_* (bindings.py:116-123).
#include <algorithm>
#include <cmath>

#include "capi_util.cuh"
#include "spmv_launch.cuh"

namespace sb {

// ---------------------------------------------------------------- row statistics
template <class I>
__global__ void __launch_bounds__(256) row_stats_kernel(int64_t rows, const I *__restrict__ rp,
                                                        unsigned long long *acc) {
    // acc: [0] min len, [1] max len, [2] sum len, [3] sum len^2, [4] empty rows,
    //      [5..8] max nnz of aligned 32/64/128/256-row blocks
    unsigned long long mn = ~0ull, mx = 0, s = 0, s2 = 0, empty = 0, bm[4] = {0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long len = (unsigned long long)(rp[i + 1] - rp[i]);
        mn = len < mn ? len : mn;
        mx = len > mx ? len : mx;
        s += len;
        s2 += len * len;
        empty += len == 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t R = 32LL << q;
            if (i % R == 0) {
                const int64_t e = i + R < rows ? i + R : rows;
                const unsigned long long bn = (unsigned long long)(rp[e] - rp[i]);
                bm[q] = bn > bm[q] ? bn : bm[q];
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_down_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
        s += __shfl_down_sync(0xffffffffu, s, o);
        s2 += __shfl_down_sync(0xffffffffu, s2, o);
        empty += __shfl_down_sync(0xffffffffu, empty, o);
#pragma unroll
        for (int q = 0; q < 4; ++q) bm[q] = max(bm[q], __shfl_down_sync(0xffffffffu, bm[q], o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(acc + 0, mn);
        atomicMax(acc + 1, mx);
        atomicAdd(acc + 2, s);
        atomicAdd(acc + 3, s2);
        atomicAdd(acc + 4, empty);
#pragma unroll
        for (int q = 0; q < 4; ++q) atomicMax(acc + 5 + q, bm[q]);
    }
}

__global__ void stats_init_kernel(unsigned long long *acc) {
    if (threadIdx.x < 16) acc[threadIdx.x] = threadIdx.x == 0 ? ~0ull : 0ull;
}

template <class I>
sb_status row_stats(int64_t rows, const void *row_ptrs, void *ws, sb_row_stats *out,
                    cudaStream_t st, sb_error *err) {
    if (!out || !ws || (rows > 0 && !row_ptrs))
        return fail(err, SB_ERR_INVALID_ARGUMENT, "row_stats: null argument");
    unsigned long long *acc = (unsigned long long *)((unsigned char *)ws + kReduceScratch);
    stats_init_kernel<<<1, 32, 0, st>>>(acc);
    if (rows > 0)
        row_stats_kernel<I><<<elem_grid(rows), 256, 0, st>>>(rows, (const I *)row_ptrs, acc);
    SB_CUDA(cudaGetLastError());
    unsigned long long h[16];
    SB_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    out->rows = rows;
    out->nnz = (int64_t)h[2];
    out->min_len = rows ? (int64_t)h[0] : 0;
    out->max_len = (int64_t)h[1];
    out->empty_rows = (int64_t)h[4];
    out->mean_len = rows ? (double)h[2] / (double)rows : 0.0;
    const double var = rows ? (double)h[3] / (double)rows - out->mean_len * out->mean_len : 0.0;
    out->std_len = var > 0 ? std::sqrt(var) : 0.0;
    for (int q = 0; q < 4; ++q) out->max_block_nnz[q] = (int64_t)h[5 + q];
    return SB_OK;
}

// ---------------------------------------------------------------- kernel selection
// Stream (bit-exact, TMA-staged) for regular short rows; vector for long regular rows;
// merge-path when the row-length distribution is irregular (max >> mean).
sb_status plan_select(const sb_row_stats *S, int vbytes, int ibytes, int force, sb_csr_plan *P,
                      sb_error *err) {
    if (!S || !P) return fail(err, SB_ERR_INVALID_ARGUMENT, "plan_select: null argument");
    std::memset(P, 0, sizeof(*P));
    const double mean = S->mean_len;
    int kernel = force;
    // stream feasibility: two stages of one R-row block must fit comfortably in smem
    int stream_R = 0, stream_cap = 0;
    // 128-row blocks first: best measured (0.946 / 0.967 of the copy peak at 128^3 / 256^3,
    // tools/tune_stream.py) -- finer tail balance at 8 CTAs of smem per SM
    const int Rs[3] = {128, 256, 64};
    const int qidx[3] = {2, 3, 1};
    for (int t = 0; t < 3; ++t) {
        const int64_t cap = S->max_block_nnz[qidx[t]];
        const size_t bytes = 2 * ((size_t)(cap + 16) * (vbytes + ibytes) + (size_t)(Rs[t] + 16) * ibytes);
        if (cap < (1 << 30) && bytes <= 96 * 1024) {
            stream_R = Rs[t];
            stream_cap = (int)std::max<int64_t>(cap, 1);
            break;
        }
    }
    if (kernel == SB_CSR_AUTO) {
        const bool irregular = (double)S->max_len > 8.0 * mean + 64.0;
        if (S->rows == 0 || S->nnz == 0) kernel = SB_CSR_STRICT;
        else if (irregular) kernel = SB_CSR_TILE;
        else if (stream_R && mean <= 48.0) kernel = SB_CSR_STREAM;
        else kernel = SB_CSR_VECTOR;
    }
    if (kernel == SB_CSR_STREAM && !stream_R) {
        return fail(err, SB_ERR_UNSUPPORTED,
                    "stream CSR kernel needs <= %d nnz per 64-row block", 96 * 1024 / 2 / (vbytes + ibytes));
    }
    P->kernel = kernel;
    if (kernel == SB_CSR_STREAM) {
        P->block_rows = stream_R;
        P->nnz_cap = stream_cap;
        const int64_t cap256 = S->max_block_nnz[3];
        const size_t bytes256 = 2 * ((size_t)(cap256 + 16) * (vbytes + ibytes) + (size_t)(256 + 16) * ibytes);
        P->nnz_cap256 = (cap256 < (1 << 30) && bytes256 <= 96 * 1024) ? (int)std::max<int64_t>(cap256, 1) : 0;
    } else if (kernel == SB_CSR_VECTOR) {
        int lanes = 2;
        while (lanes < 32 && lanes < mean / 2.0) lanes <<= 1;
        P->block_rows = lanes;
    } else if (kernel == SB_CSR_MERGE) {
        P->items_per_tile = kMergeNT * kMergeIPT;
        P->num_tiles = ceil_div(S->rows + S->nnz, P->items_per_tile);
    } else if (kernel == SB_CSR_TILE) {
        P->items_per_tile = tile_nnz_default();
        P->num_tiles = 2 * ceil_div(S->nnz, P->items_per_tile);  // lead + trail record per tile
    }
    return SB_OK;
}

template <class I>
sb_status plan_build(int64_t rows, int64_t nnz, const void *rp, sb_csr_plan *P, cudaStream_t st,
                     sb_error *err) {
    if (!P) return fail(err, SB_ERR_INVALID_ARGUMENT, "plan_build: null plan");
    if ((P->kernel != SB_CSR_MERGE && P->kernel != SB_CSR_TILE) || P->num_tiles == 0) return SB_OK;
    if (!P->tile_rows || !P->tile_nnz || !P->carry_rows || !P->carry_vals)
        return fail(err, SB_ERR_INVALID_ARGUMENT, "merge / tile plan buffers not allocated");
    if (P->kernel == SB_CSR_TILE) {
        const int64_t nt = P->num_tiles / 2;
        tile_partition_kernel<I><<<(int)ceil_div(nt + 1, 256), 256, 0, st>>>(
            rows, (const I *)rp, P->items_per_tile, nt, (int64_t *)P->tile_rows);
        SB_CUDA(cudaGetLastError());
        return SB_OK;
    }
    const int64_t n = P->num_tiles + 1;
    merge_path_partition_kernel<I><<<(int)ceil_div(n, 256), 256, 0, st>>>(
        rows, nnz, (const I *)rp, P->items_per_tile, P->num_tiles, (int64_t *)P->tile_rows,
        (int64_t *)P->tile_nnz);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

// ---------------------------------------------------------------- argument checks
inline sb_status check_apply(int64_t rows, int64_t cols, const sb_dense *b, const sb_dense *x,
                             sb_error *err) {
    if (!b || !x) return fail(err, SB_ERR_INVALID_ARGUMENT, "null dense argument");
    if (b->rows != cols || x->rows != rows || b->cols != x->cols)
        return fail(err, SB_ERR_DIMENSION_MISMATCH,
                    "apply shape mismatch: op is %lldx%lld, b is %lldx%lld, x is %lldx%lld",
                    (long long)rows, (long long)cols, (long long)b->rows, (long long)b->cols,
                    (long long)x->rows, (long long)x->cols);
    return SB_OK;
}

// one launch sequence per right-hand-side column (linop.py:115 loops the same way)
template <class V, class I>
sb_status spmv_matrix(const sb_matrix &M, const sb_dense *b, sb_dense *x, cudaStream_t st,
                      sb_error *err) {
    const int64_t rows = matrix_rows(M), cols = matrix_cols(M);
    sb_status s = check_apply(rows, cols, b, x, err);
    if (s != SB_OK) return s;
    if (M.format == SB_FMT_CSR && ((const sb_csr *)M.mat)->nnz > 0 && !((const sb_csr *)M.mat)->plan)
        return fail(err, SB_ERR_INVALID_ARGUMENT, "CSR matrix has no plan");
    int64_t j = 0;
    if (b->cols > 1 && M.format == SB_FMT_CSR) {  // stream SpMM: the matrix once per 8/4/2 columns
        const sb_csr &A = *(const sb_csr *)M.mat;
        if (A.plan && A.plan->kernel == SB_CSR_STREAM && A.rows > 0) {
            while (b->cols - j >= 2) {
                const int K = b->cols - j >= 8 ? 8 : (b->cols - j >= 4 ? 4 : 2);
                const V *bj = (const V *)b->data + j;
                V *xj = (V *)x->data + j;
                cudaError_t e = K == 8 ? launch_csr_spmm<V, I, 8>(A, bj, b->stride, xj, x->stride, st)
                                : K == 4 ? launch_csr_spmm<V, I, 4>(A, bj, b->stride, xj, x->stride, st)
                                         : launch_csr_spmm<V, I, 2>(A, bj, b->stride, xj, x->stride, st);
                SB_CUDA(e);
                j += K;
            }
        }
    }
    for (; j < b->cols; ++j) {
        const V *bj = (const V *)b->data + j;
        V *xj = (V *)x->data + j;
        SB_CUDA((matrix_apply<V, I>(M, bj, b->stride, xj, x->stride, EpiStore<V>{xj, x->stride}, st)));
    }
    return SB_OK;
}

template <class V>
__global__ void __launch_bounds__(256) advanced_kernel(int64_t rows, int64_t cols, double alpha,
                                                       const V *t, double beta, V *x, int64_t ldx) {
    // linop.apply_advanced: beta == 0 -> copy + scal(alpha); else scal(beta) + axpy(alpha, t)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / cols, j = e % cols;
        V &xi = x[i * ldx + j];
        const V ti = t[e];
        xi = beta == 0.0 ? scal_e(alpha, ti) : axpy_e(alpha, ti, scal_e(beta, xi));
    }
}

template <class V, class I>
sb_status apply_advanced(const sb_matrix *M, double alpha, const sb_dense *b, double beta,
                         sb_dense *x, void *tmp, cudaStream_t st, sb_error *err) {
    if (!M || !tmp) return fail(err, SB_ERR_INVALID_ARGUMENT, "apply_advanced: null argument");
    const int64_t rows = matrix_rows(*M), cols = matrix_cols(*M);
    sb_status s = check_apply(rows, cols, b, x, err);
    if (s != SB_OK) return s;
    sb_dense t{tmp, x->rows, x->cols, x->cols};
    s = spmv_matrix<V, I>(*M, b, &t, st, err);
    if (s != SB_OK) return s;
    if (rows * x->cols == 0) return SB_OK;
    advanced_kernel<V><<<elem_grid(rows * x->cols), 256, 0, st>>>(rows, x->cols, alpha, (const V *)tmp,
                                                                   beta, (V *)x->data, x->stride);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

}  // namespace sb

using namespace sb;

extern "C" {

sb_status sb_csr_plan_select(const sb_row_stats *stats, int32_t value_bytes, int32_t index_bytes,
                             int32_t force, sb_csr_plan *plan, sb_error *err) {
    SB_GUARD_BEGIN
    return plan_select(stats, value_bytes, index_bytes, force, plan, err);
    SB_GUARD_END
}

int64_t sb_coo_tile_entries(void) { return kCooChunk; }

#define SB_IDX_SPMV_DEFS(I, IN)                                                                    \
    sb_status sb_csr_row_stats_##IN(int64_t rows, const void *row_ptrs, void *workspace,           \
                                    sb_row_stats *out, sb_stream_t stream, sb_error *err) {        \
        SB_GUARD_BEGIN                                                                             \
        return row_stats<I>(rows, row_ptrs, workspace, out, as_stream(stream), err);               \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_csr_plan_build_##IN(int64_t rows, int64_t nnz, const void *row_ptrs,             \
                                     sb_csr_plan *plan, sb_stream_t stream, sb_error *err) {       \
        SB_GUARD_BEGIN                                                                             \
        return plan_build<I>(rows, nnz, row_ptrs, plan, as_stream(stream), err);                   \
        SB_GUARD_END                                                                               \
    }

SB_IDX_SPMV_DEFS(int32_t, i32)
SB_IDX_SPMV_DEFS(int64_t, i64)

#define SB_SPMV_DEFS(V, VN, I, IN)                                                                 \
    sb_status sb_csr_spmv_##VN##_##IN(const sb_csr *a, const sb_dense *b, sb_dense *x,             \
                                      sb_stream_t stream, sb_error *err) {                         \
        SB_GUARD_BEGIN                                                                             \
        if (!a) return fail(err, SB_ERR_INVALID_ARGUMENT, "null matrix");                          \
        sb_matrix m{SB_FMT_CSR, 0, a};                                                             \
        return spmv_matrix<V, I>(m, b, x, as_stream(stream), err);                                 \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_coo_spmv_##VN##_##IN(const sb_coo *a, const sb_dense *b, sb_dense *x,             \
                                      sb_stream_t stream, sb_error *err) {                         \
        SB_GUARD_BEGIN                                                                             \
        if (!a) return fail(err, SB_ERR_INVALID_ARGUMENT, "null matrix");                          \
        if (a->nnz > 0 && !a->plan) return fail(err, SB_ERR_INVALID_ARGUMENT, "COO without plan"); \
        sb_matrix m{SB_FMT_COO, 0, a};                                                             \
        return spmv_matrix<V, I>(m, b, x, as_stream(stream), err);                                 \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_ell_spmv_##VN##_##IN(const sb_ell *a, const sb_dense *b, sb_dense *x,             \
                                      sb_stream_t stream, sb_error *err) {                         \
        SB_GUARD_BEGIN                                                                             \
        if (!a) return fail(err, SB_ERR_INVALID_ARGUMENT, "null matrix");                          \
        sb_matrix m{SB_FMT_ELL, 0, a};                                                             \
        return spmv_matrix<V, I>(m, b, x, as_stream(stream), err);                                 \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_sellp_spmv_##VN##_##IN(const sb_sellp *a, const sb_dense *b, sb_dense *x,         \
                                        sb_stream_t stream, sb_error *err) {                       \
        SB_GUARD_BEGIN                                                                             \
        if (!a) return fail(err, SB_ERR_INVALID_ARGUMENT, "null matrix");                          \
        sb_matrix m{SB_FMT_SELLP, 0, a};                                                           \
        return spmv_matrix<V, I>(m, b, x, as_stream(stream), err);                                 \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_hybrid_spmv_##VN##_##IN(const sb_hybrid *a, const sb_dense *b, sb_dense *x,       \
                                         sb_stream_t stream, sb_error *err) {                      \
        SB_GUARD_BEGIN                                                                             \
        if (!a) return fail(err, SB_ERR_INVALID_ARGUMENT, "null matrix");                          \
        if (a->coo.nnz > 0 && !a->coo.plan)                                                        \
            return fail(err, SB_ERR_INVALID_ARGUMENT, "hybrid COO part without plan");             \
        sb_matrix m{SB_FMT_HYBRID, 0, a};                                                          \
        return spmv_matrix<V, I>(m, b, x, as_stream(stream), err);                                 \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_apply_advanced_##VN##_##IN(const sb_matrix *a, double alpha, const sb_dense *b,   \
                                            double beta, sb_dense *x, void *tmp,                   \
                                            sb_stream_t stream, sb_error *err) {                   \
        SB_GUARD_BEGIN                                                                             \
        return apply_advanced<V, I>(a, alpha, b, beta, x, tmp, as_stream(stream), err);            \
        SB_GUARD_END                                                                               \
    }

SB_SPMV_DEFS(float, float, int32_t, i32)
SB_SPMV_DEFS(float, float, int64_t, i64)
SB_SPMV_DEFS(double, double, int32_t, i32)
SB_SPMV_DEFS(double, double, int64_t, i64)

}  // extern "C"
