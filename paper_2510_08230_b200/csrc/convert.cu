// convert.cu -- storage construction and conversion on the device.
//
// Reference: coo_from_arrays (formats.py:131-166), csr_from_coo (:184-191),
// coo_from_csr (:194-199), CsrMatrix.diagonal + jacobi_create (formats.py:113-122,
// precond.py:66-84); ELL / SELL-P / Hybrid follow the canonical layouts pinned in
// SURVEY.md §8 (the reference has none).  Integer outputs are bit-exact
// with the reference / oracle; the only arithmetic is the duplicate sum of
// canonicalisation, done strictly left to right within each (row, col) run.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "capi_util.cuh"
#include "spmv_launch.cuh"

namespace sb {

template <class T>
__device__ __forceinline__ int64_t lower_bound_dev(const T *a, int64_t n, int64_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// csr_from_coo: row_ptrs[i] = #entries with row < i (== bincount + cumsum)
template <class I>
__global__ void row_ptrs_from_sorted_kernel(int64_t rows, int64_t nnz, const I *ri, I *rp) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= rows;
         i += (int64_t)gridDim.x * blockDim.x)
        rp[i] = (I)lower_bound_dev(ri, nnz, i);
}

// coo_from_csr: entry k belongs to the last row whose start is <= k (empty rows skipped)
template <class I>
__global__ void row_idxs_from_csr_kernel(int64_t rows, int64_t nnz, const I *rp, I *ri) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        // upper_bound(rp[0..rows], k) - 1
        int64_t lo = 0, hi = rows + 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)rp[mid] <= k) lo = mid + 1;
            else hi = mid;
        }
        ri[k] = (I)(lo - 1);
    }
}

// jacobi_create: stored diagonal by binary search in the sorted row (np.searchsorted),
// inv = (1 / diag in fp64) cast to V; first zero row and first non-finite row recorded.
template <class V, class I>
__global__ void jacobi_kernel(int64_t n, const I *rp, const I *ci, const V *val, V *inv,
                              unsigned long long *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b0 = rp[i], b1 = rp[i + 1];
        const int64_t k = b0 + lower_bound_dev(ci + b0, b1 - b0, i);
        const V d = (k < b1 && (int64_t)ci[k] == i) ? val[k] : (V)0;
        if (d == (V)0) {
            atomicMin(bad, (unsigned long long)i);
            inv[i] = (V)0;
            continue;
        }
        const V r = (V)__drcp_rn((double)d);  // 1.0 / d correctly rounded in fp64, then cast
        inv[i] = r;
        if (!isfinite((double)r)) atomicMin(bad + 1, (unsigned long long)i);
    }
}

__global__ void init_bad_kernel(unsigned long long *bad) {
    if (threadIdx.x < 2) bad[threadIdx.x] = ~0ull;
}

// ---------------------------------------------------------------- ELL / SELL-P / Hybrid
template <class V, class I>
__global__ void ell_fill_kernel(int64_t rows, int64_t width, int64_t stride, const I *rp,
                                const I *ci, const V *val, I *ec, V *ev, const I *tail_ptrs,
                                I *trow, I *tcol, V *tval) {
    // thread per row of the padded stride; columns beyond `width` go to the COO tail
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < stride;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b0 = i < rows ? (int64_t)rp[i] : 0;
        const int64_t len = i < rows ? (int64_t)rp[i + 1] - b0 : 0;
        for (int64_t k = 0; k < width; ++k) {
            const int64_t dst = k * stride + i;
            if (k < len) {
                ec[dst] = ci[b0 + k];
                ev[dst] = val[b0 + k];
            } else {
                ec[dst] = (I)-1;
                ev[dst] = (V)0;
            }
        }
        if (tail_ptrs && i < rows) {
            int64_t t = tail_ptrs[i];
            for (int64_t k = width; k < len; ++k, ++t) {
                trow[t] = (I)i;
                tcol[t] = ci[b0 + k];
                tval[t] = val[b0 + k];
            }
        }
    }
}

template <class I>
__global__ void slice_lengths_kernel(int64_t rows, int64_t S, const I *rp, I *sl, int64_t ns) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < ns;
         s += (int64_t)gridDim.x * blockDim.x) {
        int64_t m = 0;
        const int64_t e = (s + 1) * S < rows ? (s + 1) * S : rows;
        for (int64_t i = s * S; i < e; ++i) {
            const int64_t len = rp[i + 1] - rp[i];
            m = len > m ? len : m;
        }
        sl[s] = (I)m;
    }
}

// exclusive scan in a single CTA (out has n + 1 entries; out[n] is the total).  Used once
// per conversion on slice / row counts, so simplicity wins over a multi-CTA scan.
template <class I>
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(int64_t n, const I *in, I *out) {
    // out[0] = 0, out[i+1] = sum(in[0..i]); one CTA, each thread scans a contiguous chunk
    __shared__ long long s_part[1024];
    const int T = blockDim.x, t = threadIdx.x;
    const int64_t chunk = (n + T - 1) / T;
    const int64_t lo = t * chunk < n ? t * chunk : n;
    const int64_t hi = lo + chunk < n ? lo + chunk : n;
    long long acc = 0;
    for (int64_t i = lo; i < hi; ++i) acc += (long long)in[i];
    s_part[t] = acc;
    __syncthreads();
    if (t == 0) {
        long long run = 0;
        for (int u = 0; u < T; ++u) {
            const long long v = s_part[u];
            s_part[u] = run;
            run += v;
        }
        out[0] = 0;
    }
    __syncthreads();
    long long run = s_part[t];
    for (int64_t i = lo; i < hi; ++i) {
        run += (long long)in[i];
        out[i + 1] = (I)run;
    }
}

template <class I>
__global__ void tail_counts_kernel(int64_t rows, const I *rp, int64_t width, I *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = (int64_t)rp[i + 1] - rp[i];
        cnt[i] = (I)(len > width ? len - width : 0);
    }
}

template <class V, class I>
__global__ void sellp_fill_kernel(int64_t rows, int64_t S, int64_t ns, const I *rp, const I *ci,
                                  const V *val, const I *sl, const I *ss, I *sc, V *sv) {
    // thread per (slice row slot); loops the slice's columns (coalesced across the slice)
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ns * S;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = g / S, l = g % S, i = g;
        const int64_t len_s = sl[s];
        const int64_t b0 = i < rows ? (int64_t)rp[i] : 0;
        const int64_t len = i < rows ? (int64_t)rp[i + 1] - b0 : 0;
        const int64_t base = (int64_t)ss[s] * S + l;
        for (int64_t k = 0; k < len_s; ++k) {
            const int64_t dst = base + k * S;
            if (k < len) {
                sc[dst] = ci[b0 + k];
                sv[dst] = val[b0 + k];
            } else {
                sc[dst] = (I)-1;
                sv[dst] = (V)0;
            }
        }
    }
}

// ---------------------------------------------------------------- stencil generator
// Canonical CSR of the SURVEY.md §10 stencils without a sort: row i's entries in
// ascending column order, row_ptrs from the closed-form count of missing neighbours.
__device__ __forceinline__ int64_t count_eq(int64_t i, int64_t s, int64_t p, int64_t v) {
    // #{ j < i : (j / s) % p == v }
    const int64_t T = s * p, full = i / T, rem = i % T;
    int64_t part = rem - v * s;
    part = part < 0 ? 0 : (part > s ? s : part);
    return full * s + part;
}

template <class V, class I>
__global__ void stencil_kernel(int64_t p, int dim, double c, int64_t lo, int64_t hi, I *rp, I *ci,
                               V *val) {
    // rows [lo, hi) of the global stencil; row_ptrs relative to row lo, columns global
    const double lo_v = -1.0 - c / 2.0, hi_v = -1.0 + c / 2.0;
    auto start_of = [&](int64_t i) {
        int64_t st = (2 * dim + 1) * i;
        int64_t s = 1;
        for (int d = 0; d < dim; ++d, s *= p) st -= count_eq(i, s, p, 0) + count_eq(i, s, p, p - 1);
        return st;
    };
    const int64_t base = start_of(lo);
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= hi;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t start = start_of(i) - base;
        rp[i - lo] = (I)start;
        if (i == hi) continue;
        int64_t g[3] = {i % p, (i / p) % p, dim == 3 ? i / (p * p) : 0};
        int64_t strides[3] = {1, p, p * p};
        int64_t k = start;
        // lower neighbours, largest offset first (ascending columns)
        for (int d = dim - 1; d >= 0; --d)
            if (g[d] > 0) {
                ci[k] = (I)(i - strides[d]);
                val[k++] = (V)lo_v;
            }
        ci[k] = (I)i;
        val[k++] = (V)(2.0 * dim);
        for (int d = 0; d < dim; ++d)
            if (g[d] < p - 1) {
                ci[k] = (I)(i + strides[d]);
                val[k++] = (V)hi_v;
            }
    }
}

// ---------------------------------------------------------------- coo_from_arrays
__global__ void bounds_kernel(int64_t count, int64_t rows, int64_t cols, const int64_t *ri,
                              const int64_t *ci, unsigned long long *bad, unsigned long long *keys,
                              unsigned long long *idx) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = ri[k], c = ci[k];
        if (r < 0 || r >= rows || c < 0 || c >= cols) {
            atomicMin(bad, (unsigned long long)k);
            keys[k] = 0;
        } else {
            keys[k] = (unsigned long long)r * (unsigned long long)cols + (unsigned long long)c;
        }
        idx[k] = (unsigned long long)k;
    }
}

__global__ void heads_kernel(int64_t count, const unsigned long long *keys, unsigned long long *head) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x)
        head[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1ull : 0ull;
}

template <class T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <class V, class I>
__global__ void emit_runs_kernel(int64_t count, int64_t cols, const unsigned long long *keys,
                                 const unsigned long long *idx, const unsigned long long *run_id,
                                 const V *vals, I *orow, I *ocol, V *oval) {
    // run_id = inclusive scan of heads; a head emits its run's left-to-right sum
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (!(k == 0 || keys[k] != keys[k - 1])) continue;
        const int64_t out = (int64_t)run_id[k] - 1;
        V acc = vals[idx[k]];
        for (int64_t q = k + 1; q < count && keys[q] == keys[k]; ++q) acc = add_rn(acc, vals[idx[q]]);
        orow[out] = (I)(keys[k] / (unsigned long long)cols);
        ocol[out] = (I)(keys[k] % (unsigned long long)cols);
        oval[out] = acc;
    }
}

struct CanonWs {
    unsigned long long *bad, *k0, *k1, *i0, *i1, *head, *run;
    void *cub;
    size_t cub_bytes;
};

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

inline size_t cub_bytes_for(int64_t count) {
    size_t sort_b = 0, scan_b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (unsigned long long *)nullptr,
                                    (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (unsigned long long *)nullptr, (int)std::max<int64_t>(count, 1));
    cub::DeviceScan::InclusiveSum(nullptr, scan_b, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, (int)std::max<int64_t>(count, 1));
    return align256(std::max(sort_b, scan_b));
}

inline size_t canon_bytes(int64_t count) {
    const size_t arr = align256(sizeof(unsigned long long) * (size_t)std::max<int64_t>(count, 1));
    return 256 + 6 * arr + cub_bytes_for(count);
}

inline CanonWs carve(void *ws, int64_t count) {
    unsigned char *p = (unsigned char *)ws;
    const size_t arr = align256(sizeof(unsigned long long) * (size_t)std::max<int64_t>(count, 1));
    CanonWs w;
    w.bad = (unsigned long long *)p;
    p += 256;
    w.k0 = (unsigned long long *)p; p += arr;
    w.k1 = (unsigned long long *)p; p += arr;
    w.i0 = (unsigned long long *)p; p += arr;
    w.i1 = (unsigned long long *)p; p += arr;
    w.head = (unsigned long long *)p; p += arr;
    w.run = (unsigned long long *)p; p += arr;
    w.cub = p;
    w.cub_bytes = cub_bytes_for(count);
    return w;
}

template <class V, class I>
sb_status coo_from_arrays(int64_t rows, int64_t cols, int64_t count, const int64_t *ri,
                          const int64_t *ci, const void *values, void *out_rows, void *out_cols,
                          void *out_vals, void *ws, size_t ws_bytes, int64_t *nnz_out,
                          cudaStream_t st, sb_error *err) {
    if (rows < 0 || cols < 0) return fail(err, SB_ERR_INVALID_ARGUMENT, "rows and cols must be non-negative");
    if (!nnz_out) return fail(err, SB_ERR_INVALID_ARGUMENT, "null nnz_out");
    if (count == 0) {
        *nnz_out = 0;
        return SB_OK;
    }
    if (count > INT32_MAX) return fail(err, SB_ERR_UNSUPPORTED, "more than 2^31-1 raw triplets");
    if (ws_bytes < canon_bytes(count)) return fail(err, SB_ERR_INVALID_ARGUMENT, "workspace too small");
    CanonWs w = carve(ws, count);
    const int n = (int)count;
    init_bad_kernel<<<1, 32, 0, st>>>(w.bad);
    bounds_kernel<<<elem_grid(count), 256, 0, st>>>(count, rows, cols, ri, ci, w.bad, w.k0, w.i0);
    SB_CUDA(cudaGetLastError());
    unsigned long long bad = 0;
    SB_CUDA(cudaMemcpyAsync(&bad, w.bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    if (bad != ~0ull) {
        if (err) err->row = (int64_t)bad;
        return fail(err, SB_ERR_INDEX_BOUNDS, "triplet %lld outside %lldx%lld", (long long)bad,
                    (long long)rows, (long long)cols);
    }
    // stable radix sort of (row*cols + col) keys carrying the original position
    int end_bit = 1;
    while (end_bit < 64 && ((unsigned long long)rows * (unsigned long long)cols) > (1ull << end_bit)) ++end_bit;
    size_t cb = w.cub_bytes;
    SB_CUDA(cub::DeviceRadixSort::SortPairs(w.cub, cb, w.k0, w.k1, w.i0, w.i1, n, 0, end_bit, st));
    heads_kernel<<<elem_grid(count), 256, 0, st>>>(count, w.k1, w.head);
    SB_CUDA(cudaGetLastError());
    cb = w.cub_bytes;
    SB_CUDA(cub::DeviceScan::InclusiveSum(w.cub, cb, w.head, w.run, n, st));
    emit_runs_kernel<V, I><<<elem_grid(count), 256, 0, st>>>(count, cols, w.k1, w.i1, w.run,
                                                              (const V *)values, (I *)out_rows,
                                                              (I *)out_cols, (V *)out_vals);
    SB_CUDA(cudaGetLastError());
    unsigned long long nnz = 0;
    SB_CUDA(cudaMemcpyAsync(&nnz, w.run + (count - 1), sizeof(nnz), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    *nnz_out = (int64_t)nnz;
    return SB_OK;
}

template <class V, class I>
sb_status jacobi_create(const sb_csr *a, void *inv, void *ws, cudaStream_t st, sb_error *err) {
    if (!a || !inv || !ws) return fail(err, SB_ERR_INVALID_ARGUMENT, "jacobi_create: null argument");
    if (a->rows != a->cols)
        return fail(err, SB_ERR_DIMENSION_MISMATCH, "expected a square matrix, got %lldx%lld",
                    (long long)a->rows, (long long)a->cols);
    unsigned long long *bad = (unsigned long long *)((unsigned char *)ws + kReduceScratch);
    init_bad_kernel<<<1, 32, 0, st>>>(bad);
    if (a->rows > 0)
        jacobi_kernel<V, I><<<elem_grid(a->rows), 256, 0, st>>>(
            a->rows, (const I *)a->row_ptrs, (const I *)a->col_idxs, (const V *)a->values, (V *)inv,
            bad);
    SB_CUDA(cudaGetLastError());
    unsigned long long h[2];
    SB_CUDA(cudaMemcpyAsync(h, bad, sizeof(h), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    const unsigned long long row = h[0] != ~0ull ? h[0] : h[1];
    if (row != ~0ull) {
        if (err) err->row = (int64_t)row;
        return fail(err, SB_ERR_SINGULAR_DIAGONAL, "zero or missing diagonal at row %lld", (long long)row);
    }
    return SB_OK;
}

template <class V, class I>
sb_status ell_from_csr(const sb_csr *a, sb_ell *out, cudaStream_t st, sb_error *err) {
    if (!a || !out) return fail(err, SB_ERR_INVALID_ARGUMENT, "ell_from_csr: null argument");
    if (out->stride < a->rows) return fail(err, SB_ERR_INVALID_ARGUMENT, "ELL stride < rows");
    if (out->stride * out->width == 0) return SB_OK;
    ell_fill_kernel<V, I><<<elem_grid(out->stride), 256, 0, st>>>(
        a->rows, out->width, out->stride, (const I *)a->row_ptrs, (const I *)a->col_idxs,
        (const V *)a->values, (I *)out->col_idxs, (V *)out->values, nullptr, nullptr, nullptr, nullptr);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

template <class V, class I>
sb_status hybrid_from_csr(const sb_csr *a, const void *tail_ptrs, sb_hybrid *out, cudaStream_t st,
                          sb_error *err) {
    if (!a || !out || !tail_ptrs) return fail(err, SB_ERR_INVALID_ARGUMENT, "hybrid_from_csr: null argument");
    if (out->ell.stride < a->rows) return fail(err, SB_ERR_INVALID_ARGUMENT, "ELL stride < rows");
    if (out->ell.stride == 0) return SB_OK;
    ell_fill_kernel<V, I><<<elem_grid(out->ell.stride), 256, 0, st>>>(
        a->rows, out->ell.width, out->ell.stride, (const I *)a->row_ptrs, (const I *)a->col_idxs,
        (const V *)a->values, (I *)out->ell.col_idxs, (V *)out->ell.values, (const I *)tail_ptrs,
        (I *)out->coo.row_idxs, (I *)out->coo.col_idxs, (V *)out->coo.values);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

template <class V, class I>
sb_status sellp_from_csr(const sb_csr *a, sb_sellp *out, cudaStream_t st, sb_error *err) {
    if (!a || !out) return fail(err, SB_ERR_INVALID_ARGUMENT, "sellp_from_csr: null argument");
    if (out->num_slices == 0) return SB_OK;
    sellp_fill_kernel<V, I><<<elem_grid(out->num_slices * out->slice_size), 256, 0, st>>>(
        a->rows, out->slice_size, out->num_slices, (const I *)a->row_ptrs, (const I *)a->col_idxs,
        (const V *)a->values, (const I *)out->slice_lengths, (const I *)out->slice_sets,
        (I *)out->col_idxs, (V *)out->values);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

template <class I>
sb_status scan_counts(int64_t n, const I *in, I *out, int64_t *total, cudaStream_t st, sb_error *err) {
    exclusive_scan_kernel<I><<<1, 1024, 0, st>>>(n, in, out);
    SB_CUDA(cudaGetLastError());
    I h = 0;
    SB_CUDA(cudaMemcpyAsync(&h, out + n, sizeof(I), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    *total = (int64_t)h;
    return SB_OK;
}

template <class I>
sb_status sellp_slices(int64_t rows, const void *rp, int64_t S, void *sl, void *ss, int64_t *total,
                       cudaStream_t st, sb_error *err) {
    if (S <= 0 || !total) return fail(err, SB_ERR_INVALID_ARGUMENT, "slice size must be positive");
    const int64_t ns = ceil_div(rows, S);
    if (ns == 0) {
        SB_CUDA(cudaMemsetAsync(ss, 0, sizeof(I), st));
        *total = 0;
        return SB_OK;
    }
    slice_lengths_kernel<I><<<elem_grid(ns), 256, 0, st>>>(rows, S, (const I *)rp, (I *)sl, ns);
    SB_CUDA(cudaGetLastError());
    return scan_counts<I>(ns, (const I *)sl, (I *)ss, total, st, err);
}

template <class I>
sb_status hybrid_tail_ptrs(int64_t rows, const void *rp, int64_t width, void *tail_ptrs,
                           int64_t *tail_nnz, cudaStream_t st, sb_error *err) {
    if (!tail_nnz) return fail(err, SB_ERR_INVALID_ARGUMENT, "null tail_nnz");
    if (rows == 0) {
        SB_CUDA(cudaMemsetAsync(tail_ptrs, 0, sizeof(I), st));
        *tail_nnz = 0;
        return SB_OK;
    }
    // counts go to tail_ptrs[1..rows] first, then are scanned into place via a copy-free
    // two-step: counts into the upper slots, scan reads them before overwriting
    I *tp = (I *)tail_ptrs;
    tail_counts_kernel<I><<<elem_grid(rows), 256, 0, st>>>(rows, (const I *)rp, width, tp + 1);
    SB_CUDA(cudaGetLastError());
    // in-place exclusive scan of tp[1..rows] into tp[0..rows]: each scan thread reads its
    // chunk before writing (chunk-local), and writes land at i+1 >= read index
    return scan_counts<I>(rows, tp + 1, tp, tail_nnz, st, err);
}

template <class V, class I>
sb_status stencil(int64_t p, int dim, double c, int64_t lo, int64_t hi, void *rp, void *ci, void *val,
                  cudaStream_t st, sb_error *err) {
    if (p < 1 || (dim != 2 && dim != 3)) return fail(err, SB_ERR_INVALID_ARGUMENT, "stencil: p >= 1, dim in {2, 3}");
    const int64_t n = dim == 2 ? p * p : p * p * p;
    if (lo < 0) lo = 0;
    if (hi < 0 || hi > n) hi = n;
    if (lo > hi) return fail(err, SB_ERR_INVALID_ARGUMENT, "stencil: empty row range");
    stencil_kernel<V, I><<<elem_grid(hi - lo + 1), 256, 0, st>>>(p, dim, c, lo, hi, (I *)rp, (I *)ci, (V *)val);
    SB_CUDA(cudaGetLastError());
    return SB_OK;
}

}  // namespace sb

using namespace sb;

extern "C" {

size_t sb_coo_from_arrays_workspace_bytes(int64_t count) { return canon_bytes(count); }

#define SB_CONV_IDX(I, IN)                                                                         \
    sb_status sb_csr_row_ptrs_from_coo_##IN(int64_t rows, int64_t nnz, const void *row_idxs,       \
                                            void *row_ptrs, sb_stream_t stream, sb_error *err) {   \
        SB_GUARD_BEGIN                                                                             \
        row_ptrs_from_sorted_kernel<I><<<elem_grid(rows + 1), 256, 0, as_stream(stream)>>>(        \
            rows, nnz, (const I *)row_idxs, (I *)row_ptrs);                                        \
        SB_CUDA(cudaGetLastError());                                                               \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_coo_row_idxs_from_csr_##IN(int64_t rows, int64_t nnz, const void *row_ptrs,       \
                                            void *row_idxs, sb_stream_t stream, sb_error *err) {   \
        SB_GUARD_BEGIN                                                                             \
        if (nnz == 0) return SB_OK;                                                                \
        row_idxs_from_csr_kernel<I><<<elem_grid(nnz), 256, 0, as_stream(stream)>>>(               \
            rows, nnz, (const I *)row_ptrs, (I *)row_idxs);                                        \
        SB_CUDA(cudaGetLastError());                                                               \
        return SB_OK;                                                                              \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_sellp_slices_##IN(int64_t rows, const void *row_ptrs, int64_t slice_size,         \
                                   void *slice_lengths, void *slice_sets, int64_t *total,          \
                                   sb_stream_t stream, sb_error *err) {                            \
        SB_GUARD_BEGIN                                                                             \
        return sellp_slices<I>(rows, row_ptrs, slice_size, slice_lengths, slice_sets, total,       \
                               as_stream(stream), err);                                            \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_hybrid_tail_ptrs_##IN(int64_t rows, const void *row_ptrs, int64_t width,          \
                                       void *tail_ptrs, int64_t *tail_nnz, sb_stream_t stream,     \
                                       sb_error *err) {                                            \
        SB_GUARD_BEGIN                                                                             \
        return hybrid_tail_ptrs<I>(rows, row_ptrs, width, tail_ptrs, tail_nnz, as_stream(stream),  \
                                   err);                                                           \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_stencil_csr_double_##IN(int64_t p, int32_t dim, double c, int64_t row_lo,       \
                                         int64_t row_hi, void *row_ptrs,                           \
                                         void *col_idxs, void *values, sb_stream_t stream,         \
                                         sb_error *err) {                                          \
        SB_GUARD_BEGIN                                                                             \
        return stencil<double, I>(p, dim, c, row_lo, row_hi, row_ptrs, col_idxs, values,           \
                                  as_stream(stream), err);                                         \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_stencil_csr_float_##IN(int64_t p, int32_t dim, double c, int64_t row_lo,        \
                                        int64_t row_hi, void *row_ptrs,                            \
                                        void *col_idxs, void *values, sb_stream_t stream,          \
                                        sb_error *err) {                                           \
        SB_GUARD_BEGIN                                                                             \
        return stencil<float, I>(p, dim, c, row_lo, row_hi, row_ptrs, col_idxs, values,            \
                                 as_stream(stream), err);                                          \
        SB_GUARD_END                                                                               \
    }

SB_CONV_IDX(int32_t, i32)
SB_CONV_IDX(int64_t, i64)

#define SB_CONV_VI(V, VN, I, IN)                                                                   \
    sb_status sb_jacobi_create_##VN##_##IN(const sb_csr *a, void *inv_diag, void *workspace,      \
                                           sb_stream_t stream, sb_error *err) {                    \
        SB_GUARD_BEGIN                                                                             \
        return jacobi_create<V, I>(a, inv_diag, workspace, as_stream(stream), err);                \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_ell_from_csr_##VN##_##IN(const sb_csr *a, sb_ell *out, sb_stream_t stream,        \
                                          sb_error *err) {                                         \
        SB_GUARD_BEGIN                                                                             \
        return ell_from_csr<V, I>(a, out, as_stream(stream), err);                                 \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_sellp_from_csr_##VN##_##IN(const sb_csr *a, sb_sellp *out, sb_stream_t stream,    \
                                            sb_error *err) {                                       \
        SB_GUARD_BEGIN                                                                             \
        return sellp_from_csr<V, I>(a, out, as_stream(stream), err);                               \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_hybrid_from_csr_##VN##_##IN(const sb_csr *a, const void *coo_row_ptrs,           \
                                             sb_hybrid *out, sb_stream_t stream, sb_error *err) {  \
        SB_GUARD_BEGIN                                                                             \
        return hybrid_from_csr<V, I>(a, coo_row_ptrs, out, as_stream(stream), err);                \
        SB_GUARD_END                                                                               \
    }                                                                                              \
    sb_status sb_coo_from_arrays_##VN##_##IN(int64_t rows, int64_t cols, int64_t count,            \
                                             const int64_t *row_idxs, const int64_t *col_idxs,     \
                                             const void *values, void *out_rows, void *out_cols,   \
                                             void *out_vals, void *workspace,                      \
                                             size_t workspace_bytes, int64_t *nnz_out,             \
                                             sb_stream_t stream, sb_error *err) {                  \
        SB_GUARD_BEGIN                                                                             \
        return coo_from_arrays<V, I>(rows, cols, count, row_idxs, col_idxs, values, out_rows,      \
                                     out_cols, out_vals, workspace, workspace_bytes, nnz_out,      \
                                     as_stream(stream), err);                                      \
        SB_GUARD_END                                                                               \
    }

SB_CONV_VI(float, float, int32_t, i32)
SB_CONV_VI(float, float, int64_t, i64)
SB_CONV_VI(double, double, int32_t, i32)
SB_CONV_VI(double, double, int64_t, i64)

}  // extern "C"
