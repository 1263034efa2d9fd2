// spmv_launch.cuh -- host-side dispatch of the SpMV kernels for every storage format,
// templated on the fused epilogue so the solvers reuse the same launchers.
#pragma once

#include "../../include/sparseb200.h"
#include <algorithm>
#include <cstdlib>

#include "spmv.cuh"

namespace sb {

template <class E>
struct is_plain_store : std::false_type {};
template <class V>
struct is_plain_store<EpiStore<V>> : std::true_type {};

// persistent-grid size for a kernel instantiation (cached per instantiation)
template <class K>
int persistent_grid(K kernel, int threads, size_t smem) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (per_sm < 1) per_sm = 1;
    return per_sm * device_info().sms;
}

constexpr int kMergeNT = 128, kMergeIPT = 8;      // 1024 merge items per tile
// nnz-tile CSR: nonzeros per tile (1024 / 2048 / 4096 instantiated; 128 / 256 / 256
// threads), row pointers staged per tile = tile / 2
inline int tile_nnz_default() {
    static const int c = [] {
        const char *e = getenv("SPARSEB200_TILE_C");
        const int v = e ? atoi(e) : 2048;
        return (v == 1024 || v == 4096) ? v : 2048;
    }();
    return c;
}
constexpr int kCooNT = 128, kCooIPT = 8;          // 1024 entries per tile
constexpr int kElemThreads = 256;

inline int elem_grid(int64_t work_items) {
    int64_t g = ceil_div(work_items, kElemThreads);
    int64_t cap = (int64_t)device_info().sms * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ---------------------------------------------------------------- CSR
template <class V, class I, int R, class Epi, int NS>
cudaError_t launch_csr_stream_ns(const sb_csr &A, const V *b, int64_t ldb, const Epi &epi, cudaStream_t st) {
    const int cap = A.plan->nnz_cap;
    const StreamLayout<V, I> L(R, cap);
    const size_t smem = NS * L.stage_bytes();
    auto kern = csr_stream_kernel<V, I, R, Epi, NS>;
    ensure_max_smem((const void *)kern);
    int grid = persistent_grid(kern, R, smem);
    const int64_t nblk = ceil_div(A.rows, R);
    if (grid > nblk) grid = (int)nblk;
    if (is_plain_store<Epi>::value) {  // standalone SpMV: ordinary stream serialisation
        kern<<<grid, R, smem, st>>>(A.rows, A.nnz, (const I *)A.row_ptrs, (const I *)A.col_idxs,
                                    (const V *)A.values, b, ldb, cap, epi);
        return cudaGetLastError();
    }
    // inside solver loops: programmatic dependent launch (the matrix prefetch of the first
    // block overlaps the predecessor's drain; its predecessors never write the matrix)
    return launch_pdl(kern, grid, R, smem, st, A.rows, A.nnz, (const I *)A.row_ptrs,
                      (const I *)A.col_idxs, (const V *)A.values, b, ldb, cap, epi);
}

// TMA ring depth: 2 stages.  Measured (tools/tune_stream2.py, 128^3 fp64 R=256 / fp32
// R=256): 2 stages 36.7 / 32.3 us, 3 stages 41.6 / 33.9 us, 4 stages 50.3 / 36.4 us --
// deeper rings cost CTAs per SM without adding useful bytes in flight.
template <class V, class I, int R, class Epi>
cudaError_t launch_csr_stream(const sb_csr &A, const V *b, int64_t ldb, const Epi &epi, cudaStream_t st) {
    return launch_csr_stream_ns<V, I, R, Epi, 2>(A, b, ldb, epi, st);
}

template <class V, class I, int K>
cudaError_t launch_csr_spmm(const sb_csr &A, const V *b, int64_t ldb, V *x, int64_t ldx, cudaStream_t st) {
    constexpr int R = 128;
    const sb_csr_plan &P = *A.plan;
    const int cap = P.nnz_cap;  // a 128-row block holds at most the nnz of a 128- or 256-row plan block
    if (P.block_rows < 128) {  // 64-row plans: stage with their own cap at R = 64
        constexpr int R64 = 64;
        const size_t smem = 2 * StreamLayout<V, I>(R64, P.nnz_cap).stage_bytes();
        auto kern = csr_stream_spmm_kernel<V, I, R64, K>;
        ensure_max_smem((const void *)kern);
        int grid = persistent_grid(kern, R64, smem);
        const int64_t nblk = ceil_div(A.rows, R64);
        if (grid > nblk) grid = (int)nblk;
        kern<<<grid, R64, smem, st>>>(A.rows, A.nnz, (const I *)A.row_ptrs, (const I *)A.col_idxs,
                                      (const V *)A.values, b, ldb, x, ldx, P.nnz_cap);
        return cudaGetLastError();
    }
    const size_t smem = 2 * StreamLayout<V, I>(R, cap).stage_bytes();
    auto kern = csr_stream_spmm_kernel<V, I, R, K>;
    ensure_max_smem((const void *)kern);
    int grid = persistent_grid(kern, R, smem);
    const int64_t nblk = ceil_div(A.rows, R);
    if (grid > nblk) grid = (int)nblk;
    kern<<<grid, R, smem, st>>>(A.rows, A.nnz, (const I *)A.row_ptrs, (const I *)A.col_idxs,
                                (const V *)A.values, b, ldb, x, ldx, cap);
    return cudaGetLastError();
}

template <class V, class I, int S, class Epi>
cudaError_t launch_csr_vector(const sb_csr &A, const V *b, int64_t ldb, const Epi &epi,
                              cudaStream_t st) {
    auto kern = csr_vector_kernel<V, I, S, Epi>;
    int grid = persistent_grid(kern, 256, 0);
    const int64_t need = ceil_div(A.rows * S, 256);
    if (grid > need) grid = (int)(need > 0 ? need : 1);
    kern<<<grid, 256, 0, st>>>(A.rows, (const I *)A.row_ptrs, (const I *)A.col_idxs,
                               (const V *)A.values, b, ldb, epi);
    return cudaGetLastError();
}

template <class V, class I, class Epi>
cudaError_t launch_epilogue_pass(int64_t rows, const V *x, int64_t ldx, const Epi &epi,
                                 cudaStream_t st) {
    auto kern = epilogue_pass_kernel<V, Epi>;
    int grid = persistent_grid(kern, 256, 0);
    const int64_t need = ceil_div(rows, 256);
    if (grid > need) grid = (int)(need > 0 ? need : 1);
    kern<<<grid, 256, 0, st>>>(rows, x, ldx, epi);
    return cudaGetLastError();
}

// x written by a row-splitting kernel: carry fix-up then (for fused epilogues) a pass
template <class V>
cudaError_t launch_fixup(int64_t num_tiles, const int64_t *carry_rows, const double *carry_vals,
                         V *x, int64_t ldx, cudaStream_t st) {
    if (num_tiles <= 0) return cudaSuccess;
    carry_fixup_kernel<V><<<(int)ceil_div(num_tiles, 256), 256, 0, st>>>(num_tiles, carry_rows,
                                                                          carry_vals, x, ldx);
    return cudaGetLastError();
}

template <class V, class I>
cudaError_t launch_csr_merge(const sb_csr &A, const V *b, int64_t ldb, V *x, int64_t ldx,
                             cudaStream_t st) {
    const sb_csr_plan &P = *A.plan;
    auto kern = csr_merge_kernel<V, I, kMergeNT, kMergeIPT>;
    int grid = persistent_grid(kern, kMergeNT, 0);
    if (grid > P.num_tiles) grid = (int)P.num_tiles;
    if (grid < 1) return cudaSuccess;
    kern<<<grid, kMergeNT, 0, st>>>(A.rows, (const I *)A.row_ptrs, (const I *)A.col_idxs,
                                    (const V *)A.values, b, ldb, x, ldx,
                                    (const int64_t *)P.tile_rows, (const int64_t *)P.tile_nnz,
                                    P.num_tiles, (int64_t *)P.carry_rows, (double *)P.carry_vals);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_fixup<V>(P.num_tiles, (const int64_t *)P.carry_rows,
                           (const double *)P.carry_vals, x, ldx, st);
}

template <class V, class I, int NT, int C, int RCAP, bool DIRECT = false, int PF = 0>
cudaError_t launch_csr_tile_t(const sb_csr &A, const V *b, int64_t ldb, V *x, int64_t ldx, cudaStream_t st) {
    const sb_csr_plan &P = *A.plan;
    const int64_t ntiles = P.num_tiles / 2;
    constexpr size_t smem = TileLayout<V, I, C, RCAP, DIRECT>::SMEM;
    // unit-stride gathers: fp64 369 us either way on config #3, fp32 333 -> 358 us (the
    // 32-register fp32 kernel schedules worse), so fp64 only
    auto kern = ldb == 1 && sizeof(V) == 8 ? csr_tile_kernel<V, I, NT, C, RCAP, DIRECT, PF, true>
                                           : csr_tile_kernel<V, I, NT, C, RCAP, DIRECT, PF, false>;
    ensure_max_smem((const void *)kern);
    int grid = persistent_grid(kern, NT, smem);
    if (grid > ntiles) grid = (int)ntiles;
    if (grid < 1) return cudaSuccess;
    kern<<<grid, NT, smem, st>>>(A.rows, A.nnz, (const I *)A.row_ptrs, (const I *)A.col_idxs,
                                 (const V *)A.values, b, ldb, x, ldx, (const int64_t *)P.tile_rows, ntiles,
                                 (int64_t *)P.carry_rows, (double *)P.carry_vals);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    tile_carry_fixup_kernel<V><<<(int)ceil_div(P.num_tiles, 256), 256, 0, st>>>(
        P.num_tiles, (const int64_t *)P.carry_rows, (const double *)P.carry_vals, x, ldx);
    return cudaGetLastError();
}

// Tile shape, measured on config #3 (tools/tile_ab.py, us per SpMV fp64 / fp32; merge-path
// 562 / 452): 256 threads x 2048 nnz with values and columns read by coalesced streaming
// loads and only the row pointers TMA-staged ("direct": 24 KB of shared memory -> more
// CTAs per SM) 381 / 333 (fp64 370 with the L2 prefetch below); the same shape with values and columns TMA-staged 405 / 384;
// direct 128 x 2048 851 / 451, 256 x 1024 452 / 442, 256 x 4096 847 / 821; staged 512 x
// 2048 435 / 384; a three-stage staged ring 497 (fp64).  SPARSEB200_TILE_C = 1024 / 4096
// selects the staged kernel with that tile size (experiments).
template <class V, class I>
cudaError_t launch_csr_tile(const sb_csr &A, const V *b, int64_t ldb, V *x, int64_t ldx, cudaStream_t st) {
    const int64_t C = A.plan->items_per_tile;
    if (C == 1024) return launch_csr_tile_t<V, I, 256, 1024, 512>(A, b, ldb, x, ldx, st);
    if (C == 4096) return launch_csr_tile_t<V, I, 256, 4096, 2048>(A, b, ldb, x, ldx, st);
    // L2 prefetch of the values / columns one round ahead: fp64 380.6 -> 370.2 us on
    // config #3; fp32 333 -> 339 us (register-capped kernel), so fp64 only.
    // SPARSEB200_TILE_PF = 0 / 1 / 2 overrides (2 rounds ahead: 381.9 / 342.4 us).
    static const int pf_env = [] {
        const char *e = getenv("SPARSEB200_TILE_PF");
        return e ? atoi(e) : -1;
    }();
    const int pf = pf_env >= 0 ? pf_env : (sizeof(V) == 8 ? 1 : 0);
    if (pf == 1) return launch_csr_tile_t<V, I, 256, 2048, 1024, true, 1>(A, b, ldb, x, ldx, st);
    if (pf == 2) return launch_csr_tile_t<V, I, 256, 2048, 1024, true, 2>(A, b, ldb, x, ldx, st);
    return launch_csr_tile_t<V, I, 256, 2048, 1024, true>(A, b, ldb, x, ldx, st);
}

template <class V>
__global__ void fill_kernel(int64_t rows, int64_t cols, V *x, int64_t ldx, V v) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols;
         t += (int64_t)gridDim.x * blockDim.x)
        x[(t / cols) * ldx + t % cols] = v;
}

template <class V>
cudaError_t launch_fill(int64_t rows, int64_t cols, V *x, int64_t ldx, V v, cudaStream_t st) {
    if (rows * cols == 0) return cudaSuccess;
    fill_kernel<V><<<elem_grid(rows * cols), kElemThreads, 0, st>>>(rows, cols, x, ldx, v);
    return cudaGetLastError();
}

// x_out: where the raw SpMV result goes when the epilogue is not a plain store (the
// solvers always pass their output vector here as well).
template <class V, class I, class Epi>
cudaError_t csr_apply(const sb_csr &A, const V *b, int64_t ldb, V *x_out, int64_t ldx,
                      const Epi &epi, cudaStream_t st) {
    const sb_csr_plan *P = A.plan;
    int kernel = P ? P->kernel : SB_CSR_STRICT;
    if (A.rows == 0) return cudaSuccess;
    if (kernel == SB_CSR_STREAM) {
        // plain SpMV: 128-row blocks (0.95 of the copy peak, tools/tune_stream.py); fused
        // solver epilogues keep 256-row blocks (fewer, longer blocks hide the epilogue's own
        // loads; measured best for the CG iteration, tools/cg_ab.py).  A 256-row block holds
        // at most twice the nnz of a 128-row block.
        if (!is_plain_store<Epi>::value && P->block_rows == 128 && P->nnz_cap256 > 0) {
            sb_csr_plan P2 = *P;
            P2.nnz_cap = P->nnz_cap256;
            sb_csr A2 = A;
            A2.plan = &P2;
            return launch_csr_stream<V, I, 256>(A2, b, ldb, epi, st);
        }
        if (P->block_rows == 256) return launch_csr_stream<V, I, 256>(A, b, ldb, epi, st);
        if (P->block_rows == 128) return launch_csr_stream<V, I, 128>(A, b, ldb, epi, st);
        return launch_csr_stream<V, I, 64>(A, b, ldb, epi, st);
    }
    if (kernel == SB_CSR_VECTOR) {
        switch (P->block_rows) {
        case 2: return launch_csr_vector<V, I, 2>(A, b, ldb, epi, st);
        case 4: return launch_csr_vector<V, I, 4>(A, b, ldb, epi, st);
        case 8: return launch_csr_vector<V, I, 8>(A, b, ldb, epi, st);
        case 16: return launch_csr_vector<V, I, 16>(A, b, ldb, epi, st);
        default: return launch_csr_vector<V, I, 32>(A, b, ldb, epi, st);
        }
    }
    if (kernel == SB_CSR_MERGE || kernel == SB_CSR_TILE) {
        if constexpr (epi_has_gather<Epi>::value) return cudaErrorNotSupported;
        cudaError_t e = kernel == SB_CSR_MERGE ? launch_csr_merge<V, I>(A, b, ldb, x_out, ldx, st)
                        : A.nnz == 0            ? launch_fill<V>(A.rows, 1, x_out, ldx, (V)0, st)
                                                : launch_csr_tile<V, I>(A, b, ldb, x_out, ldx, st);
        if (e != cudaSuccess || is_plain_store<Epi>::value) return e;
        return launch_epilogue_pass<V, I>(A.rows, x_out, ldx, epi, st);
    }
    auto kern = csr_strict_kernel<V, I, Epi>;
    int grid = persistent_grid(kern, 256, 0);
    const int64_t need = ceil_div(A.rows, 256);
    if (grid > need) grid = (int)need;
    kern<<<grid, 256, 0, st>>>(A.rows, (const I *)A.row_ptrs, (const I *)A.col_idxs,
                               (const V *)A.values, b, ldb, epi);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- COO
constexpr int kCooK = 4;                      // entries per lane per warp step
constexpr int64_t kCooChunk = 32 * kCooK * 8;  // entries per warp chunk (carry granularity)

template <class V, class I>
cudaError_t coo_raw(const sb_coo &A, const V *b, int64_t ldb, V *x, int64_t ldx, bool accumulate,
                    cudaStream_t st) {
    if (A.rows == 0) return cudaSuccess;
    if (A.nnz == 0) return accumulate ? cudaSuccess : launch_fill<V>(A.rows, 1, x, ldx, (V)0, st);
    const sb_coo_plan &P = *A.plan;
    const int64_t nchunks = ceil_div(A.nnz, kCooChunk);
    if (nchunks > P.num_tiles) return cudaErrorInvalidValue;  // carry buffers too small
    auto kern = coo_warp_kernel<V, I, kCooK>;
    int grid = persistent_grid(kern, 256, 0);
    const int64_t need = ceil_div(nchunks * 32, 256);
    if (grid > need) grid = (int)need;
    kern<<<grid, 256, 0, st>>>(A.rows, A.nnz, (const I *)A.row_idxs, (const I *)A.col_idxs,
                               (const V *)A.values, b, ldb, x, ldx, kCooChunk, nchunks,
                               (int64_t *)P.carry_rows, (double *)P.carry_vals, accumulate);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_fixup<V>(nchunks, (const int64_t *)P.carry_rows, (const double *)P.carry_vals,
                           x, ldx, st);
}

template <class V, class I, class Epi>
cudaError_t coo_apply(const sb_coo &A, const V *b, int64_t ldb, V *x_out, int64_t ldx,
                      const Epi &epi, cudaStream_t st) {
    if (A.plan && A.plan->row_ptrs && A.plan->csr_plan) {
        // sorted COO rows == CSR rows: run the CSR kernels on the row-pointer index
        // (bitwise what spmv_coo computes: each row-run summed in stored order)
        const sb_csr C{A.rows, A.cols, A.nnz, A.plan->row_ptrs, A.col_idxs, A.values, A.plan->csr_plan};
        return csr_apply<V, I>(C, b, ldb, x_out, ldx, epi, st);
    }
    if constexpr (epi_has_gather<Epi>::value) return cudaErrorNotSupported;
    cudaError_t e = coo_raw<V, I>(A, b, ldb, x_out, ldx, false, st);
    if (e != cudaSuccess || is_plain_store<Epi>::value) return e;
    return launch_epilogue_pass<V, I>(A.rows, x_out, ldx, epi, st);
}

// ---------------------------------------------------------------- ELL / SELL-P / Hybrid
template <class V, class I>
constexpr int rows_per_thread() {
    return 16 / sizeof(V);  // one 16-byte value vector per thread per column
}

template <class V, class I, class Epi, int RPT>
cudaError_t ell_apply_rpt(const sb_ell &A, const V *b, int64_t ldb, const Epi &epi, cudaStream_t st) {
    const bool vec_ok = (A.stride % RPT == 0) && ((uintptr_t)A.values % 16 == 0) &&
                        ((uintptr_t)A.col_idxs % (RPT * sizeof(I) >= 16 ? 16 : RPT * sizeof(I)) == 0);
    if (vec_ok) {
        auto kern = ldb == 1 ? ell_kernel<V, I, RPT, Epi, true> : ell_kernel<V, I, RPT, Epi, false>;
        int grid = persistent_grid(kern, 256, 0);
        const int64_t need = ceil_div(ceil_div(A.rows, RPT), 256);
        if (grid > need) grid = (int)need;
        kern<<<grid, 256, 0, st>>>(A.rows, A.width, A.stride, (const I *)A.col_idxs,
                                   (const V *)A.values, b, ldb, epi);
    } else {
        auto kern = ldb == 1 ? ell_kernel<V, I, 1, Epi, true> : ell_kernel<V, I, 1, Epi, false>;
        int grid = persistent_grid(kern, 256, 0);
        const int64_t need = ceil_div(A.rows, 256);
        if (grid > need) grid = (int)need;
        kern<<<grid, 256, 0, st>>>(A.rows, A.width, A.stride, (const I *)A.col_idxs,
                                   (const V *)A.values, b, ldb, epi);
    }
    return cudaGetLastError();
}

template <class V, class I, class Epi>
cudaError_t ell_apply(const sb_ell &A, const V *b, int64_t ldb, const Epi &epi, cudaStream_t st) {
    if (A.rows == 0) return cudaSuccess;
    if constexpr (sizeof(V) == 4) {
        // fp32: two rows per thread (8-byte value / index vectors) and the four-column tail
        // step: 128^3 ELL 29.5 -> 23.8 us (0.86), Hybrid 28.1 -> 23.5; SPARSEB200_ELL_RPT32=4
        // restores four rows per thread
        static const int r32 = getenv("SPARSEB200_ELL_RPT32") ? atoi(getenv("SPARSEB200_ELL_RPT32")) : 2;
        if (r32 == 2) return ell_apply_rpt<V, I, Epi, 2>(A, b, ldb, epi, st);
    }
    return ell_apply_rpt<V, I, Epi, rows_per_thread<V, I>()>(A, b, ldb, epi, st);
}

template <class V, class I, int S, class Epi>
cudaError_t launch_sellp_stream(const sb_sellp &A, const V *b, int64_t ldb, const Epi &epi,
                                cudaStream_t st) {
    constexpr int VV = 16 / sizeof(V), VI = 16 / sizeof(I);
    // stage capacity: the largest block if it fits 2048 entries, else chunks of 2048
    // entries (whole columns) streamed through the ring
    const int cap = (int)std::min<int64_t>(A.max_block_entries, std::max<int64_t>(2048 / S * S, S));
    const size_t cap_v = (size_t)cap + 2 * VV, cap_c = (size_t)cap + 2 * VI;
    const size_t off_c = (cap_v * sizeof(V) + 15) & ~size_t(15);
    const size_t stage = (off_c + cap_c * sizeof(I) + 15) & ~size_t(15);
    // whole slice blocks when the largest fits a 2048-entry stage, else column chunks
    auto kern = A.max_block_entries <= cap
                    ? (ldb == 1 ? sellp_block_kernel<V, I, S, Epi, true> : sellp_block_kernel<V, I, S, Epi, false>)
                    : (ldb == 1 ? sellp_chunk_kernel<V, I, S, Epi, true> : sellp_chunk_kernel<V, I, S, Epi, false>);
    ensure_max_smem((const void *)kern);
    int grid = persistent_grid(kern, 128, 2 * stage);
    const int64_t nblk = ceil_div(A.num_slices, 128 / S);
    if (grid > nblk) grid = (int)nblk;
    kern<<<grid, 128, 2 * stage, st>>>(A.rows, A.num_slices, (const I *)A.slice_lengths,
                                       (const I *)A.slice_sets, (const I *)A.col_idxs,
                                       (const V *)A.values, b, ldb, cap, epi, (const I *)A.row_perm);
    return cudaGetLastError();
}

// split-piece SELL-P (the plan's blocks cut into pieces; raw row sums into x_out)
template <class V, class I, int S>
cudaError_t launch_sellp_pieces(const sb_sellp &A, const V *b, int64_t ldb, V *x_out, int64_t ldx, cudaStream_t st) {
    constexpr int VV = 16 / sizeof(V), VI = 16 / sizeof(I);
    const int cap = (int)std::min<int64_t>(A.max_block_entries, std::max<int64_t>(2048 / S * S, S));
    const size_t cap_v = (size_t)cap + 2 * VV, cap_c = (size_t)cap + 2 * VI;
    const size_t off_c = (cap_v * sizeof(V) + 15) & ~size_t(15);
    const size_t stage = (off_c + cap_c * sizeof(I) + 15) & ~size_t(15);
    if (A.piece_entries <= 0 || A.piece_entries % (cap / S * S) != 0) return cudaErrorInvalidValue;
    auto kern = ldb == 1 ? sellp_piece_kernel<V, I, S, true> : sellp_piece_kernel<V, I, S, false>;
    ensure_max_smem((const void *)kern);
    int grid = persistent_grid(kern, 128, 2 * stage);
    if (grid > A.num_pieces) grid = (int)A.num_pieces;
    kern<<<grid, 128, 2 * stage, st>>>(A.rows, A.num_slices, (const I *)A.slice_lengths, (const I *)A.slice_sets,
                                       (const I *)A.col_idxs, (const V *)A.values, b, ldb, cap,
                                       (const int64_t *)A.piece_plan, A.num_pieces, A.piece_entries,
                                       (double *)A.carry, x_out, ldx, (const I *)A.row_perm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || A.num_split == 0) return e;
    const int fg = (int)std::min<int64_t>(A.num_split, 148 * 16);
    sellp_piece_fixup_kernel<V, I, S><<<fg, 128, 0, st>>>(A.rows, A.num_slices, (const int64_t *)A.piece_plan,
                                                          A.num_pieces, A.num_split, (const double *)A.carry,
                                                          x_out, ldx, (const I *)A.row_perm);
    return cudaGetLastError();
}

inline bool sellp_split(const sb_sellp &A) {
    return A.piece_plan && A.carry && A.num_pieces > 0 && A.max_block_entries > 0 &&
           (A.slice_size == 32 || A.slice_size == 64 || A.slice_size == 128);
}

template <class V, class I, class Epi>
cudaError_t sellp_apply(const sb_sellp &A, const V *b, int64_t ldb, V *x_out, int64_t ldx, const Epi &epi,
                        cudaStream_t st) {
    if (A.rows == 0) return cudaSuccess;
    if (sellp_split(A) && ((uintptr_t)A.values % 16 == 0) && ((uintptr_t)A.col_idxs % 16 == 0)) {
        // row-splitting: raw sums first, the epilogue (if any) as a pass over x
        if constexpr (epi_has_gather<Epi>::value) return cudaErrorNotSupported;
        cudaError_t e = A.slice_size == 64   ? launch_sellp_pieces<V, I, 64>(A, b, ldb, x_out, ldx, st)
                        : A.slice_size == 32 ? launch_sellp_pieces<V, I, 32>(A, b, ldb, x_out, ldx, st)
                                             : launch_sellp_pieces<V, I, 128>(A, b, ldb, x_out, ldx, st);
        if (e != cudaSuccess || is_plain_store<Epi>::value) return e;
        return launch_epilogue_pass<V, I>(A.rows, x_out, ldx, epi, st);
    }
    const bool staged = A.max_block_entries > 0 &&
                        ((uintptr_t)A.values % 16 == 0) && ((uintptr_t)A.col_idxs % 16 == 0) &&
                        (A.slice_size == 32 || A.slice_size == 64 || A.slice_size == 128);
    if (staged) {
        if (A.slice_size == 64) return launch_sellp_stream<V, I, 64>(A, b, ldb, epi, st);
        if (A.slice_size == 32) return launch_sellp_stream<V, I, 32>(A, b, ldb, epi, st);
        return launch_sellp_stream<V, I, 128>(A, b, ldb, epi, st);
    }
    constexpr int RPT = rows_per_thread<V, I>();
    const bool vec_ok = (A.slice_size % RPT == 0) && ((uintptr_t)A.values % 16 == 0) &&
                        ((uintptr_t)A.col_idxs % (RPT * sizeof(I) >= 16 ? 16 : RPT * sizeof(I)) == 0);
    const int64_t slots = A.num_slices * A.slice_size;
    if (vec_ok) {
        auto kern = ldb == 1 ? sellp_kernel<V, I, RPT, Epi, true> : sellp_kernel<V, I, RPT, Epi, false>;
        int grid = persistent_grid(kern, 256, 0);
        const int64_t need = ceil_div(slots / RPT, 256);
        if (grid > need) grid = (int)(need > 0 ? need : 1);
        kern<<<grid, 256, 0, st>>>(A.rows, A.slice_size, (const I *)A.slice_lengths,
                                   (const I *)A.slice_sets, (const I *)A.col_idxs,
                                   (const V *)A.values, b, ldb, epi, (const I *)A.row_perm);
    } else {
        auto kern = ldb == 1 ? sellp_kernel<V, I, 1, Epi, true> : sellp_kernel<V, I, 1, Epi, false>;
        int grid = persistent_grid(kern, 256, 0);
        const int64_t need = ceil_div(slots, 256);
        if (grid > need) grid = (int)(need > 0 ? need : 1);
        kern<<<grid, 256, 0, st>>>(A.rows, A.slice_size, (const I *)A.slice_lengths,
                                   (const I *)A.slice_sets, (const I *)A.col_idxs,
                                   (const V *)A.values, b, ldb, epi, (const I *)A.row_perm);
    }
    return cudaGetLastError();
}

template <class V, class I, class Epi>
cudaError_t hybrid_apply(const sb_hybrid &A, const V *b, int64_t ldb, V *x_out, int64_t ldx,
                         const Epi &epi, cudaStream_t st) {
    if constexpr (epi_has_gather<Epi>::value) return cudaErrorNotSupported;
    cudaError_t e = ell_apply<V, I>(A.ell, b, ldb, EpiStore<V>{x_out, ldx}, st);
    if (e != cudaSuccess) return e;
    if (A.coo.nnz > 0) {
        e = coo_raw<V, I>(A.coo, b, ldb, x_out, ldx, true, st);
        if (e != cudaSuccess) return e;
    }
    if (is_plain_store<Epi>::value) return cudaSuccess;
    return launch_epilogue_pass<V, I>(A.ell.rows, x_out, ldx, epi, st);
}

// ---------------------------------------------------------------- any format
template <class V, class I, class Epi>
cudaError_t matrix_apply(const sb_matrix &M, const V *b, int64_t ldb, V *x_out, int64_t ldx,
                         const Epi &epi, cudaStream_t st) {
    switch (M.format) {
    case SB_FMT_CSR: return csr_apply<V, I>(*(const sb_csr *)M.mat, b, ldb, x_out, ldx, epi, st);
    case SB_FMT_COO: return coo_apply<V, I>(*(const sb_coo *)M.mat, b, ldb, x_out, ldx, epi, st);
    case SB_FMT_ELL: return ell_apply<V, I>(*(const sb_ell *)M.mat, b, ldb, epi, st);
    case SB_FMT_SELLP: return sellp_apply<V, I>(*(const sb_sellp *)M.mat, b, ldb, x_out, ldx, epi, st);
    case SB_FMT_HYBRID:
        return hybrid_apply<V, I>(*(const sb_hybrid *)M.mat, b, ldb, x_out, ldx, epi, st);
    default: return cudaErrorInvalidValue;
    }
}

// Formats / kernels whose SpMV owns whole rows and so can evaluate a gathered operand
// on the fly (epilogue gather hook): CSR strict / stream / vector, ELL, SELL-P.
inline bool matrix_row_owning(const sb_matrix &M) {
    switch (M.format) {
    case SB_FMT_CSR: {
        const sb_csr &A = *(const sb_csr *)M.mat;
        return !A.plan || (A.plan->kernel != SB_CSR_MERGE && A.plan->kernel != SB_CSR_TILE);
    }
    case SB_FMT_COO: {  // row-pointer-indexed COO runs the CSR kernels
        const sb_coo &A = *(const sb_coo *)M.mat;
        return A.plan && A.plan->row_ptrs && A.plan->csr_plan &&
               A.plan->csr_plan->kernel != SB_CSR_MERGE && A.plan->csr_plan->kernel != SB_CSR_TILE;
    }
    case SB_FMT_ELL: return true;
    case SB_FMT_SELLP: return !sellp_split(*(const sb_sellp *)M.mat);
    default: return false;
    }
}

inline int64_t matrix_rows(const sb_matrix &M) {
    switch (M.format) {
    case SB_FMT_CSR: return ((const sb_csr *)M.mat)->rows;
    case SB_FMT_COO: return ((const sb_coo *)M.mat)->rows;
    case SB_FMT_ELL: return ((const sb_ell *)M.mat)->rows;
    case SB_FMT_SELLP: return ((const sb_sellp *)M.mat)->rows;
    case SB_FMT_HYBRID: return ((const sb_hybrid *)M.mat)->ell.rows;
    default: return -1;
    }
}
inline int64_t matrix_cols(const sb_matrix &M) {
    switch (M.format) {
    case SB_FMT_CSR: return ((const sb_csr *)M.mat)->cols;
    case SB_FMT_COO: return ((const sb_coo *)M.mat)->cols;
    case SB_FMT_ELL: return ((const sb_ell *)M.mat)->cols;
    case SB_FMT_SELLP: return ((const sb_sellp *)M.mat)->cols;
    case SB_FMT_HYBRID: return ((const sb_hybrid *)M.mat)->ell.cols;
    default: return -1;
    }
}

}  // namespace sb
