/*
 * sparseb200.h -- C ABI of libsparseb200.so, the B200-native (sm_100a) SpMV + Krylov library.
 *
 * Drop-in boundary for the reference's typed binding layer.  The reference exposes one
 * callable per (operation x value type [x index type]) with a type suffix
 * (pkg/frontend/src/pysparseops/bindings.py:27-40, built at :81-145, registered at
 * :148-159) and routes to them by runtime dtype (dispatch.py:44-66).  This header
 * exports the same instantiation scheme as plain C symbols:
 *
 *     sb_<op>_<value>[_<index>]     value in {float, double}, index in {i32, i64}
 *
 * e.g. sb_csr_spmv_double_i32 replaces bindings.csr_spmv_double_i32
 * (bindings.py:116-119 -> sparseops.linop.spmv_csr, linop.py:102-121).  Every entry
 * point replaces the reference function cited beside it; INTEGRATION.md shows the
 * ctypes binding a maintainer adds on the reference side.
 *
 * Conventions
 *   - Memory: every pointer in a struct below is DEVICE memory owned by the caller
 *     (the Python frontend allocates it with torch); the library never allocates
 *     device memory.  Host-side structs are passed by pointer and only read during the
 *     call.  Workspace sizes are queried with sb_*_workspace_bytes.
 *   - Streams: all work is enqueued on the caller's `stream` (a cudaStream_t; 0 = the
 *     legacy default stream).  SpMV / BLAS-1 updates return without synchronising;
 *     calls that must return a host value (dot, norm2, solvers, row stats) synchronise
 *     the stream before returning.
 *   - Errors: every call returns an sb_status whose codes map 1:1 onto the reference's
 *     exception kinds (sparseops/errors.py:8-131); `err` (nullable) receives the code,
 *     the failing row / iteration and a message.
 *   - Numerics: fp64 accumulation, fp32 products rounded before the add, no FMA,
 *     deterministic reductions (see paper_2510_08230_b200/csrc/common.cuh).
 */
#ifndef SPARSEB200_H
#define SPARSEB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* exported even when the library is compiled with -fvisibility=hidden */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef void *sb_stream_t; /* cudaStream_t */

/* status codes <-> reference exception kinds (sparseops/errors.py) */
typedef enum {
    SB_OK = 0,
    SB_ERR_INVALID_ARGUMENT = 1,   /* InvalidArgumentError      "invalid-argument"   errors.py:14 */
    SB_ERR_DIMENSION_MISMATCH = 2, /* DimensionMismatchError    "dimension-mismatch" errors.py:31 */
    SB_ERR_PRECISION_MISMATCH = 3, /* PrecisionMismatchError    "precision-mismatch" errors.py:35 */
    SB_ERR_UNSUPPORTED = 4,        /* UnsupportedFeatureError   "unsupported-feature" errors.py:27 */
    SB_ERR_INDEX_BOUNDS = 5,       /* IndexBoundsError (row = offending triplet)     errors.py:39 */
    SB_ERR_BREAKDOWN = 6,          /* BreakdownError (iteration)                     errors.py:85-93 */
    SB_ERR_NUMERIC_FAILURE = 7,    /* NumericFailureError                            errors.py:96 */
    SB_ERR_SINGULAR_DIAGONAL = 8,  /* SingularDiagonalError (row)                    errors.py:115-121 */
    SB_ERR_CUDA = 9,               /* CUDA runtime failure (no reference analogue) */
    SB_ERR_NCCL = 10,              /* NCCL failure (multi-GPU only) */
    SB_ERR_ZERO_PIVOT = 11,        /* ZeroPivotError (row)        precond.py:155-187 */
    SB_ERR_INDEFINITE_PIVOT = 12,  /* IndefinitePivotError (row)  precond.py:205-256 */
    SB_ERR_NOT_TRIANGULAR = 13,    /* NotTriangularError (row)    linop.py:169-198 */
    SB_ERR_SINGULAR_TRIANGLE = 14  /* SingularTriangleError (row) linop.py:169-198 */
} sb_status;

typedef struct {
    int32_t code;
    int32_t pad;
    int64_t row;       /* SingularDiagonalError.row / IndexBoundsError triplet */
    int64_t iteration; /* BreakdownError.iteration */
    char msg[256];
} sb_error;

/* core.DenseMatrix (core.py:226-301): row-major, element (i, j) at data[i*stride + j]. */
typedef struct {
    void *data;
    int64_t rows, cols, stride;
} sb_dense;

/* ------------------------------------------------------------------ sparse formats */
/* CSR SpMV kernel selection (filled by sb_csr_plan_select from row statistics). */
enum {
    SB_CSR_AUTO = 0,
    SB_CSR_STRICT = 1, /* thread per row, global loads: the reference loop on the device */
    SB_CSR_STREAM = 2, /* TMA-staged row blocks, thread per row (regular rows; bit-exact) */
    SB_CSR_VECTOR = 3, /* sub-warp per row (long regular rows) */
    SB_CSR_MERGE = 4,  /* load-balanced merge-path (irregular rows) */
    SB_CSR_TILE = 5    /* fixed nnz tiles, TMA-staged, parallel gathers, per-row segment
                          sums + deterministic carry records (irregular rows) */
};

typedef struct {
    int64_t rows, nnz, min_len, max_len, empty_rows;
    double mean_len, std_len;
    int64_t max_block_nnz[4]; /* max nnz over aligned blocks of 32, 64, 128, 256 rows */
} sb_row_stats;

typedef struct {
    int32_t kernel;         /* SB_CSR_* */
    int32_t block_rows;     /* stream: rows per block R; vector: lanes per row */
    int32_t nnz_cap;        /* stream: max nnz of one R-row block */
    int32_t nnz_cap256;     /* stream: max nnz of one 256-row block (solver epilogues) */
    int64_t num_tiles;      /* merge: tiles of items_per_tile merge items;
                               tile: 2 x ceil(nnz / items_per_tile) carry records
                               (tile_rows = first row of every tile, tile_nnz unused) */
    int64_t items_per_tile;
    void *tile_rows;        /* merge: int64[num_tiles + 1] */
    void *tile_nnz;         /* merge: int64[num_tiles + 1] */
    void *carry_rows;       /* merge: int64[num_tiles] */
    void *carry_vals;       /* merge: double[num_tiles] */
} sb_csr_plan;

/* formats.CsrMatrix (formats.py:84-128) */
typedef struct {
    int64_t rows, cols, nnz;
    const void *row_ptrs, *col_idxs, *values;
    const sb_csr_plan *plan;
} sb_csr;

typedef struct {
    int64_t num_tiles; /* ceil(nnz / sb_coo_tile_entries()) */
    void *carry_rows;  /* int64[num_tiles] */
    void *carry_vals;  /* double[num_tiles] */
    /* optional row-pointer index of the sorted row array (rows + 1, index width) and a
       CSR plan over it: set -> the SpMV runs the CSR kernels on (row_ptrs, col_idxs,
       values) and never re-reads row_idxs; NULL -> segmented-reduction warp kernel */
    const void *row_ptrs;
    const sb_csr_plan *csr_plan;
} sb_coo_plan;

/* formats.CooMatrix (formats.py:57-81): canonical (sorted, unique) entries */
typedef struct {
    int64_t rows, cols, nnz;
    const void *row_idxs, *col_idxs, *values;
    const sb_coo_plan *plan;
} sb_coo;

/* ELL(width, stride): entry k of row i at k*stride + i; padding col = -1, val = 0.
 * (absent from the reference; layout pinned in SURVEY.md §8) */
typedef struct {
    int64_t rows, cols, width, stride;
    const void *col_idxs, *values;
} sb_ell;

/* SELL-P(slice_size): entry k of row i (slice s = i / S) at (slice_sets[s] + k)*S + i%S.
 * max_block_entries: max stored entries of any 128/S consecutive slices (aligned), for the
 * TMA-staged kernel (0 = use the direct kernel).
 * row_perm (SELL-C-sigma, optional): stored row i holds matrix row row_perm[i] (rows sorted
 * by length inside windows of sigma rows); NULL = identity (plain SELL-P). */
typedef struct {
    int64_t rows, cols, slice_size, num_slices;
    const void *slice_lengths, *slice_sets, *col_idxs, *values;
    int64_t max_block_entries;
    const void *row_perm;
    /* split plan (optional, staged kernel only; NULL = every block is one work item):
     * int64 [first piece of each block (nblk + 1) | block of each piece (num_pieces) |
     * blocks of more than one piece (num_split)], nblk = ceil(num_slices / (128 / S));
     * a piece is at most piece_entries stored entries of its block; carry holds
     * num_pieces x 128 doubles (partial row sums of split blocks, summed in piece order). */
    const void *piece_plan;
    int64_t num_pieces, num_split, piece_entries;
    void *carry;
} sb_sellp;

/* Hybrid(w): the first min(len_i, w) entries of each row in ELL(w), the rest in COO */
typedef struct {
    sb_ell ell;
    sb_coo coo;
} sb_hybrid;

enum { SB_FMT_CSR = 0, SB_FMT_COO = 1, SB_FMT_ELL = 2, SB_FMT_SELLP = 3, SB_FMT_HYBRID = 4 };

/* a LinOp (linop.py:44-73) of any storage format */
typedef struct {
    int32_t format; /* SB_FMT_* */
    int32_t pad;
    const void *mat; /* sb_csr* / sb_coo* / sb_ell* / sb_sellp* / sb_hybrid* */
} sb_matrix;

/* ------------------------------------------------------------------ solvers */
/* solvers.Iteration / ResidualNorm (solvers.py:52-76) reduced to OR semantics:
 * stop when it >= max_iters (min over Iteration entries) or, if has_residual,
 * when ||r|| <= reduction_factor * ||b|| (max over ResidualNorm entries; absolute if
 * ||b|| == 0).  check_criteria, solvers.py:121-135. */
typedef struct {
    int64_t max_iters;
    int32_t has_residual;
    int32_t pad;
    double reduction_factor;
} sb_criteria;

/* solvers.ConvergenceLog (solvers.py:79-87); history is a HOST buffer of history_cap
 * doubles filled with one residual per criteria check. */
typedef struct {
    int64_t iterations;
    int32_t converged;
    int32_t stop_reason; /* 0 "residual", 1 "max_iters" */
    int64_t history_len;
    double *history;
    int64_t history_cap;
} sb_log;

/* library / device */
int sb_version(void);
const char *sb_status_string(int code);
/* CUDA graph + conditional-node solver loop (1, default) or host-polled launches (0) */
void sb_set_graph_mode(int enabled);
/* CG loop shape: 3 (default) = one persistent cooperative kernel per solve for TMA-stream
   CSR matrices up to 24 MB per vector, else 1; 1 = CUDA-graph loop of two kernels per
   iteration, the search direction evaluated inside the SpMV gather (row-owning formats);
   0 = three kernels per iteration (SpMV+dot, update, direction).  Modes 0 and 1 give
   bitwise identical iterates; 3 differs only in the summation order of the dots. */
void sb_set_cg_fused(int mode);
/* Grid barriers per iteration of the persistent CG kernel: 2 (default) = SpMV phase and
   update phase; 1 = single-sync kernel (the update of iteration k-1 re-evaluated at every
   out-of-block gathered column of SpMV k, beta from an exact algebraic expansion of r.z:
   A + 9 V n bytes per iteration; stored vector elements computed with the same rounding
   steps, beta within a few ulps; measured slower on B200, kept opt-in).  Replaces nothing
   in the reference (solvers.py:188-224 is one loop shape). */
void sb_set_cg_sync(int barriers);
/* Persistent CG (two-barrier kernel): 1 (default) = the x update x += alpha p runs inside
   the grid-barrier waits and is flushed before its p buffer is reused (bitwise the same
   x); 0 = x updated in the update phase.  Replaces nothing in the reference
   (solvers.py:200-224 updates x in place each iteration; the element arithmetic is that). */
void sb_set_cg_xw(int on);
/* Loop shape used by this thread's last CG solve: 0 three-kernel graph loop, 1 fused-
   direction graph loop, 3 persistent cooperative kernel (one launch per solve). */
int sb_cg_last_loop(void);
/* Rows per block (= threads per CTA) of this thread's last persistent CG solve (512 or
   256; 0 if the last solve ran a graph loop). */
int sb_cg_last_block_rows(void);

#define SB_VALUE_DECLS(VN)                                                                       \
    /* core.dot / norm2 / axpy / scal / copy_into (core.py:358-401); jacobi apply (precond.py:57-63) */ \
    sb_status sb_dot_##VN(const sb_dense *x, const sb_dense *y, double *out, void *workspace,     \
                          sb_stream_t stream, sb_error *err);                                     \
    sb_status sb_norm2_##VN(const sb_dense *x, double *out, void *workspace, sb_stream_t stream,  \
                            sb_error *err);                                                       \
    sb_status sb_axpy_##VN(double alpha, const sb_dense *x, sb_dense *y, sb_stream_t stream,      \
                           sb_error *err);                                                        \
    sb_status sb_scal_##VN(double alpha, sb_dense *x, sb_stream_t stream, sb_error *err);         \
    sb_status sb_copy_##VN(const sb_dense *src, sb_dense *dst, sb_stream_t stream, sb_error *err); \
    sb_status sb_fill_##VN(sb_dense *x, double value, sb_stream_t stream, sb_error *err);         \
    sb_status sb_jacobi_apply_##VN(const void *inv_diag, const sb_dense *b, sb_dense *x,          \
                                   sb_stream_t stream, sb_error *err);

#define SB_INDEX_DECLS(VN, IN)                                                                    \
    /* SpMV x = A b: linop.spmv_csr / spmv_coo (linop.py:102-159) and the formats the            \
       reference lacks (ELL / SELL-P / Hybrid) */                                    \
    sb_status sb_csr_spmv_##VN##_##IN(const sb_csr *a, const sb_dense *b, sb_dense *x,            \
                                      sb_stream_t stream, sb_error *err);                         \
    sb_status sb_coo_spmv_##VN##_##IN(const sb_coo *a, const sb_dense *b, sb_dense *x,            \
                                      sb_stream_t stream, sb_error *err);                         \
    sb_status sb_ell_spmv_##VN##_##IN(const sb_ell *a, const sb_dense *b, sb_dense *x,            \
                                      sb_stream_t stream, sb_error *err);                         \
    sb_status sb_sellp_spmv_##VN##_##IN(const sb_sellp *a, const sb_dense *b, sb_dense *x,        \
                                        sb_stream_t stream, sb_error *err);                       \
    sb_status sb_hybrid_spmv_##VN##_##IN(const sb_hybrid *a, const sb_dense *b, sb_dense *x,      \
                                         sb_stream_t stream, sb_error *err);                      \
    /* LinOp.apply_advanced x = alpha A b + beta x (linop.py:81-99); tmp: rows x cols workspace */ \
    sb_status sb_apply_advanced_##VN##_##IN(const sb_matrix *a, double alpha, const sb_dense *b,  \
                                            double beta, sb_dense *x, void *tmp,                  \
                                            sb_stream_t stream, sb_error *err);                   \
    /* jacobi_create (precond.py:66-84) incl. CsrMatrix.diagonal (formats.py:113-122) */          \
    sb_status sb_jacobi_create_##VN##_##IN(const sb_csr *a, void *inv_diag, void *workspace,     \
                                           sb_stream_t stream, sb_error *err);                    \
    /* format conversions (formats.py:184-199 + canonical layouts of SURVEY.md §8) */             \
    sb_status sb_ell_from_csr_##VN##_##IN(const sb_csr *a, sb_ell *out, sb_stream_t stream,       \
                                          sb_error *err);                                         \
    sb_status sb_sellp_from_csr_##VN##_##IN(const sb_csr *a, sb_sellp *out, sb_stream_t stream,   \
                                            sb_error *err);                                       \
    sb_status sb_hybrid_from_csr_##VN##_##IN(const sb_csr *a, const void *coo_row_ptrs,           \
                                             sb_hybrid *out, sb_stream_t stream, sb_error *err);  \
    /* coo_from_arrays (formats.py:131-166): canonicalise raw int64 triplets on the device.       \
       Returns the canonical nnz in *nnz_out; out arrays sized for the raw count. */              \
    sb_status sb_coo_from_arrays_##VN##_##IN(int64_t rows, int64_t cols, int64_t count,           \
                                             const int64_t *row_idxs, const int64_t *col_idxs,    \
                                             const void *values, void *out_rows, void *out_cols,  \
                                             void *out_vals, void *workspace,                     \
                                             size_t workspace_bytes, int64_t *nnz_out,            \
                                             sb_stream_t stream, sb_error *err);                  \
    /* solvers: Cg (solvers.py:188-224), Cgs (:231-284), Gmres (:322-399), BiCGSTAB (new) */      \
    sb_status sb_cg_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,                   \
                                      const sb_dense *b, sb_dense *x, const sb_criteria *crit,    \
                                      void *workspace, sb_log *log, sb_stream_t stream,           \
                                      sb_error *err);                                             \
    sb_status sb_cgs_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,                  \
                                       const sb_dense *b, sb_dense *x, const sb_criteria *crit,   \
                                       void *workspace, sb_log *log, sb_stream_t stream,          \
                                       sb_error *err);                                            \
    sb_status sb_bicgstab_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,             \
                                            const sb_dense *b, sb_dense *x,                       \
                                            const sb_criteria *crit, void *workspace,             \
                                            sb_log *log, sb_stream_t stream, sb_error *err);      \
    sb_status sb_gmres_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,                \
                                         const sb_dense *b, sb_dense *x, const sb_criteria *crit, \
                                         int64_t krylov_dim, void *workspace, sb_log *log,        \
                                         sb_stream_t stream, sb_error *err);

SB_VALUE_DECLS(float)
SB_VALUE_DECLS(double)
SB_INDEX_DECLS(float, i32)
SB_INDEX_DECLS(float, i64)
SB_INDEX_DECLS(double, i32)
SB_INDEX_DECLS(double, i64)

/* index-only operations */
#define SB_IDX_DECLS(IN)                                                                          \
    /* row-length statistics (drive the CSR kernel choice); workspace: 256 bytes */              \
    sb_status sb_csr_row_stats_##IN(int64_t rows, const void *row_ptrs, void *workspace,          \
                                    sb_row_stats *out, sb_stream_t stream, sb_error *err);        \
    /* fill plan->tile_* for the merge-path kernel (plan from sb_csr_plan_select) */              \
    sb_status sb_csr_plan_build_##IN(int64_t rows, int64_t nnz, const void *row_ptrs,            \
                                     sb_csr_plan *plan, sb_stream_t stream, sb_error *err);       \
    /* csr_from_coo (formats.py:184-191): row_ptrs from sorted row indices */                     \
    sb_status sb_csr_row_ptrs_from_coo_##IN(int64_t rows, int64_t nnz, const void *row_idxs,      \
                                            void *row_ptrs, sb_stream_t stream, sb_error *err);   \
    /* coo_from_csr (formats.py:194-199): expand row_ptrs into row indices */                     \
    sb_status sb_coo_row_idxs_from_csr_##IN(int64_t rows, int64_t nnz, const void *row_ptrs,      \
                                            void *row_idxs, sb_stream_t stream, sb_error *err);   \
    /* SELL-P slice metadata (slice_lengths, slice_sets) and ELL / Hybrid widths */               \
    sb_status sb_sellp_slices_##IN(int64_t rows, const void *row_ptrs, int64_t slice_size,        \
                                   void *slice_lengths, void *slice_sets, int64_t *total,         \
                                   sb_stream_t stream, sb_error *err);                            \
    /* Hybrid: per-row COO-tail counts as row_ptrs of the tail (length rows+1), total returned */ \
    sb_status sb_hybrid_tail_ptrs_##IN(int64_t rows, const void *row_ptrs, int64_t width,         \
                                       void *tail_ptrs, int64_t *tail_nnz, sb_stream_t stream,    \
                                       sb_error *err);                                            \
    /* synthetic stencil generators straight into canonical CSR: rows          \
       [row_lo, row_hi) (-1 = all) with global columns and row_ptrs relative to row_lo;          \
       dim 2 -> 5-point Poisson, dim 3 -> 7-point with convection c (0 = Poisson) */              \
    sb_status sb_stencil_csr_double_##IN(int64_t p, int32_t dim, double c, int64_t row_lo,       \
                                         int64_t row_hi, void *row_ptrs, void *col_idxs,          \
                                         void *values, sb_stream_t stream, sb_error *err);        \
    sb_status sb_stencil_csr_float_##IN(int64_t p, int32_t dim, double c, int64_t row_lo,        \
                                        int64_t row_hi, void *row_ptrs, void *col_idxs,           \
                                        void *values, sb_stream_t stream, sb_error *err);

SB_IDX_DECLS(i32)
SB_IDX_DECLS(i64)

/* host-side CSR kernel choice from row statistics (force = SB_CSR_* or SB_CSR_AUTO);
 * fills plan->kernel/block_rows/nnz_cap/num_tiles/items_per_tile.  The caller then
 * allocates the tile/carry buffers (when num_tiles > 0) and calls sb_csr_plan_build. */
sb_status sb_csr_plan_select(const sb_row_stats *stats, int32_t value_bytes, int32_t index_bytes,
                             int32_t force, sb_csr_plan *plan, sb_error *err);
/* COO tile size (entries per carry slot) */
int64_t sb_coo_tile_entries(void);
/* workspace sizes (bytes) */
size_t sb_reduce_workspace_bytes(void);
size_t sb_coo_from_arrays_workspace_bytes(int64_t count);
size_t sb_solver_workspace_bytes(int32_t solver, int32_t value_bytes, int64_t n, int64_t krylov_dim,
                                 int64_t history_cap);

/* ------------------------------------------------------------------ row-partitioned solves */
/* One rank's (NCCL) or one partition's (single-GPU loopback) share of a row-partitioned
 * system: local rows with columns renumbered to [own rows | ghosts],
 * ghost blocks ordered by owner, and the halo pattern. */
typedef struct {
    sb_matrix a;                /* n_local x (n_local + n_ghost), all local rows */
    int32_t num_views;          /* 0: SpMV after the halo; else views[0] = interior rows (run */
    int32_t num_neighbors;      /*    while the halo is in flight), views[1..] = the rest    */
    sb_matrix views[3];
    int64_t view_row0[3];       /* first local row of each view */
    int64_t n_local, n_ghost;
    const int32_t *nbr;         /* host: neighbour ranks / partition indices, ascending */
    const int64_t *send_count;  /* host, per neighbour */
    const int64_t *send_lo;     /* host: first local row of a contiguous send block, or -1 */
    const int64_t *send_off;    /* host: offset into send_idx / send_buf */
    const int64_t *recv_count;  /* host */
    const int64_t *recv_off;    /* host: offset inside the ghost region */
    const void *send_idx;       /* device int64 local rows (non-contiguous neighbours) */
    void *send_buf;             /* device value buffer (sum of send counts) */
    const void *inv_diag;       /* device: local Jacobi inverse diagonal, or NULL */
    sb_dense b, x;              /* local rows (contiguous, 16-byte aligned) */
    void *workspace;            /* sb_dist_workspace_bytes */
} sb_dist_part;

/* NCCL (loaded at run time from the process's libnccl.so.2); the unique id is exchanged by
 * the caller (torch.distributed store). */
sb_status sb_nccl_unique_id(char out[128], sb_error *err);
sb_status sb_nccl_comm_init(int32_t nranks, const char id[128], int32_t rank, void **comm,
                            sb_error *err);
sb_status sb_nccl_comm_destroy(void *comm, sb_error *err);
size_t sb_dist_workspace_bytes(int32_t value_bytes, int64_t n_local, int64_t n_ghost,
                               int64_t history_cap);

/* workspace of one partition for solver kind SB_SOLVER_CG / _BICGSTAB / _GMRES
 * (sb_dist_workspace_bytes == the CG size) */
size_t sb_dist_solver_workspace_bytes(int32_t solver, int32_t value_bytes, int64_t n_local,
                                      int64_t n_ghost, int64_t krylov_dim, int64_t history_cap);

/* Row-partitioned Jacobi-preconditioned solvers with the single-GPU solvers' semantics
 * (CG solvers.py:188-224, GMRES(m) :322-399, BiCGSTAB oracle/sbref.cpp): halo exchange of
 * every SpMV input (overlapped with the interior rows), fused local dots combined with
 * ncclAllReduce (comm != NULL, nparts == 1) or summed across `nparts` partitions living
 * on this one GPU (comm == NULL: the loopback transport that tests the decomposition).
 * inv_diag == NULL in a partition = no preconditioner. */
#define SB_DIST_DECLS(VN, IN)                                                                    \
    sb_status sb_dist_cg_solve_##VN##_##IN(sb_dist_part *parts, int32_t nparts, void *comm,       \
                                           const sb_criteria *crit, sb_log *log,                  \
                                           sb_stream_t stream, sb_error *err);                    \
    sb_status sb_dist_bicgstab_solve_##VN##_##IN(sb_dist_part *parts, int32_t nparts, void *comm, \
                                                 const sb_criteria *crit, sb_log *log,            \
                                                 sb_stream_t stream, sb_error *err);              \
    sb_status sb_dist_gmres_solve_##VN##_##IN(sb_dist_part *parts, int32_t nparts, void *comm,    \
                                              const sb_criteria *crit, int64_t krylov_dim,        \
                                              sb_log *log, sb_stream_t stream, sb_error *err);
SB_DIST_DECLS(float, i32)
SB_DIST_DECLS(float, i64)
SB_DIST_DECLS(double, i32)
SB_DIST_DECLS(double, i64)

/* ---------------------------------------------------------------- ILU(0) / IC(0) + SpTRSV
   SURVEY.md 8f f4: precond.py:155-287 (ilu0_factorize, _split_lu, ic0_factorize,
   IluFactors / IcFactor.apply), linop.py:169-198 (solve_lower_tri / solve_upper_tri),
   _kernels.py:91-137.  Sync-free device sweeps (rows claimed in solve order, per-row ready
   flags), bit-exact with the reference loops.  Workspace: sb_tri_workspace_bytes(n). */
size_t sb_tri_workspace_bytes(int64_t n);

/* a two-factor triangular preconditioner x = U^{-1} (L^{-1} b) for the device solvers:
   ILU(0): l = strict lower (unit diagonal implicit, l_unit = 1), u = upper incl. diagonal;
   IC(0):  l = L (l_unit = 0), u = L^T */
typedef struct {
    const sb_csr *l;
    int32_t l_unit;
    int32_t pad;
    const sb_csr *u;
    void *workspace; /* sb_tri_workspace_bytes(rows) */
} sb_tri_precond;

#define SB_TRI_DECLS(VN, IN)                                                                      \
    /* x = T^{-1} b (lower: forward, upper: backward); NotTriangular / SingularTriangle rows */  \
    sb_status sb_csr_trisolve_##VN##_##IN(const sb_csr *t, int32_t lower, int32_t unit_diag,     \
                                          const sb_dense *b, sb_dense *x, void *workspace,       \
                                          sb_stream_t stream, sb_error *err);                    \
    sb_status sb_csr_tri_check_##VN##_##IN(const sb_csr *t, int32_t lower, int32_t unit_diag,    \
                                           void *workspace, sb_stream_t stream, sb_error *err);  \
    /* ILU(0) values on A's pattern (values_out: nnz); diag_workspace: int64[rows] */            \
    sb_status sb_ilu0_##VN##_##IN(const sb_csr *a, void *values_out, void *workspace,            \
                                  void *diag_workspace, sb_stream_t stream, sb_error *err);      \
    /* IC(0) on the lower pattern (lp, lc, la = A's entries with col <= row); scratch:         \
       double[nnz of the lower pattern] */                                                      \
    sb_status sb_ic0_##VN##_##IN(int64_t n, const void *lp, const void *lc, const void *la,      \
                                 void *values_out, void *workspace, void *scratch,               \
                                 sb_stream_t stream, sb_error *err);                             \
    /* _split_lu scatter given the split row pointers (lp, up = row_ptrs - lp) */              \
    sb_status sb_csr_split_scatter_##VN##_##IN(int64_t n, const void *rp, const void *ci,        \
                                               const void *val, const void *lp, const void *up,  \
                                               void *lc, void *lv, void *uc, void *uv,           \
                                               sb_stream_t stream, sb_error *err);               \
    /* CG / GMRES with a triangular-factor preconditioner (ILU / IC) */                         \
    sb_status sb_cg_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,           \
                                          const sb_dense *b, sb_dense *x,                        \
                                          const sb_criteria *crit, void *workspace, sb_log *log, \
                                          sb_stream_t stream, sb_error *err);                    \
    sb_status sb_gmres_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,        \
                                             const sb_dense *b, sb_dense *x,                     \
                                             const sb_criteria *crit, int64_t krylov_dim,        \
                                             void *workspace, sb_log *log, sb_stream_t stream,   \
                                             sb_error *err);                                     \
    /* CGS / BiCGSTAB with ILU / IC: both applications per iteration (solvers.py:261, :273) */ \
    sb_status sb_cgs_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,          \
                                           const sb_dense *b, sb_dense *x,                       \
                                           const sb_criteria *crit, void *workspace,             \
                                           sb_log *log, sb_stream_t stream, sb_error *err);      \
    sb_status sb_bicgstab_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,     \
                                                const sb_dense *b, sb_dense *x,                  \
                                                const sb_criteria *crit, void *workspace,        \
                                                sb_log *log, sb_stream_t stream, sb_error *err);

SB_TRI_DECLS(float, i32)
SB_TRI_DECLS(float, i64)
SB_TRI_DECLS(double, i32)
SB_TRI_DECLS(double, i64)

/* per-row counts of entries with col < row (incl_diag: col <= row), for _split_lu */
sb_status sb_csr_split_count_i32(int64_t n, const void *rp, const void *ci, int32_t incl_diag,
                                 int64_t *counts, sb_stream_t stream, sb_error *err);
sb_status sb_csr_split_count_i64(int64_t n, const void *rp, const void *ci, int32_t incl_diag,
                                 int64_t *counts, sb_stream_t stream, sb_error *err);

/* solver ids for sb_solver_workspace_bytes */
enum { SB_SOLVER_CG = 0, SB_SOLVER_CGS = 1, SB_SOLVER_GMRES = 2, SB_SOLVER_BICGSTAB = 3 };

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* SPARSEB200_H */
