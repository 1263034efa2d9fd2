// dist_cg.cu -- row-partitioned Jacobi-CG across GPUs.
//
// Each rank owns a contiguous block of rows; its local CSR has columns renumbered to
// [own rows | ghost rows] with the ghosts grouped by owner.  Per iteration:
//   halo exchange of p (NCCL grouped send/recv on a side stream, overlapped with the
//   SpMV of the interior rows) -> SpMV of the remaining rows -> ncclAllReduce of the
//   fused p.q partials -> alpha -> fused x/r/z update with r.r, r.z partials ->
//   ncclAllReduce -> criteria / beta -> p = z + beta p.
// The scalar logic is the reference's (solvers.py:200-224) evaluated identically on
// every rank from the reduced dots, so every rank stops at the same iteration.
// comm == NULL selects the loopback transport: `nparts` partitions on this one GPU,
// halos as device copies and dot sums in partition order -- the single-GPU test of the
// decomposition (NCCL rejects two ranks on one device).
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <vector>

#include "solver_common.cuh"

namespace sb {

// ---------------------------------------------------------------- NCCL, loaded at run time
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    bool ok = false;
};

static NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    const char *env = getenv("SPARSEB200_NCCL_LIB");
    void *h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.send = (decltype(api.send))dlsym(h, "ncclSend");
    api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart &&
             api.groupEnd && api.send && api.recv && api.allReduce && api.errorString;
    return api;
}

#define SB_NCCL(call)                                                                       \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return ::sb::fail(err, SB_ERR_NCCL, "%s: %s", #call, nccl().errorString(r_)); \
    } while (0)

template <class V>
constexpr ncclDataType_t nccl_type() {
    return sizeof(V) == 8 ? ncclFloat64 : ncclFloat32;
}

// ---------------------------------------------------------------- kernels
template <int SLOT, int N>
struct StoreTotals {  // last block: local totals -> ctl->dot[SLOT..SLOT+N)
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[N]) const {
        for (int k = 0; k < N; ++k) c->dot[SLOT + k] = tot[k];
    }
};

template <class V>
struct DCopy : SkipNone {  // dst = src (x into the extended vector)
    using value_type = V;
    const V *src;
    V *dst;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        stp<W>(dst, i, ldp<W>(src, i));
    }
};

template <class V>
struct DInit : SkipNone {  // CgInit (cg.cu) with the dots left for the allreduce
    using value_type = V;
    const V *b, *t, *inv;
    V *r, *z, *p;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[3]) const {
        const auto B = ldp<W>(b, i), T = ldp<W>(t, i), D = ldp_or_one<W>(inv, i);
        Pk<V, W> R, Z;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-1.0, T.v[w], B.v[w]);
            Z.v[w] = inv ? vmul(R.v[w], D.v[w]) : R.v[w];
            part[0] = addd(part[0], mulp(B.v[w], B.v[w]));
            part[1] = addd(part[1], mulp(R.v[w], R.v[w]));
            part[2] = addd(part[2], mulp(R.v[w], Z.v[w]));
        }
        stp<W>(r, i, R);
        stp<W>(z, i, Z);
        stp<W>(p, i, Z);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[3]) const {
        StoreTotals<0, 3>{}.last(c, tot);
    }
};

template <class V>
struct DUpdate : SkipNone {  // CgUpdate (cg.cu) with the dots left for the allreduce
    using value_type = V;
    const V *p, *q, *inv;
    V *x, *r, *z;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[2]) const {
        const auto P = ldp<W>(p, i), Q = ldp<W>(q, i), D = ldp_or_one<W>(inv, i);
        auto X = ldp<W>(x, i), R = ldp<W>(r, i);
        Pk<V, W> Z;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            X.v[w] = axpy_e(alpha, P.v[w], X.v[w]);
            R.v[w] = axpy_e(-alpha, Q.v[w], R.v[w]);
            Z.v[w] = inv ? vmul(R.v[w], D.v[w]) : R.v[w];
            part[0] = addd(part[0], mulp(R.v[w], R.v[w]));
            part[1] = addd(part[1], mulp(R.v[w], Z.v[w]));
        }
        stp<W>(x, i, X);
        stp<W>(r, i, R);
        stp<W>(z, i, Z);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[2]) const {
        StoreTotals<6, 2>{}.last(c, tot);
    }
};

template <class V>
struct DDirection : SkipNone {
    using value_type = V;
    const V *z;
    V *p;
    double beta;
    __device__ __forceinline__ void prepare(const Ctl *c) { beta = c->beta; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        const auto Z = ldp<W>(z, i);
        auto P = ldp<W>(p, i);
#pragma unroll
        for (int w = 0; w < W; ++w) P.v[w] = axpy_e(1.0, Z.v[w], scal_e(beta, P.v[w]));
        stp<W>(p, i, P);
    }
};

// scalar steps on the reduced dots (identical on every rank / partition)
struct DInitCheck {
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
    __device__ __forceinline__ void run(Ctl *c) const {
        c->bnorm = sqrt(c->dot[0]);
        c->rnorm = sqrt(c->dot[1]);
        c->iter = 0;
        if (c->rnorm == 0.0) {
            exact_log(c);
            return;
        }
        c->rz = c->dot[2];
    }
};

struct DAlpha {  // solvers.py:202-206
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
    __device__ __forceinline__ void run(Ctl *c) const {
        const int64_t it = c->iter + 1;
        c->iter = it;
        const double pq = addd(addd(c->dot[3], c->dot[4]), c->dot[5]);
        if (!isfinite(pq) || pq <= kBreakdownRtol * fabs(c->rz)) {
            breakdown(c, it);
            return;
        }
        c->alpha = c->rz / pq;
    }
};

struct DCheck {  // solvers.py:207-222
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
    __device__ __forceinline__ void run(Ctl *c) const {
        const int64_t it = c->iter;
        const double rnorm = sqrt(c->dot[6]);
        c->rnorm = rnorm;
        record(c, it, rnorm);
        int reason = check_criteria(c, it, rnorm, c->bnorm);
        if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
        if (reason != STOP_NONE) {
            finish_with(c, it, reason);
            return;
        }
        const double rz_new = c->dot[7];
        if (!isfinite(rz_new) || c->rz == 0.0) {
            breakdown(c, it);
            return;
        }
        c->beta = rz_new / c->rz;
        c->rz = rz_new;
        // the SpMV views write at most slots 3..5 and the allreduce sums in place: clear
        // them so a partition with fewer views never re-adds last iteration's sums
        c->dot[3] = c->dot[4] = c->dot[5] = 0.0;
    }
};

template <class V>
__global__ void pack_kernel(int64_t n, const int64_t *idx, const V *src, V *dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[idx[k]];
}

constexpr int kMaxLoopbackParts = 16;
struct CtlList {
    Ctl *c[kMaxLoopbackParts];
    int n;
};

// loopback "allreduce": sum the partitions' dots in partition order, write to all
__global__ void loopback_sum_kernel(CtlList L, int slot, int count) {
    const int k = threadIdx.x;
    if (k >= count) return;
    double s = 0.0;
    for (int p = 0; p < L.n; ++p) s = addd(s, L.c[p]->dot[slot + k]);
    for (int p = 0; p < L.n; ++p) L.c[p]->dot[slot + k] = s;
}

__global__ void zero_dots_kernel(Ctl *c) {
    if (threadIdx.x < 8) c->dot[threadIdx.x] = 0.0;
}

// ---------------------------------------------------------------- workspace
inline size_t dist_ws_bytes(int vbytes, int64_t nl, int64_t ng, int64_t cap) {
    const size_t v = a256((size_t)vbytes * (size_t)(nl > 0 ? nl : 1));
    const size_t ve = a256((size_t)vbytes * (size_t)(nl + ng > 0 ? nl + ng : 1));
    return kCtlBytes + a256(3 * kMaxGrid * sizeof(double)) +
           a256(sizeof(double) * (size_t)(cap > 0 ? cap : 1)) + 4 * v + ve;
}

template <class V>
struct PartBufs {
    Ctl *ctl;
    double *partials, *hist;
    V *r, *z, *q, *t, *pe;  // pe: extended search direction [own | ghosts]
};

template <class V>
PartBufs<V> carve_dist(void *ws, int64_t nl, int64_t cap) {
    unsigned char *p = (unsigned char *)ws;
    const size_t v = a256(sizeof(V) * (size_t)(nl > 0 ? nl : 1));
    PartBufs<V> b;
    b.ctl = (Ctl *)p;
    p += kCtlBytes;
    b.partials = (double *)p;
    p += a256(3 * kMaxGrid * sizeof(double));
    b.hist = (double *)p;
    p += a256(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
    b.r = (V *)p;
    p += v;
    b.z = (V *)p;
    p += v;
    b.q = (V *)p;
    p += v;
    b.t = (V *)p;
    p += v;
    b.pe = (V *)p;
    return b;
}

// ---------------------------------------------------------------- solve
template <class V, class I>
sb_status dist_cg(sb_dist_part *parts, int np, void *comm_v, const sb_criteria *crit, sb_log *log,
                  cudaStream_t st, sb_error *err) {
    if (!parts || np < 1 || !crit || !log) return fail(err, SB_ERR_INVALID_ARGUMENT, "dist_cg: null argument");
    ncclComm_t comm = (ncclComm_t)comm_v;
    if (comm && np != 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "NCCL mode takes one partition per rank");
    if (!comm && np > kMaxLoopbackParts) return fail(err, SB_ERR_UNSUPPORTED, "loopback: at most 16 partitions");
    if (comm && !nccl().ok) return fail(err, SB_ERR_NCCL, "libnccl.so.2 could not be loaded");
    if (crit->max_iters < 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "max_iters must be positive");
    const int64_t cap = log->history_cap;
    std::vector<PartBufs<V>> B(np);
    CtlList L{};
    L.n = np;
    for (int k = 0; k < np; ++k) {
        const sb_dist_part &P = parts[k];
        if (P.b.cols != 1 || P.x.cols != 1 || P.b.rows != P.n_local || P.x.rows != P.n_local ||
            P.b.stride != 1 || P.x.stride != 1)
            return fail(err, SB_ERR_DIMENSION_MISMATCH, "partition %d: b / x must be n_local x 1 contiguous", k);
        if (((uintptr_t)P.b.data | (uintptr_t)P.x.data | (uintptr_t)P.inv_diag) % 16)
            return fail(err, SB_ERR_UNSUPPORTED, "partition %d: vectors must be 16-byte aligned", k);
        B[k] = carve_dist<V>(P.workspace, P.n_local, cap);
        L.c[k] = B[k].ctl;
        Ctl h;
        std::memset(&h, 0, sizeof(h));
        h.max_iters = crit->max_iters;
        h.has_rf = crit->has_residual;
        h.rf = crit->reduction_factor;
        h.stop_reason = STOP_NONE;
        h.hist = B[k].hist;
        h.hist_cap = cap;
        SB_CUDA(cudaMemcpyAsync(B[k].ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    }

    // halo: ghosts of the extended search direction of every local partition
    cudaStream_t side = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    const bool overlap = comm && parts[0].num_views > 0;
    if (overlap) {
        SB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        SB_CUDA(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
        SB_CUDA(cudaEventCreateWithFlags(&ev_halo, cudaEventDisableTiming));
    }
    auto halo = [&](cudaStream_t s) -> sb_status {
        if (comm) {
            const sb_dist_part &P = parts[0];
            V *pe = B[0].pe;
            for (int j = 0; j < P.num_neighbors; ++j)
                if (P.send_lo[j] < 0 && P.send_count[j] > 0)
                    pack_kernel<V><<<elem_grid(P.send_count[j]), 256, 0, s>>>(
                        P.send_count[j], (const int64_t *)P.send_idx + P.send_off[j], pe,
                        (V *)P.send_buf + P.send_off[j]);
            SB_CUDA(cudaGetLastError());
            SB_NCCL(nccl().groupStart());
            for (int j = 0; j < P.num_neighbors; ++j) {
                const V *src = P.send_lo[j] >= 0 ? pe + P.send_lo[j] : (const V *)P.send_buf + P.send_off[j];
                if (P.send_count[j] > 0)
                    SB_NCCL(nccl().send(src, P.send_count[j], nccl_type<V>(), P.nbr[j], comm, s));
                if (P.recv_count[j] > 0)
                    SB_NCCL(nccl().recv(pe + P.n_local + P.recv_off[j], P.recv_count[j], nccl_type<V>(),
                                        P.nbr[j], comm, s));
            }
            SB_NCCL(nccl().groupEnd());
            return SB_OK;
        }
        for (int k = 0; k < np; ++k) {  // loopback: pack every sender first
            const sb_dist_part &P = parts[k];
            for (int j = 0; j < P.num_neighbors; ++j)
                if (P.send_lo[j] < 0 && P.send_count[j] > 0)
                    pack_kernel<V><<<elem_grid(P.send_count[j]), 256, 0, s>>>(
                        P.send_count[j], (const int64_t *)P.send_idx + P.send_off[j], B[k].pe,
                        (V *)P.send_buf + P.send_off[j]);
        }
        SB_CUDA(cudaGetLastError());
        for (int k = 0; k < np; ++k) {
            const sb_dist_part &P = parts[k];
            for (int j = 0; j < P.num_neighbors; ++j) {
                if (P.recv_count[j] == 0) continue;
                const int src_part = P.nbr[j];
                const sb_dist_part &S = parts[src_part];
                int jj = -1;
                for (int u = 0; u < S.num_neighbors; ++u)
                    if (S.nbr[u] == k) jj = u;
                if (jj < 0 || S.send_count[jj] != P.recv_count[j])
                    return fail(err, SB_ERR_INVALID_ARGUMENT, "loopback halo pattern mismatch (%d <- %d)", k, src_part);
                const V *src = S.send_lo[jj] >= 0 ? B[src_part].pe + S.send_lo[jj]
                                                  : (const V *)S.send_buf + S.send_off[jj];
                SB_CUDA(cudaMemcpyAsync(B[k].pe + P.n_local + P.recv_off[j], src, sizeof(V) * P.recv_count[j],
                                        cudaMemcpyDeviceToDevice, s));
            }
        }
        return SB_OK;
    };
    auto allreduce = [&](int slot, int count, cudaStream_t s) -> sb_status {
        if (comm) {
            SB_NCCL(nccl().allReduce(&B[0].ctl->dot[slot], &B[0].ctl->dot[slot], count, ncclFloat64, ncclSum,
                                     comm, s));
            return SB_OK;
        }
        if (np > 1) {
            loopback_sum_kernel<<<1, 32, 0, s>>>(L, slot, count);
            SB_CUDA(cudaGetLastError());
        }
        return SB_OK;
    };
    // q = A p on every partition; dots p.q into slots 3.. (one per launch)
    auto spmv_pq = [&](cudaStream_t s) -> sb_status {
        for (int k = 0; k < np; ++k) {
            const sb_dist_part &P = parts[k];
            V *pe = B[k].pe, *q = B[k].q;
            if (P.num_views == 0) {
                SB_CUDA((matrix_apply<V, I>(P.a, pe, 1, q, 1,
                                            EpiSolver<V, 1, StoreTotals<3, 1>>{q, pe, nullptr, B[k].ctl, B[k].partials, {}},
                                            s)));
            }
        }
        return SB_OK;
    };
    auto spmv_views = [&](int first, int last, cudaStream_t s) -> sb_status {
        for (int k = 0; k < np; ++k) {
            const sb_dist_part &P = parts[k];
            for (int v = first; v < last && v < P.num_views; ++v) {
                const int64_t r0 = P.view_row0[v];
                V *pe = B[k].pe, *q = B[k].q + r0;
                cudaError_t e;
                if (v == 0)
                    e = matrix_apply<V, I>(P.views[v], pe, 1, q, 1,
                                           EpiSolver<V, 1, StoreTotals<3, 1>>{q, pe + r0, nullptr, B[k].ctl, B[k].partials, {}}, s);
                else if (v == 1)
                    e = matrix_apply<V, I>(P.views[v], pe, 1, q, 1,
                                           EpiSolver<V, 1, StoreTotals<4, 1>>{q, pe + r0, nullptr, B[k].ctl, B[k].partials, {}}, s);
                else
                    e = matrix_apply<V, I>(P.views[v], pe, 1, q, 1,
                                           EpiSolver<V, 1, StoreTotals<5, 1>>{q, pe + r0, nullptr, B[k].ctl, B[k].partials, {}}, s);
                SB_CUDA(e);
            }
        }
        return SB_OK;
    };

    auto iteration = [&](cudaStream_t s) -> sb_status {
        sb_status r;
        bool any_views = false;
        for (int k = 0; k < np; ++k) any_views |= parts[k].num_views > 0;
        if (overlap) {
            SB_CUDA(cudaEventRecord(ev_ready, s));
            SB_CUDA(cudaStreamWaitEvent(side, ev_ready, 0));
            if ((r = halo(side)) != SB_OK) return r;
            SB_CUDA(cudaEventRecord(ev_halo, side));
            if ((r = spmv_views(0, 1, s)) != SB_OK) return r;
            SB_CUDA(cudaStreamWaitEvent(s, ev_halo, 0));
            if ((r = spmv_views(1, 3, s)) != SB_OK) return r;
        } else {
            if ((r = halo(s)) != SB_OK) return r;
            if ((r = spmv_pq(s)) != SB_OK) return r;
            if (any_views && (r = spmv_views(0, 3, s)) != SB_OK) return r;
        }
        if ((r = allreduce(3, 3, s)) != SB_OK) return r;
        for (int k = 0; k < np; ++k) scalar_kernel<<<1, 1, 0, s>>>(B[k].ctl, DAlpha{});
        SB_CUDA(cudaGetLastError());
        for (int k = 0; k < np; ++k) {
            const sb_dist_part &P = parts[k];
            SB_CUDA(launch_ew<2>(P.n_local, B[k].ctl, B[k].partials,
                                 DUpdate<V>{{}, B[k].pe, B[k].q, (const V *)P.inv_diag, (V *)P.x.data, B[k].r, B[k].z, 0.0}, s));
        }
        if ((r = allreduce(6, 2, s)) != SB_OK) return r;
        for (int k = 0; k < np; ++k) scalar_kernel<<<1, 1, 0, s>>>(B[k].ctl, DCheck{});
        SB_CUDA(cudaGetLastError());
        for (int k = 0; k < np; ++k)
            SB_CUDA(launch_ew<0>(parts[k].n_local, B[k].ctl, B[k].partials, DDirection<V>{{}, B[k].z, B[k].pe, 0.0}, s));
        return SB_OK;
    };

    // ---- setup: t = A x (x copied into the extended vector + halo), r, z, p, dots
    sb_status r;
    for (int k = 0; k < np; ++k) {
        zero_dots_kernel<<<1, 32, 0, st>>>(B[k].ctl);
        SB_CUDA(launch_ew<0>(parts[k].n_local, B[k].ctl, B[k].partials,
                             DCopy<V>{{}, (const V *)parts[k].x.data, B[k].pe}, st));
    }
    if ((r = halo(st)) != SB_OK) return r;
    for (int k = 0; k < np; ++k)
        SB_CUDA((matrix_apply<V, I>(parts[k].a, B[k].pe, 1, B[k].t, 1, EpiStore<V>{B[k].t, 1}, st)));
    for (int k = 0; k < np; ++k) {
        const sb_dist_part &P = parts[k];
        SB_CUDA(launch_ew<3>(P.n_local, B[k].ctl, B[k].partials,
                             DInit<V>{{}, (const V *)P.b.data, B[k].t, (const V *)P.inv_diag, B[k].r, B[k].z, B[k].pe}, st));
    }
    if ((r = allreduce(0, 3, st)) != SB_OK) return r;
    for (int k = 0; k < np; ++k) scalar_kernel<<<1, 1, 0, st>>>(B[k].ctl, DInitCheck{});
    SB_CUDA(cudaGetLastError());

    // ---- iterations: chunks captured once into a CUDA graph, done flag polled a chunk behind
    const int chunk = 8;
    cudaGraphExec_t exec = nullptr;
    if (graph_mode_enabled()) {
        cudaStream_t cs;
        SB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g = nullptr;
        bool okc = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        sb_status cap_status = SB_OK;
        for (int c = 0; okc && c < chunk && cap_status == SB_OK; ++c) cap_status = iteration(cs);
        if (okc) okc = cudaStreamEndCapture(cs, &g) == cudaSuccess && cap_status == SB_OK;
        if (okc) okc = cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        cudaStreamDestroy(cs);
        if (!okc) {
            exec = nullptr;
            cudaGetLastError();
            clear_error(err);
        }
    }
    int *pinned = nullptr;
    cudaEvent_t evs[2];
    SB_CUDA(cudaMallocHost(&pinned, 2 * sizeof(int)));
    SB_CUDA(cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming));
    SB_CUDA(cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming));
    for (int64_t k = 0;; ++k) {
        if (exec) {
            SB_CUDA(cudaGraphLaunch(exec, st));
        } else {
            for (int c = 0; c < chunk; ++c)
                if ((r = iteration(st)) != SB_OK) return r;
        }
        SB_CUDA(cudaMemcpyAsync(&pinned[k & 1], &B[0].ctl->done, sizeof(int), cudaMemcpyDeviceToHost, st));
        SB_CUDA(cudaEventRecord(evs[k & 1], st));
        if (k >= 1) {
            SB_CUDA(cudaEventSynchronize(evs[(k - 1) & 1]));
            if (pinned[(k - 1) & 1]) break;
        }
    }
    Ctl h;
    SB_CUDA(cudaMemcpyAsync(&h, B[0].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    cudaFreeHost(pinned);
    cudaEventDestroy(evs[0]);
    cudaEventDestroy(evs[1]);
    if (exec) cudaGraphExecDestroy(exec);
    if (overlap) {
        cudaStreamDestroy(side);
        cudaEventDestroy(ev_ready);
        cudaEventDestroy(ev_halo);
    }
    SolverWs w{};
    w.hist = B[0].hist;
    SolveArgs a{nullptr, nullptr, nullptr, nullptr, crit, 0, nullptr, log, st, err};
    return finish_log(h, a, w);
}

}  // namespace sb

using namespace sb;

extern "C" {

sb_status sb_nccl_unique_id(char out[128], sb_error *err) {
    SB_GUARD_BEGIN
    if (!nccl().ok) return fail(err, SB_ERR_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    SB_NCCL(nccl().getUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return SB_OK;
    SB_GUARD_END
}

sb_status sb_nccl_comm_init(int32_t nranks, const char id[128], int32_t rank, void **comm, sb_error *err) {
    SB_GUARD_BEGIN
    if (!nccl().ok) return fail(err, SB_ERR_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId uid;
    memcpy(&uid, id, 128);
    ncclComm_t c;
    SB_NCCL(nccl().commInitRank(&c, nranks, uid, rank));
    *comm = (void *)c;
    return SB_OK;
    SB_GUARD_END
}

sb_status sb_nccl_comm_destroy(void *comm, sb_error *err) {
    SB_GUARD_BEGIN
    if (comm) SB_NCCL(nccl().commDestroy((ncclComm_t)comm));
    return SB_OK;
    SB_GUARD_END
}

size_t sb_dist_workspace_bytes(int32_t value_bytes, int64_t n_local, int64_t n_ghost, int64_t history_cap) {
    return dist_ws_bytes(value_bytes, n_local, n_ghost, history_cap);
}

#define SB_DEFS(V, VN, I, IN)                                                                      \
    sb_status sb_dist_cg_solve_##VN##_##IN(sb_dist_part *parts, int32_t nparts, void *comm,        \
                                           const sb_criteria *crit, sb_log *log,                   \
                                           sb_stream_t stream, sb_error *err) {                    \
        SB_GUARD_BEGIN                                                                             \
        return dist_cg<V, I>(parts, nparts, comm, crit, log, as_stream(stream), err);              \
        SB_GUARD_END                                                                               \
    }

SB_DEFS(float, float, int32_t, i32)
SB_DEFS(float, float, int64_t, i64)
SB_DEFS(double, double, int32_t, i32)
SB_DEFS(double, double, int64_t, i64)

}  // extern "C"
