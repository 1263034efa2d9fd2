// dist_krylov.cu -- row-partitioned Krylov solvers across GPUs: Jacobi-CG,
// BiCGSTAB and restarted GMRES(m) over one engine.
//
// Each rank owns a contiguous block of rows; its local CSR has columns renumbered to
// [own rows | ghost rows] with the ghosts grouped by owner.  The iteration kernels are the
// single-GPU solvers' own fused steps (cg.cuh, bicgstab.cuh, gmres.cuh) run on the local
// rows; every reduction is split in two: the kernel's last block stores its LOCAL totals in
// ctl->dot[slot..] (Deferred / StoreTo), the totals are summed across ranks in place
// (ncclAllReduce, or in partition order for the loopback transport), and a one-thread
// kernel runs the unchanged finaliser on the global totals (dlast_kernel): the scalar
// logic -- criteria, breakdown tests, Givens rotations -- is bit for bit the single-GPU
// solver's on every rank, so every rank stops at the same iteration.  Each SpMV input
// lives in an extended vector [own | ghosts] whose ghosts the halo exchange fills (NCCL
// grouped send / recv on a side stream, overlapped with the SpMV of the interior rows
// when the boundary rows are a prefix + suffix of the block).
//
// Sync points per iteration: CG 2 (p.q; r.r + r.z), BiCGSTAB 4 (sigma;
// ||s||; t.t + t.s; r.r + rhat.r), GMRES one per MGS step (h_0j fused into the SpMV, then
// h_ij for i = 1..j and ||w||) -- the reference's single-pass modified Gram-Schmidt order
// (solvers.py:353-358), not a reordered classical Gram-Schmidt.
//
// The loop body is captured ONCE into a CUDA-graph WHILE loop (run_loop, cached across
// solves by buffer identity); the finaliser that decides to stop clears the condition,
// so no iteration runs past convergence and the host waits once.  comm == NULL selects
// the loopback transport: `nparts` partitions on this one GPU, halos as device copies --
// the single-GPU test of the decomposition (NCCL rejects two ranks on one device).
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <vector>

#include "bicgstab.cuh"
#include "cg.cuh"
#include "gmres.cuh"
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

// ---------------------------------------------------------------- split reductions
// slots of ctl->dot: SpMV-fused dots, one group of N per SpMV view (3 views max), and the
// elementwise passes' dots.  A slot group is consumed (and zeroed) by the dlast_kernel
// that follows its allreduce, before the next producer writes it.
constexpr int kSlotSpmv = 0;  // 3 views x up to 2 dots
constexpr int kSlotEw = 8;    // up to 3 dots

// an elementwise step whose last block stores its local totals instead of finalising
template <class Op, int N>
struct Deferred : Op {
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[N]) const {
#pragma unroll
        for (int d = 0; d < N; ++d) c->dot[kSlotEw + d] = tot[d];
    }
};

// SpMV-epilogue finaliser storing the local totals of one view; skips like `Sk`
template <int N, class Sk>
struct StoreTo {
    int slot;
    Sk sk;
    __device__ __forceinline__ bool skip(const Ctl *c) const { return sk.skip(c); }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[N]) const {
#pragma unroll
        for (int d = 0; d < N; ++d) c->dot[slot + d] = tot[d];
    }
};

// global totals = sum of the `nv` view groups (fixed order); zero the slots; finalise
template <class F, int N>
__global__ void dlast_kernel(Ctl *c, F f, int slot, int nv) {
    double tot[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
        tot[d] = 0.0;
        for (int v = 0; v < nv; ++v) tot[d] = addd(tot[d], c->dot[slot + v * N + d]);
    }
    for (int k = 0; k < nv * N; ++k) c->dot[slot + k] = 0.0;
    if (loop_done(c) || f.skip(c)) return;
    f.last(c, tot);
}

template <class V>
struct DCopy : SkipNone {  // dst = src (a local vector into an extended one)
    using value_type = V;
    const V *src;
    V *dst;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        stp<W>(dst, i, ldp<W>(src, i));
    }
};

template <class V>
struct GmCopyZ : SkipCycleEnd {  // z = v_j (GMRES without a preconditioner)
    using value_type = V;
    const V *vj;
    V *z;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&)[1]) const {
        stp<W>(z, i, ldp<W>(vj, i));
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

// loopback "allreduce": sum the partitions' slots in partition order, write to all
__global__ void loopback_sum_kernel(CtlList L, int slot, int count) {
    const int k = threadIdx.x;
    if (k >= count) return;
    double s = 0.0;
    for (int p = 0; p < L.n; ++p) s = addd(s, L.c[p]->dot[slot + k]);
    for (int p = 0; p < L.n; ++p) L.c[p]->dot[slot + k] = s;
}

__global__ void zero_dots_kernel(Ctl *c) {
    for (int k = threadIdx.x; k < 24; k += blockDim.x) c->dot[k] = 0.0;
}

// ---------------------------------------------------------------- workspace
// per partition: Ctl | partials | history | GMRES small arrays | nloc local vectors
// (n_local) | next extended vectors (n_local + n_ghost)
inline void dist_counts(int kind, int64_t dim, int &nloc, int &next) {
    switch (kind) {
    case SB_SOLVER_CG: nloc = 4; next = 1; break;              // r z q t | p
    case SB_SOLVER_BICGSTAB: nloc = 6; next = 2; break;        // r rh p v s t | ph sh
    default: nloc = (int)dim + 1 + 3; next = 1; break;         // V_0..V_m r t w | z
    }
}

inline size_t dist_ws_bytes(int kind, int vbytes, int64_t nl, int64_t ng, int64_t dim, int64_t cap) {
    int nloc, next;
    dist_counts(kind, dim, nloc, next);
    const size_t v = a256((size_t)vbytes * (size_t)(nl > 0 ? nl : 1));
    const size_t ve = a256((size_t)vbytes * (size_t)(nl + ng > 0 ? nl + ng : 1));
    return kCtlBytes + a256(3 * kMaxGrid * sizeof(double)) + a256(sizeof(double) * (size_t)(cap > 0 ? cap : 1)) +
           (kind == SB_SOLVER_GMRES ? gmres_small_bytes(dim) : 0) + (size_t)nloc * v + (size_t)next * ve;
}

template <class V>
struct PartBufs {
    Ctl *ctl;
    double *partials, *hist, *small;
    std::vector<V *> loc, ext;
    size_t vstride;  // elements between consecutive local vectors
};

template <class V>
PartBufs<V> carve_dist(int kind, void *ws, int64_t nl, int64_t ng, int64_t dim, int64_t cap) {
    int nloc, next;
    dist_counts(kind, dim, nloc, next);
    unsigned char *p = (unsigned char *)ws;
    const size_t v = a256(sizeof(V) * (size_t)(nl > 0 ? nl : 1));
    const size_t ve = a256(sizeof(V) * (size_t)(nl + ng > 0 ? nl + ng : 1));
    PartBufs<V> b;
    b.ctl = (Ctl *)p;
    p += kCtlBytes;
    b.partials = (double *)p;
    p += a256(3 * kMaxGrid * sizeof(double));
    b.hist = (double *)p;
    p += a256(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
    b.small = (double *)p;
    if (kind == SB_SOLVER_GMRES) p += gmres_small_bytes(dim);
    for (int k = 0; k < nloc; ++k, p += v) b.loc.push_back((V *)p);
    for (int k = 0; k < next; ++k, p += ve) b.ext.push_back((V *)p);
    b.vstride = v / sizeof(V);
    return b;
}

// ---------------------------------------------------------------- the engine
struct SideRes {  // per device: the halo stream and its fork / join events (kept for good)
    cudaStream_t side = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
};

static SideRes &side_res() {
    static std::mutex mu;
    static std::map<int, SideRes> res;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    SideRes &r = res[dev];
    if (!r.side) {
        cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&r.ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming);
    }
    return r;
}

template <class V, class I>
struct DistEngine {
    sb_dist_part *parts;
    int np;
    ncclComm_t comm;
    std::vector<PartBufs<V>> B;
    CtlList L{};
    bool overlap;
    SideRes side;
    sb_error *err;
    sb_status nccl_status = SB_OK;  // first NCCL failure inside a body (bodies return cudaError_t)

    sb_status init(int kind, int64_t dim, int64_t cap) {
        if (comm && np != 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "NCCL mode takes one partition per rank");
        if (!comm && np > kMaxLoopbackParts) return fail(err, SB_ERR_UNSUPPORTED, "loopback: at most 16 partitions");
        if (comm && !nccl().ok) return fail(err, SB_ERR_NCCL, "libnccl.so.2 could not be loaded");
        B.resize(np);
        L.n = np;
        for (int k = 0; k < np; ++k) {
            const sb_dist_part &P = parts[k];
            if (P.b.cols != 1 || P.x.cols != 1 || P.b.rows != P.n_local || P.x.rows != P.n_local ||
                P.b.stride != 1 || P.x.stride != 1)
                return fail(err, SB_ERR_DIMENSION_MISMATCH, "partition %d: b / x must be n_local x 1 contiguous", k);
            if (((uintptr_t)P.b.data | (uintptr_t)P.x.data | (uintptr_t)P.inv_diag) % 16)
                return fail(err, SB_ERR_UNSUPPORTED, "partition %d: vectors must be 16-byte aligned", k);
            B[k] = carve_dist<V>(kind, P.workspace, P.n_local, P.n_ghost, dim, cap);
            L.c[k] = B[k].ctl;
        }
        overlap = comm && parts[0].num_views > 0;
        if (overlap) side = side_res();
        return SB_OK;
    }

    std::string key(const char *kind, int64_t dim) const {
        std::string s = std::string("dist|") + kind + std::to_string(sizeof(V)) + std::to_string(sizeof(I)) + "|" +
                        std::to_string(dim) + "|" + ptr_key({comm}) + std::to_string(np);
        for (int k = 0; k < np; ++k) {
            const sb_dist_part &P = parts[k];
            s += "|" + matrix_key(P.a) + ptr_key({P.workspace, P.b.data, P.x.data, P.inv_diag, P.send_buf, P.send_idx});
            for (int v = 0; v < P.num_views; ++v) s += matrix_key(P.views[v]);
            s += std::to_string(P.n_local) + "," + std::to_string(P.n_ghost) + "," + std::to_string(P.num_neighbors);
        }
        return s;
    }

    cudaError_t nccl_fail(ncclResult_t r, const char *what) {
        if (nccl_status == SB_OK) nccl_status = fail(err, SB_ERR_NCCL, "%s: %s", what, nccl().errorString(r));
        return cudaErrorUnknown;
    }

    // ghosts of the extended vectors ext[k] (own rows already final)
    cudaError_t halo(int e, cudaStream_t s) {
        if (comm) {
            const sb_dist_part &P = parts[0];
            V *pe = B[0].ext[e];
            for (int j = 0; j < P.num_neighbors; ++j)
                if (P.send_lo[j] < 0 && P.send_count[j] > 0)
                    pack_kernel<V><<<elem_grid(P.send_count[j]), 256, 0, s>>>(
                        P.send_count[j], (const int64_t *)P.send_idx + P.send_off[j], pe, (V *)P.send_buf + P.send_off[j]);
            cudaError_t ce = cudaGetLastError();
            if (ce != cudaSuccess) return ce;
            ncclResult_t r = nccl().groupStart();
            if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
            for (int j = 0; j < P.num_neighbors; ++j) {
                const V *src = P.send_lo[j] >= 0 ? pe + P.send_lo[j] : (const V *)P.send_buf + P.send_off[j];
                if (P.send_count[j] > 0 &&
                    (r = nccl().send(src, P.send_count[j], nccl_type<V>(), P.nbr[j], comm, s)) != ncclSuccess)
                    return nccl_fail(r, "ncclSend");
                if (P.recv_count[j] > 0 &&
                    (r = nccl().recv(pe + P.n_local + P.recv_off[j], P.recv_count[j], nccl_type<V>(), P.nbr[j], comm,
                                     s)) != ncclSuccess)
                    return nccl_fail(r, "ncclRecv");
            }
            if ((r = nccl().groupEnd()) != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
            return cudaSuccess;
        }
        for (int k = 0; k < np; ++k) {  // loopback: pack every sender first
            const sb_dist_part &P = parts[k];
            for (int j = 0; j < P.num_neighbors; ++j)
                if (P.send_lo[j] < 0 && P.send_count[j] > 0)
                    pack_kernel<V><<<elem_grid(P.send_count[j]), 256, 0, s>>>(
                        P.send_count[j], (const int64_t *)P.send_idx + P.send_off[j], B[k].ext[e],
                        (V *)P.send_buf + P.send_off[j]);
        }
        cudaError_t ce = cudaGetLastError();
        if (ce != cudaSuccess) return ce;
        for (int k = 0; k < np; ++k) {
            const sb_dist_part &P = parts[k];
            for (int j = 0; j < P.num_neighbors; ++j) {
                if (P.recv_count[j] == 0) continue;
                const int src_part = P.nbr[j];
                const sb_dist_part &S = parts[src_part];
                int jj = -1;
                for (int u = 0; u < S.num_neighbors; ++u)
                    if (S.nbr[u] == k) jj = u;
                if (jj < 0 || S.send_count[jj] != P.recv_count[j]) return cudaErrorInvalidValue;
                const V *src = S.send_lo[jj] >= 0 ? B[src_part].ext[e] + S.send_lo[jj]
                                                  : (const V *)S.send_buf + S.send_off[jj];
                ce = cudaMemcpyAsync(B[k].ext[e] + P.n_local + P.recv_off[j], src, sizeof(V) * P.recv_count[j],
                                     cudaMemcpyDeviceToDevice, s);
                if (ce != cudaSuccess) return ce;
            }
        }
        return cudaSuccess;
    }

    cudaError_t allreduce(int slot, int count, cudaStream_t s) {
        if (comm) {
            ncclResult_t r = nccl().allReduce(&B[0].ctl->dot[slot], &B[0].ctl->dot[slot], count, ncclFloat64,
                                              ncclSum, comm, s);
            return r == ncclSuccess ? cudaSuccess : nccl_fail(r, "ncclAllReduce");
        }
        if (np > 1) loopback_sum_kernel<<<1, 32, 0, s>>>(L, slot, count);
        return cudaGetLastError();
    }

    // elementwise step on every partition with N split dots -> allreduce -> finaliser
    template <int N, class Op, class Make>
    cudaError_t ew_reduce(Make make, cudaStream_t s) {
        for (int k = 0; k < np; ++k) {
            const Op op = make(k);
            cudaError_t e = launch_ew<N>(parts[k].n_local, B[k].ctl, B[k].partials, Deferred<Op, N>{op}, s);
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = allreduce(kSlotEw, N, s);
        if (e != cudaSuccess) return e;
        for (int k = 0; k < np; ++k) dlast_kernel<Op, N><<<1, 1, 0, s>>>(B[k].ctl, make(k), kSlotEw, 1);
        return cudaGetLastError();
    }

    // elementwise step without a reduction (or with a purely local finaliser) on every partition
    template <int N, class Op, class Make>
    cudaError_t ew_local(Make make, cudaStream_t s) {
        for (int k = 0; k < np; ++k) {
            cudaError_t e = launch_ew<N>(parts[k].n_local, B[k].ctl, B[k].partials, make(k), s);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }

    // y_k = A_k ext_k[e] after the halo of ext[e]; N fused dots of y against u0 / u1 (null
    // u0 = y.y), finalised by Fin on the global totals.  COMP: compensated partials.
    template <int N, bool COMP, class Fin, class Sk>
    cudaError_t spmv_reduce(int e, int yi, int u0i, int u1i, Fin fin, Sk sk, cudaStream_t s) {
        auto view_apply = [&](int k, int v, cudaStream_t st) -> cudaError_t {
            const sb_dist_part &P = parts[k];
            const bool whole = P.num_views == 0;
            const sb_matrix &M = whole ? P.a : P.views[v];
            const int64_t r0 = whole ? 0 : P.view_row0[v];
            V *y = B[k].loc[yi] + r0;
            const V *u0 = u0i < 0 ? nullptr : (u0i >= 100 ? B[k].ext[u0i - 100] : B[k].loc[u0i]) + r0;
            const V *u1 = u1i < 0 ? nullptr : (u1i >= 100 ? B[k].ext[u1i - 100] : B[k].loc[u1i]) + r0;
            const StoreTo<N, Sk> st_fin{kSlotSpmv + v * N, sk};
            if constexpr (COMP)
                return matrix_apply<V, I>(M, B[k].ext[e], 1, y, 1,
                                          EpiSolverC<V, N, StoreTo<N, Sk>>{y, u0, u1, B[k].ctl, B[k].partials, st_fin}, st);
            else
                return matrix_apply<V, I>(M, B[k].ext[e], 1, y, 1,
                                          EpiSolver<V, N, StoreTo<N, Sk>>{y, u0, u1, B[k].ctl, B[k].partials, st_fin}, st);
        };
        cudaError_t ce;
        if (overlap) {  // NCCL, one partition: interior rows while the halo is in flight
            if ((ce = cudaEventRecord(side.ready, s)) != cudaSuccess) return ce;
            if ((ce = cudaStreamWaitEvent(side.side, side.ready, 0)) != cudaSuccess) return ce;
            if ((ce = halo(e, side.side)) != cudaSuccess) return ce;
            if ((ce = cudaEventRecord(side.done, side.side)) != cudaSuccess) return ce;
            if ((ce = view_apply(0, 0, s)) != cudaSuccess) return ce;
            if ((ce = cudaStreamWaitEvent(s, side.done, 0)) != cudaSuccess) return ce;
            for (int v = 1; v < parts[0].num_views; ++v)
                if ((ce = view_apply(0, v, s)) != cudaSuccess) return ce;
        } else {
            if ((ce = halo(e, s)) != cudaSuccess) return ce;
            for (int k = 0; k < np; ++k) {
                const int nv = parts[k].num_views > 0 ? parts[k].num_views : 1;
                for (int v = 0; v < nv; ++v)
                    if ((ce = view_apply(k, v, s)) != cudaSuccess) return ce;
            }
        }
        if ((ce = allreduce(kSlotSpmv, 3 * N, s)) != cudaSuccess) return ce;
        for (int k = 0; k < np; ++k) dlast_kernel<Fin, N><<<1, 1, 0, s>>>(B[k].ctl, fin, kSlotSpmv, 3);
        return cudaGetLastError();
    }

    // t = A ext[e] (store only; the setup / restart products)
    cudaError_t spmv_store(int e, int yi, cudaStream_t s) {
        cudaError_t ce = halo(e, s);
        if (ce != cudaSuccess) return ce;
        for (int k = 0; k < np; ++k)
            if ((ce = matrix_apply<V, I>(parts[k].a, B[k].ext[e], 1, B[k].loc[yi], 1, EpiStore<V>{B[k].loc[yi], 1}, s)) !=
                cudaSuccess)
                return ce;
        return cudaSuccess;
    }

    template <class Op>
    cudaError_t scalar_all(Op op, cudaStream_t s) {
        for (int k = 0; k < np; ++k) scalar_kernel<<<1, 1, 0, s>>>(B[k].ctl, op);
        return cudaGetLastError();
    }

    // initial control blocks; run the loop; the log from partition 0
    sb_status run(LoopSpec &spec, const sb_criteria *crit, int64_t cap, sb_log *log, cudaStream_t st,
                  const std::function<void(Ctl &, int)> &extra = nullptr) {
        std::vector<Ctl> hs(np);
        for (int k = 0; k < np; ++k) {
            Ctl &h = hs[k];
            std::memset(&h, 0, sizeof(h));
            h.max_iters = crit->max_iters;
            h.has_rf = crit->has_residual;
            h.rf = crit->reduction_factor;
            h.stop_reason = STOP_NONE;
            h.hist = B[k].hist;
            h.hist_cap = cap;
            if (extra) extra(h, k);
            SB_CUDA(cudaMemcpyAsync(B[k].ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, st));
            zero_dots_kernel<<<1, 32, 0, st>>>(B[k].ctl);
        }
        SB_CUDA(cudaGetLastError());
        spec.local_fallback = true;
        sb_status s = run_loop(spec, B[0].ctl, hs[0], st, err);
        if (nccl_status != SB_OK) return nccl_status;
        if (s != SB_OK) return s;
        SolverWs w{};
        w.hist = B[0].hist;
        SolveArgs a{nullptr, nullptr, nullptr, nullptr, crit, 0, nullptr, log, st, err};
        return finish_log(hs[0], a, w);
    }
};

// finalisers that only skip like a given rule (SpMV-fused dots)
struct SkipNever {
    __device__ __forceinline__ bool skip(const Ctl *) const { return false; }
};
struct SkipIfCycleEnd {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->cycle_end != 0; }
};
struct SkipIfEarly {
    __device__ __forceinline__ bool skip(const Ctl *c) const { return c->early != 0; }
};

// ---------------------------------------------------------------- CG (solvers.py:188-224)
template <class V, class I>
sb_status dist_cg(sb_dist_part *parts, int np, void *comm, const sb_criteria *crit, sb_log *log, cudaStream_t st,
                  sb_error *err) {
    if (!parts || np < 1 || !crit || !log) return fail(err, SB_ERR_INVALID_ARGUMENT, "dist_cg: null argument");
    if (crit->max_iters < 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "max_iters must be positive");
    DistEngine<V, I> E{parts, np, (ncclComm_t)comm};
    E.err = err;
    const int64_t cap = log->history_cap;
    sb_status s = E.init(SB_SOLVER_CG, 0, cap);
    if (s != SB_OK) return s;
    enum { R = 0, Z = 1, Q = 2, T = 3 };  // local vectors; ext[0] = p
    auto inv = [&](int k) { return (const V *)parts[k].inv_diag; };
    LoopSpec spec;
    spec.key = E.key("cg", 0);
    spec.poll_chunk = 8;
    spec.setup = [&, inv](cudaStream_t q) -> cudaError_t {  // r = b - A x0, z = M r, p = z
        cudaError_t e = E.template ew_local<0, DCopy<V>>(
            [&](int k) { return DCopy<V>{{}, (const V *)parts[k].x.data, E.B[k].ext[0]}; }, q);
        if (e != cudaSuccess) return e;
        if ((e = E.spmv_store(0, T, q)) != cudaSuccess) return e;
        return E.template ew_reduce<3, CgInit<V>>([&, inv](int k) {
            auto &b = E.B[k];
            return CgInit<V>{{}, (const V *)parts[k].b.data, b.loc[T], inv(k), b.loc[R], b.loc[Z], b.ext[0]};
        }, q);
    };
    spec.body = [&, inv](cudaStream_t q) -> cudaError_t {
        // q = A p, p.q -> alpha
        cudaError_t e = E.template spmv_reduce<1, false>(0, Q, 100, -1, CgPqFin{}, SkipNever{}, q);
        if (e != cudaSuccess) return e;
        // x += alpha p; r -= alpha q; z = M r; r.r, r.z -> criteria, beta
        e = E.template ew_reduce<2, CgUpdate<V>>([&, inv](int k) {
            auto &b = E.B[k];
            return CgUpdate<V>{{}, b.ext[0], b.loc[Q], inv(k), (V *)parts[k].x.data, b.loc[R], b.loc[Z], 0.0};
        }, q);
        if (e != cudaSuccess) return e;
        // p = z + beta p
        return E.template ew_local<0, CgDirection<V>>(
            [&](int k) { return CgDirection<V>{{}, E.B[k].loc[Z], E.B[k].ext[0], 0.0}; }, q);
    };
    return E.run(spec, crit, cap, log, st);
}

// ---------------------------------------------------------------- BiCGSTAB (oracle/sbref.cpp)
template <class V, class I>
sb_status dist_bicgstab(sb_dist_part *parts, int np, void *comm, const sb_criteria *crit, sb_log *log,
                        cudaStream_t st, sb_error *err) {
    if (!parts || np < 1 || !crit || !log) return fail(err, SB_ERR_INVALID_ARGUMENT, "dist_bicgstab: null argument");
    if (crit->max_iters < 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "max_iters must be positive");
    DistEngine<V, I> E{parts, np, (ncclComm_t)comm};
    E.err = err;
    const int64_t cap = log->history_cap;
    sb_status s = E.init(SB_SOLVER_BICGSTAB, 0, cap);
    if (s != SB_OK) return s;
    enum { R = 0, RH = 1, P = 2, VV = 3, S = 4, T = 5 };  // ext[0] = phat, ext[1] = shat
    auto inv = [&](int k) { return (const V *)parts[k].inv_diag; };
    LoopSpec spec;
    spec.key = E.key("bicgstab", 0);
    spec.poll_chunk = 8;
    spec.setup = [&](cudaStream_t q) -> cudaError_t {  // r = b - A x0, rhat = r
        cudaError_t e = E.template ew_local<0, DCopy<V>>(
            [&](int k) { return DCopy<V>{{}, (const V *)parts[k].x.data, E.B[k].ext[0]}; }, q);
        if (e != cudaSuccess) return e;
        if ((e = E.spmv_store(0, T, q)) != cudaSuccess) return e;
        return E.template ew_reduce<2, BiShadowInit<V>>([&](int k) {
            auto &b = E.B[k];
            return BiShadowInit<V>{{{}, (const V *)parts[k].b.data, b.loc[T], b.loc[R], b.loc[RH]}};
        }, q);
    };
    spec.body = [&, inv](cudaStream_t q) -> cudaError_t {
        // p = r + beta (p - omega v); phat = M p
        cudaError_t e = E.template ew_local<0, BiDirection<V>>([&, inv](int k) {
            auto &b = E.B[k];
            return BiDirection<V>{{}, b.loc[R], b.loc[VV], inv(k), b.loc[P], b.ext[0], 0, 0, false};
        }, q);
        if (e != cudaSuccess) return e;
        // v = A phat, sigma = rhat.v -> alpha
        if ((e = E.template spmv_reduce<1, true>(0, VV, RH, -1, BiSigmaFin{}, SkipNever{}, q)) != cudaSuccess) return e;
        // s = r - alpha v; shat = M s; ||s|| (early stop)
        e = E.template ew_reduce<1, BiS<V>>([&, inv](int k) {
            auto &b = E.B[k];
            return BiS<V>{{}, b.loc[R], b.loc[VV], inv(k), b.loc[S], b.ext[1], 0};
        }, q);
        if (e != cudaSuccess) return e;
        e = E.template ew_local<1, BiEarlyX<V>>(
            [&](int k) { return BiEarlyX<V>{E.B[k].ext[0], (V *)parts[k].x.data, 0}; }, q);
        if (e != cudaSuccess) return e;
        // t = A shat; t.t, t.s -> omega
        if ((e = E.template spmv_reduce<2, true>(1, T, -1, S, BiOmegaFin{}, SkipIfEarly{}, q)) != cudaSuccess) return e;
        // x += alpha phat + omega shat; r = s - omega t; r.r, rhat.r
        return E.template ew_reduce<2, BiUpdate<V>>([&](int k) {
            auto &b = E.B[k];
            return BiUpdate<V>{{}, b.ext[0], b.ext[1], b.loc[S], b.loc[T], b.loc[RH], (V *)parts[k].x.data, b.loc[R], 0, 0};
        }, q);
    };
    return E.run(spec, crit, cap, log, st);
}

// ---------------------------------------------------------------- GMRES(m) (solvers.py:322-399)
template <class V, class I>
sb_status dist_gmres(sb_dist_part *parts, int np, void *comm, const sb_criteria *crit, int64_t m, sb_log *log,
                     cudaStream_t st, sb_error *err) {
    if (!parts || np < 1 || !crit || !log) return fail(err, SB_ERR_INVALID_ARGUMENT, "dist_gmres: null argument");
    if (crit->max_iters < 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "max_iters must be positive");
    if (m < 1) return fail(err, SB_ERR_INVALID_ARGUMENT, "krylov_dim must be positive");
    if (m > 4096) return fail(err, SB_ERR_UNSUPPORTED, "krylov_dim > 4096");
    DistEngine<V, I> E{parts, np, (ncclComm_t)comm};
    E.err = err;
    const int64_t cap = log->history_cap;
    sb_status s = E.init(SB_SOLVER_GMRES, m, cap);
    if (s != SB_OK) return s;
    const int R = (int)m + 1, T = (int)m + 2, Wv = (int)m + 3;  // loc[0..m] = basis; ext[0] = z / x
    auto inv = [&](int k) { return (const V *)parts[k].inv_diag; };
    LoopSpec spec;
    spec.key = E.key("gmres", m);
    spec.poll_chunk = 1;
    spec.setup = [&](cudaStream_t q) -> cudaError_t {
        return E.template ew_reduce<1, NormB<V>>([&](int k) { return NormB<V>{{}, (const V *)parts[k].b.data}; }, q);
    };
    spec.body = [&, inv](cudaStream_t q) -> cudaError_t {  // one restart cycle
        // r = b - A x, beta = ||r|| (restart; exact solution / finish tests in GmRestart::last)
        cudaError_t e = E.template ew_local<0, DCopy<V>>(
            [&](int k) { return DCopy<V>{{}, (const V *)parts[k].x.data, E.B[k].ext[0]}; }, q);
        if (e != cudaSuccess) return e;
        if ((e = E.spmv_store(0, T, q)) != cudaSuccess) return e;
        e = E.template ew_reduce<1, GmRestart<V>>([&](int k) {
            auto &b = E.B[k];
            return GmRestart<V>{{}, (const V *)parts[k].b.data, b.loc[T], b.loc[R]};
        }, q);
        if (e != cudaSuccess) return e;
        e = E.template ew_local<0, GmFirstBasis<V>>(
            [&](int k) { return GmFirstBasis<V>{{}, E.B[k].loc[R], E.B[k].loc[0], 0.0}; }, q);
        if (e != cudaSuccess) return e;
        for (int64_t j = 0; j < m; ++j) {
            // z = M v_j (own rows of the extended vector), halo, w = A z with h_0j fused
            if (parts[0].inv_diag) {
                e = E.template ew_local<0, GmPrecond<V>>([&, inv, j](int k) {
                    return GmPrecond<V>{{}, E.B[k].loc[j], inv(k), E.B[k].ext[0]};
                }, q);
            } else {
                e = E.template ew_local<0, GmCopyZ<V>>(
                    [&, j](int k) { return GmCopyZ<V>{{}, E.B[k].loc[j], E.B[k].ext[0]}; }, q);
            }
            if (e != cudaSuccess) return e;
            if ((e = E.template spmv_reduce<1, false>(0, Wv, 0, -1, GmH0Fin{}, SkipIfCycleEnd{}, q)) != cudaSuccess)
                return e;
            // single-pass MGS: w -= h_i v_i with h_{i+1} = v_{i+1}.w, one allreduce per step
            for (int64_t i = 0; i < j; ++i) {
                e = E.template ew_reduce<1, GmMgsStep<V>>([&, i](int k) {
                    auto &b = E.B[k];
                    return GmMgsStep<V>{{}, b.loc[i], b.loc[i + 1], b.loc[Wv], (int)i, 0.0};
                }, q);
                if (e != cudaSuccess) return e;
            }
            // w -= h_jj v_j, ||w|| -> rotations, estimate, criteria, cycle end
            e = E.template ew_reduce<1, GmMgsLast<V>>([&, j](int k) {
                auto &b = E.B[k];
                return GmMgsLast<V>{{}, b.loc[j], b.loc[Wv], (int)j, 0.0};
            }, q);
            if (e != cudaSuccess) return e;
            if (j + 1 < m) {
                e = E.template ew_local<0, GmNextBasis<V>>(
                    [&, j](int k) { return GmNextBasis<V>{{}, E.B[k].loc[Wv], E.B[k].loc[j + 1], 0.0}; }, q);
                if (e != cudaSuccess) return e;
            }
        }
        if ((e = E.scalar_all(GmBackSub{}, q)) != cudaSuccess) return e;
        // x += M (V_k y); finish if a criterion fired (local per partition)
        return E.template ew_local<1, GmUpdate<V, 0>>([&, inv](int k) {
            auto &b = E.B[k];
            return GmUpdate<V, 0>{{}, b.loc[0], b.vstride, inv(k), (V *)parts[k].x.data, nullptr, 0};
        }, q);
    };
    return E.run(spec, crit, cap, log, st, [&](Ctl &h, int k) {
        double *sm = E.B[k].small;
        h.dim = m;
        h.hcol = sm;
        h.g = sm + (m + 2);
        h.cs = sm + 2 * (m + 2);
        h.sn = sm + 3 * (m + 2);
        h.y = sm + 4 * (m + 2);
        h.R = sm + 4 * (m + 2) + m;
    });
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
    return dist_ws_bytes(SB_SOLVER_CG, value_bytes, n_local, n_ghost, 0, history_cap);
}

size_t sb_dist_solver_workspace_bytes(int32_t solver, int32_t value_bytes, int64_t n_local, int64_t n_ghost,
                                      int64_t krylov_dim, int64_t history_cap) {
    return dist_ws_bytes(solver, value_bytes, n_local, n_ghost, krylov_dim, history_cap);
}

#define SB_DEFS(V, VN, I, IN)                                                                       \
    sb_status sb_dist_cg_solve_##VN##_##IN(sb_dist_part *parts, int32_t nparts, void *comm,         \
                                           const sb_criteria *crit, sb_log *log,                    \
                                           sb_stream_t stream, sb_error *err) {                     \
        SB_GUARD_BEGIN                                                                              \
        return dist_cg<V, I>(parts, nparts, comm, crit, log, as_stream(stream), err);               \
        SB_GUARD_END                                                                                \
    }                                                                                               \
    sb_status sb_dist_bicgstab_solve_##VN##_##IN(sb_dist_part *parts, int32_t nparts, void *comm,   \
                                                 const sb_criteria *crit, sb_log *log,              \
                                                 sb_stream_t stream, sb_error *err) {               \
        SB_GUARD_BEGIN                                                                              \
        return dist_bicgstab<V, I>(parts, nparts, comm, crit, log, as_stream(stream), err);         \
        SB_GUARD_END                                                                                \
    }                                                                                               \
    sb_status sb_dist_gmres_solve_##VN##_##IN(sb_dist_part *parts, int32_t nparts, void *comm,      \
                                              const sb_criteria *crit, int64_t krylov_dim,          \
                                              sb_log *log, sb_stream_t stream, sb_error *err) {     \
        SB_GUARD_BEGIN                                                                              \
        return dist_gmres<V, I>(parts, nparts, comm, crit, krylov_dim, log, as_stream(stream), err); \
        SB_GUARD_END                                                                                \
    }

SB_DEFS(float, float, int32_t, i32)
SB_DEFS(float, float, int64_t, i64)
SB_DEFS(double, double, int32_t, i32)
SB_DEFS(double, double, int64_t, i64)

}  // extern "C"
