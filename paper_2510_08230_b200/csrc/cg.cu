// cg.cu -- preconditioned CG on the device (solvers.py:188-224): 3 fused kernels per iteration.
#include <cmath>
#include <atomic>
#include <cstdlib>
#include <vector>

#include "cg.cuh"
#include "solver_common.cuh"
#include "trisolve.cuh"

namespace sb {

// ---------------------------------------------------------------- fused-direction CG
// Two kernels per iteration instead of three.  Iteration k's SpMV evaluates the search
// direction p_k = z + beta p_{k-1} (scal then axpy, the reference's exact rounding) on
// the fly at every gathered column, so p_k is never a separate pass: the epilogue
// stores q = A p_k and the row's own p_k (ping-pong buffers: iteration k reads
// buf[(k-1)&1] and writes buf[k&1], so no CTA overwrites a value another CTA still
// gathers) and accumulates p_k.q; the update kernel then reads p_k back for x.
// Per iteration: A + 12 V n bytes instead of A + 13 V n, and one launch fewer; every
// value is bitwise what the three-kernel loop computes.
template <class V>
__device__ __forceinline__ V cg_direction(bool first, double beta, V zc, V pc) {
    return first ? zc : axpy_e(1.0, zc, scal_e(beta, pc));  // p = z + beta p (scal; axpy)
}

template <class V>
struct EpiCgFused {
    static constexpr int N = 1;
    static constexpr int kMinThreadsPerSM = 1024;
    V *q, *pnew;
    const V *z, *pold;
    Ctl *ctl;
    double *partials;
    double beta;
    int first;
    __device__ __forceinline__ bool skip() const { return loop_done(ctl); }
    __device__ __forceinline__ void prepare() {
        // read before any CTA of this launch can finish (the last CTA, which rewrites
        // iter, starts its finalisation only after every CTA has arrived)
        first = ctl->iter == 0;
        beta = ctl->beta;
    }
    __device__ __forceinline__ V gather(int64_t c) const {
        return cg_direction(first, beta, __ldg(z + c), __ldg(pold + c));
    }
    __device__ __forceinline__ void row(int64_t i, double acc, double (&part)[N]) const {
        const V qi = (V)acc;
        q[i] = qi;
        const V pi = gather(i);
        pnew[i] = pi;
        part[0] = addd(part[0], mulp(pi, qi));
    }
    __device__ __forceinline__ void finish(double (&part)[N]) const {
        double tot[N];
        if (grid_reduce<N>(part, partials, &ctl->ticket[0], tot) && threadIdx.x == 0)
            CgPqFin{}.last(ctl, tot);
    }
};

// ---------------------------------------------------------------- persistent CG
// The whole iteration loop as ONE cooperative kernel (CSR, TMA-staged row blocks): every
// CTA owns the row blocks bid, bid + G, ... for the SpMV *and* the vector updates, and
// the two reductions of an iteration are grid barriers after which every CTA sums the
// per-CTA partials in the same fixed order (deterministic, identical scalars in every
// CTA, so all CTAs take the same stop decision).  Per iteration:
//   A: q = A p_k with p_k = z + beta p_{k-1} gathered on the fly (as EpiCgFused), store
//      q and the own p_k, partial p_k.q; when its blocks are done, the CTA already
//      issues the TMA copy of its first block of the NEXT SpMV (the matrix is
//      immutable), so the stream restarts without a ramp after the barriers;
//   barrier -> alpha (breakdown test);
//   B: own rows: x += alpha p_k, r -= alpha q, z = M r, partials r.r, r.z;
//   barrier -> ||r||, history, criteria, beta.
// Vectors written by other CTAs inside the launch are read with plain (L1-cached)
// loads: the acquire side of every grid barrier invalidates the SM's L1 (CCTL.IVALL in
// the SASS), so no line cached before the barrier survives it.  The arithmetic of every element is the reference's
// (and the graph loop's); only the summation order of the dots differs.
struct CgPArgs {
    int64_t n, nnz;
    int64_t nblk;  // row blocks: nblk = kb * G of bq or bq + 1 rows (cg_block_row)
    int64_t bq, rem;
    int kb;        // blocks per CTA (every CTA owns exactly kb blocks: no 13-vs-14 tail)
    const void *rp, *ci, *val, *inv;
    void *x, *r, *z, *p0, *p1, *q;
    Ctl *ctl;
    double *partials;  // 3 G doubles: [p.q | r.r, r.z] (+ G arrival stamps when profiling)
    unsigned long long *prof;  // optional: arrival stamps of barriers 10..27 (18 G) + CTA 0 releases
    int nnz_cap;
    int pf;  // update-phase L2 prefetch distance in blocks (SPARSEB200_CG_PF; 0 = off; 128^3:
             // 1 / 2 / 3 blocks ahead 72.4 / 73.2 / 74.4 us per iteration)
    void *q1;  // single-sync kernel: second q buffer (z doubles as the second r buffer)
    int xa;    // two-barrier kernel: x update deferred into the next SpMV phase
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier over all CTAs of a cooperative launch: a monotonic 64-bit arrival counter
// (reset per solve).  Thread 0 of each CTA arrives with a fire-and-forget release
// reduction and polls with acquire loads until every CTA of this epoch has arrived;
// the acquire also invalidates the SM's L1, the surrounding __syncthreads extend the
// ordering to the whole CTA.
__device__ __forceinline__ void grid_barrier(unsigned long long *count, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(count) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// The same barrier with CTA-local work in the wait: after arriving, the CTA runs work()
// steps (each uniform across the CTA; false = nothing left) between polls of the
// counter, so an early CTA spends the arrival spread on deferred work instead of idling.
struct NoWork {
    __device__ __forceinline__ bool operator()() const { return false; }
};
template <class W>
__device__ __forceinline__ void grid_barrier_w(unsigned long long *count, unsigned long long target, W &work) {
    __shared__ int s_go[2];
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
    for (unsigned k = 0;; ++k) {
        if (threadIdx.x == 0) {
            unsigned long long v;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(count) : "memory");
            s_go[k & 1] = v >= target;
        }
        __syncthreads();
        if (s_go[k & 1]) return;  // slot k & 1 is rewritten only after the next __syncthreads
        if (!work()) break;
    }
    if (threadIdx.x == 0) {
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(count) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// every CTA publishes its N partials, waits, then sums all G partials in index order
template <int N, int R, class W = NoWork>
__device__ __forceinline__ void grid_allreduce(double (&v)[N], double *partials, unsigned long long *count,
                                               unsigned long long target, double (&tot)[N],
                                               unsigned long long *stamps = nullptr, W *work = nullptr) {
    __shared__ double scratch[32][N];
    __shared__ double s_tot[N];
    block_reduce<N>(v, scratch);
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) partials[k * G + blockIdx.x] = v[k];
        if (stamps && target / G >= 10 && target / G < 28)  // arrival stamps of barriers 10..27
            stamps[(target / G - 10) * G + blockIdx.x] = gtimer();
    }
    if constexpr (!std::is_same<W, NoWork>::value)
        grid_barrier_w(count, target, *work);
    else
        grid_barrier(count, target);
    unsigned long long t_rel = 0;
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0) t_rel = gtimer();
    double a[N];
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = 0.0;
    constexpr int U = N > 2 ? 1 : 4;  // independent loads in flight per thread (registers: N U doubles)
    for (int i0 = threadIdx.x; i0 < G; i0 += U * R) {
        double t[N][U];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < N; ++k) t[k][u] = i0 + u * R < G ? __ldcg(partials + k * G + i0 + u * R) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < N; ++k) a[k] = addd(a[k], t[k][u]);
    }
    block_reduce<N>(a, scratch);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < N; ++k) s_tot[k] = a[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) tot[k] = s_tot[k];
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0 && target / G >= 10 && target / G < 28)
        stamps[18 * G + (target / G - 10)] = t_rel;  // CTA 0's release time
}

// first row of block b.  Blocks are whole 32-row units (warp-aligned vector accesses):
// blocks 0 .. rem-1 hold bq + 1 units, the others bq (bq = units / nblk, rem = units %
// nblk precomputed on the host, units = ceil(n / 32): no division in the kernel); the
// last block is clipped to n by the caller's row bound.
__host__ __device__ __forceinline__ int64_t cg_block_row(int64_t b, int64_t bq, int64_t rem) {
    return 32 * (b * bq + (b < rem ? b : rem));
}

// PROF: phase timers and barrier arrival stamps (SPARSEB200_CG_PROFILE; a separate
// instantiation, so the timed kernel carries no timer registers)
// BT: update-phase operands (q, p_k, x, r, M) TMA-staged two blocks ahead into the stage
// slot the SpMV ring leaves free during the update (see below)
// XW: the x update (x += alpha_k p_k on the own rows, needed by nothing inside the loop)
// is deferred and run in the grid-barrier waits (grid_barrier_w): it only has to land
// before p_k's buffer is rewritten two SpMV phases later, and each CTA owns the same
// rows of x and p in both phases, so the deadline is CTA-local.  What the waits leave
// over is flushed right after the next alpha (in row order: x_k = x_{k-1} + alpha_k p_k
// per element, the reference's rounding); the staged update phase reads q, r, M only.
template <class V, class I, int R, bool PROF = false, bool BT = false, bool XW = false>
__global__ void __launch_bounds__(R, 1024 / R) cg_persistent_kernel(CgPArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ __align__(8) uint64_t barB[4];
    __shared__ StreamMeta meta[2];
    Ctl *c = a.ctl;
    if (c->done) return;  // setup found the exact solution
    const I *rp = (const I *)a.rp, *ci = (const I *)a.ci;
    const V *val = (const V *)a.val, *inv = (const V *)a.inv;
    V *x = (V *)a.x, *r = (V *)a.r, *z = (V *)a.z, *q = (V *)a.q;
    const int64_t n = a.n, nnz = a.nnz;
    const StreamLayout<V, I> L(R, a.nnz_cap);
    const size_t sb = L.stage_bytes();
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int64_t nblk = a.nblk, bq = a.bq, rem = a.rem;
    const int kb = a.kb;
    const int64_t bid = blockIdx.x;
    const uint64_t pol = policy_evict_first();
    unsigned long long *count = &c->barrier;
    unsigned long long epoch = 0;  // barriers passed in this launch
    // row-pointer bounds of this CTA's kb blocks, loaded once: issue() then starts its bulk
    // copies without a dependent global load (thread 0 was a full L2 round trip behind
    // the other threads of every block, which the block-end __syncthreads exposed)
    int64_t *kbnd = reinterpret_cast<int64_t *>(smem + 2 * sb);
    for (int q2 = tid; q2 < kb; q2 += R) {
        const int64_t blk = bid + (int64_t)q2 * G;
        kbnd[2 * q2] = rp[cg_block_row(blk, bq, rem)];
        kbnd[2 * q2 + 1] = rp[min(cg_block_row(blk + 1, bq, rem), n)];
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        for (int h = 0; h < 4; ++h) mbar_init(&barB[h], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // update-phase staging: with BT the SpMV ring issues the next SpMV's first block only
    // after the update phase, so both stage slots are free during it: four half-slots,
    // each holding one block's five operand ranges (four blocks in flight per CTA)
    constexpr size_t kVecB = ((size_t)R * sizeof(V) + 15) & ~size_t(15);
    const size_t hb = (sb / 2) & ~size_t(15);
    uint32_t bseq = 0;  // update-phase blocks consumed in this launch (half-slot bseq & 3)
    int bpend = 0;      // update-phase blocks issued but not consumed
    auto issueB = [&](int j, int h, const V *pk) {  // thread 0 only
        unsigned char *dst = smem + (h >> 1) * sb + (h & 1) * hb;
        const int64_t blk = bid + (int64_t)j * G;
        const int64_t r0 = cg_block_row(blk, bq, rem), r1 = min(cg_block_row(blk + 1, bq, rem), n);
        const V *src[5] = {q, XW ? nullptr : pk, XW ? nullptr : x, r, inv};
        uint32_t by[5], tot = 0;
        int64_t base = r0;
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            by[v] = src[v] ? stage_range(src[v], r0, r1, n, reinterpret_cast<V *>(dst + v * kVecB), base) : 0;
            tot += by[v];
        }
        mbar_arrive_expect_tx(&barB[h], tot);
#pragma unroll
        for (int v = 0; v < 5; ++v)
            if (by[v]) bulk_g2s(dst + v * kVecB, src[v] + base, by[v], &barB[h]);
    };
    auto issue = [&](int64_t blk, int s) {  // thread 0 only (as csr_stream_kernel)
        unsigned char *st = smem + s * sb;
        V *sv = reinterpret_cast<V *>(st);
        I *sc = reinterpret_cast<I *>(st + L.off_c());
        I *sr = reinterpret_cast<I *>(st + L.off_r());
        const int64_t r0 = cg_block_row(blk, bq, rem), r1 = min(cg_block_row(blk + 1, bq, rem), n);
        const int64_t q2 = (blk - bid) / G;
        const int64_t k0 = kbnd[2 * q2], k1 = kbnd[2 * q2 + 1];
        StreamMeta m;
        m.r0 = r0;
        m.r1 = r1;
        uint32_t bv = stage_range(val, k0, k1, nnz, sv, m.av);
        uint32_t bc = stage_range(ci, k0, k1, nnz, sc, m.ac);
        uint32_t br = stage_range(rp, r0, r1 + 1, n + 1, sr, m.ar);
        meta[s] = m;
        mbar_arrive_expect_tx(&bar[s], bv + bc + br);
        if (bv) bulk_g2s(sv, val + m.av, bv, &bar[s], pol);
        if (bc) bulk_g2s(sc, ci + m.ac, bc, &bar[s], pol);
        if (br) bulk_g2s(sr, rp + m.ar, br, &bar[s], pol);
    };
    uint32_t seq = 0;  // ring position: stage seq & 1, parity (seq >> 1) & 1
    bool apend = true;  // a next-SpMV block is staged when the loop ends
    if (tid == 0 && bid < nblk) issue(bid, 0);

    int64_t it = c->iter;
    double rz = c->rz, beta = 0.0;
    const double bnorm = c->bnorm;
    bool first = true;
    // x update deferred into the next SpMV phase (x_{k-1} += alpha_{k-1} p_{k-1} where the
    // own p_{k-1} is already loaded): the update phase no longer reads p or x
    const bool xa = a.xa;
    bool flush = false;
    double alpha = 0.0;
    V *pold = (V *)a.p0, *pnew = (V *)a.p1;
    unsigned long long tp[4] = {0, 0, 0, 0}, t0 = PROF ? gtimer() : 0, t1;
    // XW: outstanding x update x += xalpha xp on this CTA's blocks xj .. kb-1
    double xalpha = 0.0;
    const V *xp = nullptr;
    int xj = kb;
    // two blocks per step (four loads in flight per thread; four blocks per step and a
    // poll issued behind the step's loads measured no better: profiles/README.md)
    constexpr int XB = 2;
    auto xstep = [&]() -> bool {
        if (xj >= kb) return false;
        int64_t ix[XB];
        bool ok[XB];
        V pv[XB], xv[XB];
#pragma unroll
        for (int u = 0; u < XB; ++u) {
            const int64_t bu = bid + (int64_t)(xj + u) * G;
            ix[u] = cg_block_row(bu, bq, rem) + tid;
            ok[u] = xj + u < kb && ix[u] < min(cg_block_row(bu + 1, bq, rem), n);
            pv[u] = ok[u] ? xp[ix[u]] : V(0);
            xv[u] = ok[u] ? x[ix[u]] : V(0);
        }
#pragma unroll
        for (int u = 0; u < XB; ++u)
            if (ok[u]) x[ix[u]] = axpy_e(xalpha, pv[u], xv[u]);
        xj += XB;
        return true;
    };
    for (;;) {
        // ---- A: q = A p_k, p_k = z + beta p_{k-1} gathered on the fly
        double part[1] = {0.0};
        for (int64_t blk = bid; blk < nblk; blk += G, ++seq) {
            const int s = seq & 1;
            const int64_t nxt = blk + G < nblk ? blk + G : bid;  // wrap: next SpMV's first block
            // (every block has <= R rows: nblk >= ceil(n / R))
            if (tid == 0 && (!BT || blk + G < nblk)) issue(nxt, s ^ 1);  // BT: wrap after the update
            mbar_wait(&bar[s], (seq >> 1) & 1);
            const unsigned char *st = smem + s * sb;
            const V *sv = reinterpret_cast<const V *>(st);
            const I *sc = reinterpret_cast<const I *>(st + L.off_c());
            const I *sr = reinterpret_cast<const I *>(st + L.off_r());
            const StreamMeta m = meta[s];
            const int64_t i = m.r0 + tid;
            if (i < m.r1) {
                // 32-bit stage offsets of the row (as csr_stream_kernel)
                const int64_t kb = sr[i - m.ar], ke = sr[i + 1 - m.ar];
                const int ov = (int)(kb - m.av), oc = (int)(kb - m.ac), cnt = (int)(ke - kb);
                double acc = 0.0;
                for (int t = 0; t < cnt; t += 8) {
                    V vv[8], bb[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int kk = t + j < cnt ? t + j : cnt - 1;
                        const int64_t col = (int64_t)sc[oc + kk];
                        vv[j] = sv[ov + kk];
                        bb[j] = cg_direction(first, beta, z[col], pold[col]);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (t + j < cnt) acc = addd(acc, mulp(vv[j], bb[j]));
                }
                const V qi = (V)acc;
                const V po = pold[i];
                const V pi = cg_direction(first, beta, z[i], po);
                if (xa && !first) x[i] = axpy_e(alpha, po, x[i]);  // x_{k-1} (deferred update)
                q[i] = qi;
                pnew[i] = pi;
                part[0] = addd(part[0], mulp(pi, qi));
            }
            __syncthreads();  // stage s consumed before it is re-issued
        }
        if constexpr (PROF) {
            t1 = gtimer();
            tp[0] += t1 - t0;
            t0 = t1;
        }
        if constexpr (BT) {
            // q and p_k were just stored by this CTA's threads: order those generic writes
            // before the async-proxy (TMA) reads, then stage the first two update blocks so
            // their loads overlap barrier 1
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                for (int j = 0; j < 4 && j < kb; ++j) issueB(j, (bseq + j) & 3, pnew);
            }
            bpend = kb < 4 ? kb : 4;
        }
        double pq[1];
        if constexpr (XW)
            grid_allreduce<1, R>(part, a.partials, count, ++epoch * G, pq, PROF ? a.prof : nullptr, &xstep);
        else
            grid_allreduce<1, R>(part, a.partials, count, ++epoch * G, pq, PROF ? a.prof : nullptr);
        if constexpr (XW)
            while (xstep()) {
            }  // the rest of x_{k-1} += alpha_{k-1} p_{k-1} before p_{k+1} reuses that buffer
        if constexpr (PROF) {
            t1 = gtimer();
            tp[1] += t1 - t0;
            t0 = t1;
        }
        ++it;
        if (!isfinite(pq[0]) || pq[0] <= kBreakdownRtol * fabs(rz)) {
            if (bid == 0 && tid == 0) breakdown(c, it);
            if (BT && tid == 0)  // no bulk copy outlives the CTA
                for (int j = 0; j < bpend; ++j) mbar_wait(&barB[(bseq + j) & 3], ((bseq + j) >> 2) & 1);
            apend = !BT;  // BT: the next SpMV's first block is not staged yet
            break;
        }
        alpha = rz / pq[0];
        if constexpr (XW) {
            xalpha = alpha;
            xp = pnew;
            xj = 0;
        }
        // ---- B: x += alpha p_k; r -= alpha q; z = M r; r.r, r.z on the rows of this CTA's
        // own SpMV blocks (same moving window over memory as phase A; measured faster than
        // a balanced contiguous split, which scatters the accesses over the whole vectors)
        double part2[2] = {0.0, 0.0};
        if constexpr (BT) {
            for (int j = 0; j < kb; ++j, ++bseq) {
                const int h = bseq & 3;
                mbar_wait(&barB[h], (bseq >> 2) & 1);
                const unsigned char *src = smem + (h >> 1) * sb + (h & 1) * hb;
                const V *sq = reinterpret_cast<const V *>(src), *sp = reinterpret_cast<const V *>(src + kVecB),
                        *sx = reinterpret_cast<const V *>(src + 2 * kVecB), *sr = reinterpret_cast<const V *>(src + 3 * kVecB),
                        *sd = reinterpret_cast<const V *>(src + 4 * kVecB);
                const int64_t blk = bid + (int64_t)j * G;
                const int64_t i = cg_block_row(blk, bq, rem) + tid;  // block rows start 32-aligned: slot index tid
                if (i < min(cg_block_row(blk + 1, bq, rem), n)) {
                    if constexpr (!XW) x[i] = axpy_e(alpha, sp[tid], sx[tid]);
                    const V ri = axpy_e(-alpha, sq[tid], sr[tid]);
                    const V zi = inv ? vmul(ri, sd[tid]) : ri;
                    r[i] = ri;
                    z[i] = zi;
                    part2[0] = addd(part2[0], mulp(ri, ri));
                    part2[1] = addd(part2[1], mulp(ri, zi));
                }
                __syncthreads();  // half-slot consumed before it is re-issued
                if (tid == 0 && j + 4 < kb) issueB(j + 4, h, pnew);
            }
            bpend = 0;
            if (tid == 0 && bid < nblk) issue(bid, seq & 1);  // the next SpMV's first block (overlaps barrier 2)
        } else
        for (int j = 0; j < kb; ++j) {
            const int64_t blk = bid + (int64_t)j * G;
            const int64_t i = cg_block_row(blk, bq, rem) + tid;
            const bool own = i < min(cg_block_row(blk + 1, bq, rem), n);
            // five threads hint the next block's operands into L2 (cp.async.bulk.prefetch):
            // doubles the bytes in flight of this one-row-per-thread pass (128^3: 73.2 ->
            // 71.1 us per iteration; the same hint for the SpMV phase's gathered vectors
            // measured no better, and for the stream SpMV's matrix ranges beyond its TMA
            // ring slower: 36.0 -> 37.6 us at 128^3)
            if (a.pf && tid < 5 && j + a.pf < kb) {
                const int64_t nb = blk + (int64_t)a.pf * G;
                const int64_t b0 = cg_block_row(nb, bq, rem), b1 = min(cg_block_row(nb + 1, bq, rem), n);
                const V *vp = tid == 0 ? (xa ? nullptr : x) : tid == 1 ? r : tid == 2 ? q : tid == 3 ? (xa ? nullptr : pnew) : inv;
                if (vp) l2_prefetch_range(vp + b0, vp + b1);
            }
            if (own) {
                const V qi = q[i];
                if (!xa) x[i] = axpy_e(alpha, pnew[i], x[i]);
                const V ri = axpy_e(-alpha, qi, r[i]);
                const V zi = inv ? vmul(ri, inv[i]) : ri;
                r[i] = ri;
                z[i] = zi;
                part2[0] = addd(part2[0], mulp(ri, ri));
                part2[1] = addd(part2[1], mulp(ri, zi));
            }
        }
        if constexpr (PROF) {
            t1 = gtimer();
            tp[2] += t1 - t0;
            t0 = t1;
        }
        double tot[2];
        if constexpr (XW)
            grid_allreduce<2, R>(part2, a.partials + G, count, ++epoch * G, tot, PROF ? a.prof : nullptr, &xstep);
        else
            grid_allreduce<2, R>(part2, a.partials + G, count, ++epoch * G, tot, PROF ? a.prof : nullptr);
        if constexpr (PROF) {
            t1 = gtimer();
            tp[3] += t1 - t0;
            t0 = t1;
        }
        const double rnorm = sqrt(tot[0]);
        int reason = check_criteria(c, it, rnorm, bnorm);
        if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
        if (bid == 0 && tid == 0) {
            c->rnorm = rnorm;
            record(c, it, rnorm);
        }
        if (reason != STOP_NONE) {
            if (bid == 0 && tid == 0) finish_with(c, it, reason);
            flush = xa;
            break;
        }
        if (!isfinite(tot[1]) || rz == 0.0) {
            if (bid == 0 && tid == 0) breakdown(c, it);
            flush = xa;
            break;
        }
        beta = tot[1] / rz;
        rz = tot[1];
        first = false;
        V *t = pold;
        pold = pnew;
        pnew = t;
    }
    if constexpr (XW)
        while (xstep()) {
        }  // the outstanding x update (every exit: x holds the last accepted iterate)
    if (flush)  // the last iteration's x update (x_k = x_{k-1} + alpha_k p_k, own rows)
        for (int j = 0; j < kb; ++j) {
            const int64_t blk = bid + (int64_t)j * G;
            const int64_t i = cg_block_row(blk, bq, rem) + tid;
            if (i < min(cg_block_row(blk + 1, bq, rem), n)) x[i] = axpy_e(alpha, pnew[i], x[i]);
        }
    if (tid == 0 && bid < nblk && apend) mbar_wait(&bar[seq & 1], (seq >> 1) & 1);  // drain the prefetch
    if (PROF && a.prof && tid == 0) {  // SM of every CTA (profiling: arrival spread by SM / die)
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.prof[19 * (size_t)G + bid] = smid;
    }
    if (bid == 0 && tid == 0) {
        c->rz = rz;
        c->beta = beta;
        if (PROF)
            for (int k = 0; k < 4; ++k) c->tphase[k] = tp[k];
        c->tphase[4] = G;
    }
}

// ---------------------------------------------------------------- single-sync persistent CG
// The same CG with ONE grid barrier per iteration.  Phase j (one SpMV) no longer waits
// for the update of iteration j-1: every gathered column re-evaluates that update on the
// fly from the previous phase's vectors,
//     r_j = r_{j-1} - alpha_{j-1} q_{j-1},  z_j = M r_j,  p_j = z_j + beta_{j-1} p_{j-1},
// with the reference's rounding of each step (axpy; vmul; scal then axpy), so every
// element of r, z, p, q and x is bitwise what the two-barrier loop stores.  The CTA
// owning row i stores r_j, p_j, q_j = (A p_j)_i and x_j = x_{j-1} + alpha_{j-1} p_{j-1}
// (x lags one phase), into the other buffer of each ping-pong pair (r: r | z, q: q | q1,
// p: p0 | p1), so no CTA overwrites a value another CTA still gathers.  The barrier of
// phase j reduces five partials: p_j.q_j (alpha_j), r_j.r_j (the criteria of iteration
// j, exact), r_j.z_j (rz_j, exact) and z_j.q_j, q_j.M q_j, from which
//     rz_{j+1} = sum M (r_j - alpha_j q_j)^2 = rz_j - 2 alpha_j z_j.q_j + alpha_j^2 q_j.M q_j
// gives beta_j before r_{j+1} exists (no orthogonality is assumed: the identity is exact,
// only its rounding differs from the direct dot, by a few ulps of rz_j; rz_{j+1} itself
// is recomputed exactly at the next barrier for alpha_{j+1} and the breakdown test).
// Per iteration: A + 9 V n bytes (gathered r, q, p, M; own x read; r, p, q, x stored)
// instead of A + 12 V n, and one barrier instead of two.  The stop decision of iteration
// j is taken after phase j, so the last phase's p, q are computed and discarded.
// Stage of the single-sync kernel: the block's matrix ranges (StreamLayout) followed by
// five own-row vector ranges [r0, r1) -- r_{j-1}, p_{j-1}, q_{j-1}, M, x -- all moved by
// TMA one block ahead, so the own-row update never waits on global memory.
template <class V, class I>
struct Cg1Layout {
    StreamLayout<V, I> L;
    int cap_x;  // elements per vector range (R rows + alignment slack)
    __host__ __device__ Cg1Layout(int R, int nnz_cap) : L(R, nnz_cap) { cap_x = (R + 2 * (16 / (int)sizeof(V)) + 3) & ~3; }
    __host__ __device__ size_t vec_bytes() const { return ((size_t)cap_x * sizeof(V) + 15) & ~size_t(15); }
    __host__ __device__ size_t off_x(int k) const { return L.stage_bytes() + (size_t)k * vec_bytes(); }
    __host__ __device__ size_t stage_bytes() const { return off_x(5); }
};

template <class V, class I, int R, int MB>
__global__ void __launch_bounds__(R, MB) cg1_persistent_kernel(CgPArgs a) {
    // gathered out-of-block columns in flight per thread (four loads each)
    constexpr int kGU = 4;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ StreamMeta meta[2];
    __shared__ int64_t vbase[2];
    Ctl *c = a.ctl;
    if (c->done) return;  // setup found the exact solution
    const I *rp = (const I *)a.rp, *ci = (const I *)a.ci;
    const V *val = (const V *)a.val, *inv = (const V *)a.inv;
    V *x = (V *)a.x;
    const int64_t n = a.n, nnz = a.nnz;
    const Cg1Layout<V, I> CL(R, a.nnz_cap);
    const size_t sb = CL.stage_bytes();
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int64_t nblk = a.nblk, bq = a.bq, rem = a.rem;
    const int64_t bid = blockIdx.x;
    const uint64_t pol = policy_evict_first();
    unsigned long long *count = &c->barrier;
    unsigned long long epoch = 0;
    // row-pointer bounds of this CTA's kb blocks, loaded once (issue() then starts its
    // bulk copies without a dependent global load on the critical thread)
    int64_t *kbnd = reinterpret_cast<int64_t *>(smem + 2 * sb);
    for (int q = tid; q < a.kb; q += R) {
        const int64_t blk = bid + (int64_t)q * G;
        kbnd[2 * q] = rp[cg_block_row(blk, bq, rem)];
        kbnd[2 * q + 1] = rp[min(cg_block_row(blk + 1, bq, rem), n)];
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // stage block blk for phase jc into slot s (thread 0 only): matrix ranges + own-row
    // vectors of phase jc (phase 0: r_0 and z_0 = p_0; phase jc > 0: r, p, q of jc - 1)
    auto issue = [&](int64_t blk, int s, int64_t jc) {
        unsigned char *st = smem + s * sb;
        V *sv = reinterpret_cast<V *>(st);
        I *sc = reinterpret_cast<I *>(st + CL.L.off_c());
        I *sr = reinterpret_cast<I *>(st + CL.L.off_r());
        const int64_t r0 = cg_block_row(blk, bq, rem), r1 = min(cg_block_row(blk + 1, bq, rem), n);
        const int64_t q = (blk - bid) / G;
        const int64_t k0 = kbnd[2 * q], k1 = kbnd[2 * q + 1];
        StreamMeta m;
        m.r0 = r0;
        m.r1 = r1;
        uint32_t bv = stage_range(val, k0, k1, nnz, sv, m.av);
        uint32_t bc = stage_range(ci, k0, k1, nnz, sc, m.ac);
        uint32_t br = stage_range(rp, r0, r1 + 1, n + 1, sr, m.ar);
        const bool odd = jc & 1;
        const V *src[5] = {(const V *)(jc == 0 ? a.r : odd ? a.r : a.z),
                           (const V *)(jc == 0 ? a.z : odd ? a.p0 : a.p1),
                           jc == 0 ? nullptr : (const V *)(odd ? a.q : a.q1), inv, x};
        uint32_t bx[5];
        int64_t base = r0;
#pragma unroll
        for (int k = 0; k < 5; ++k)
            bx[k] = src[k] ? stage_range(src[k], r0, r1, n, reinterpret_cast<V *>(st + CL.off_x(k)), base) : 0;
        meta[s] = m;
        vbase[s] = base;
        mbar_arrive_expect_tx(&bar[s], bv + bc + br + bx[0] + bx[1] + bx[2] + bx[3] + bx[4]);
        if (bv) bulk_g2s(sv, val + m.av, bv, &bar[s], pol);
        if (bc) bulk_g2s(sc, ci + m.ac, bc, &bar[s], pol);
        if (br) bulk_g2s(sr, rp + m.ar, br, &bar[s], pol);
#pragma unroll
        for (int k = 0; k < 5; ++k)
            if (bx[k]) bulk_g2s(reinterpret_cast<V *>(st + CL.off_x(k)), src[k] + base, bx[k], &bar[s]);
    };
    uint32_t seq = 0;
    if (tid == 0 && bid < nblk) issue(bid, 0, 0);

    const int64_t it0 = c->iter;
    double rz = c->rz, alpha = 0.0, beta = 0.0;
    bool bad_beta = false;  // rz_{j+1} expansion not finite: stop at the next barrier
    const double bnorm = c->bnorm;
    for (int64_t j = 0;; ++j) {
        const bool first = j == 0;
        const bool odd = j & 1;  // phase j writes buffer j & 1, reads the other
        // r_0 in r; z holds z_0 for phase 0, then the odd r's
        const V *rin = (const V *)(odd ? a.r : a.z), *qin = (const V *)(odd ? a.q : a.q1),
                *pin = (const V *)(first ? a.z : odd ? a.p0 : a.p1);
        V *rout = (V *)(odd ? a.z : a.r), *qout = (V *)(odd ? a.q1 : a.q), *pout = (V *)(odd ? a.p1 : a.p0);
        double part[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // p.q, r.r, r.z, z.q, q.Mq
        for (int64_t blk = bid; blk < nblk; blk += G, ++seq) {
            const int s = seq & 1;
            const bool wrap = blk + G >= nblk;  // next: this phase's next block or the next phase's first
            // (a CTA owning one block stages its next-phase copy only after writing it)
            const bool defer = wrap && blk == bid;
            if (tid == 0 && !defer) issue(wrap ? bid : blk + G, s ^ 1, wrap ? j + 1 : j);
            mbar_wait(&bar[s], (seq >> 1) & 1);
            unsigned char *st = smem + s * sb;
            const V *sv = reinterpret_cast<const V *>(st);
            const I *sc = reinterpret_cast<const I *>(st + CL.L.off_c());
            const I *sr = reinterpret_cast<const I *>(st + CL.L.off_r());
            V *s_r = reinterpret_cast<V *>(st + CL.off_x(0));  // r_{j-1}, then z_j
            V *s_p = reinterpret_cast<V *>(st + CL.off_x(1));  // p_{j-1}, then p_j
            const V *s_q = reinterpret_cast<const V *>(st + CL.off_x(2));
            const V *s_m = reinterpret_cast<const V *>(st + CL.off_x(3));
            const V *s_x = reinterpret_cast<const V *>(st + CL.off_x(4));
            const StreamMeta m = meta[s];
            const int64_t vb = vbase[s];
            const int64_t i = m.r0 + tid;
            const int64_t nr = m.r1 - m.r0;
            const bool own = i < m.r1;
            const int64_t t = i - vb;
            // own rows: r_j, z_j, p_j, x_j from the staged vectors; p_j replaces p_{j-1} in
            // the stage (in-block gathers read it there), z_j replaces r_{j-1}
            if (own) {
                V ri, zi, pi;
                if (first) {
                    ri = s_r[t];
                    zi = s_p[t];
                    pi = zi;
                } else {
                    const V pp = s_p[t];
                    ri = axpy_e(-alpha, s_q[t], s_r[t]);
                    zi = inv ? vmul(ri, s_m[t]) : ri;
                    pi = axpy_e(1.0, zi, scal_e(beta, pp));
                    x[i] = axpy_e(alpha, pp, s_x[t]);
                    rout[i] = ri;
                }
                pout[i] = pi;
                s_p[t] = pi;
                s_r[t] = zi;
                part[1] = addd(part[1], mulp(ri, ri));
                part[2] = addd(part[2], mulp(ri, zi));
            }
            __syncthreads();
            if (own) {
                const int64_t kb = sr[i - m.ar], ke = sr[i + 1 - m.ar];
                double acc = 0.0;
                for (int64_t k = kb; k < ke; k += kGU) {
                    V vv[kGU], bb[kGU];
#pragma unroll
                    for (int u = 0; u < kGU; ++u) {
                        const int64_t kk = k + u < ke ? k + u : ke - 1;
                        const int64_t col = (int64_t)sc[kk - m.ac];
                        vv[u] = sv[kk - m.av];
                        const uint64_t off = (uint64_t)(col - m.r0);
                        if (off < (uint64_t)nr) {
                            bb[u] = s_p[col - vb];
                        } else if (first) {
                            bb[u] = pin[col];
                        } else {  // p_j re-evaluated at an out-of-block column
                            const V rc = axpy_e(-alpha, qin[col], rin[col]);
                            const V zc = inv ? vmul(rc, inv[col]) : rc;
                            bb[u] = axpy_e(1.0, zc, scal_e(beta, pin[col]));
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kGU; ++u)
                        if (k + u < ke) acc = addd(acc, mulp(vv[u], bb[u]));
                }
                const V qi = (V)acc;
                qout[i] = qi;
                const double di = inv ? (double)s_m[t] : 1.0;
                part[0] = addd(part[0], mulp(s_p[t], qi));
                part[3] = addd(part[3], __dmul_rn((double)s_r[t], (double)qi));
                part[4] = addd(part[4], __dmul_rn(__dmul_rn((double)qi, di), (double)qi));
            }
            // the next phase stages r, p, q, x by TMA (async proxy): order this thread's
            // generic stores before it, then release the stage
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncthreads();
            if (tid == 0 && defer) issue(bid, s ^ 1, j + 1);
        }
        double tot[5];
        // partial slots ping-pong by epoch: a CTA that is one barrier ahead never
        // overwrites the slots another CTA is still summing
        ++epoch;
        grid_allreduce<5, R>(part, a.partials + (epoch & 1) * 5 * G, count, epoch * G, tot);
        const int64_t it = it0 + j;  // iterations completed: x_j, r_j
        if (!first) {  // end of iteration j (solvers.py:207-216): criteria on ||r_j||
            const double rnorm = sqrt(tot[1]);
            int reason = check_criteria(c, it, rnorm, bnorm);
            if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
            if (bid == 0 && tid == 0) {
                c->rnorm = rnorm;
                record(c, it, rnorm);
            }
            if (reason != STOP_NONE) {
                if (bid == 0 && tid == 0) finish_with(c, it, reason);
                break;
            }
            if (!isfinite(tot[2]) || rz == 0.0 || bad_beta) {  // rz_new (solvers.py:217-222)
                if (bid == 0 && tid == 0) breakdown(c, it);
                break;
            }
            rz = tot[2];
        }
        // iteration j + 1 (solvers.py:202-206): alpha from p_j.q_j
        const double pq = tot[0];
        if (!isfinite(pq) || pq <= kBreakdownRtol * fabs(rz)) {
            if (bid == 0 && tid == 0) breakdown(c, it + 1);
            break;
        }
        alpha = rz / pq;
        const double rz_next = rz - 2.0 * alpha * tot[3] + alpha * alpha * tot[4];
        beta = rz_next / rz;
        bad_beta = !isfinite(beta);  // (the phase still runs; its barrier reports the breakdown)
    }
    if (tid == 0 && bid < nblk) mbar_wait(&bar[seq & 1], (seq >> 1) & 1);  // drain the prefetch
    if (bid == 0 && tid == 0) {
        c->rz = rz;
        c->beta = beta;
        c->tphase[4] = G;
    }
}

// max stored entries of any block of the balanced partition (the stage capacity)
template <class I>
__global__ void cg_block_nnz_max_kernel(const I *rp, int64_t n, int64_t nblk, int64_t bq, int64_t rem, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblk; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = (int64_t)rp[min(cg_block_row(b + 1, bq, rem), n)] - (int64_t)rp[min(cg_block_row(b, bq, rem), n)];
        m = k > (int64_t)m ? (unsigned long long)k : m;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// Launch the persistent loop if the matrix is a stream-kernel CSR whose R-row block
// stage fits, and the grid can be co-resident (cooperative launch); false = not
// applicable (the caller runs the graph loop).  The rows are cut into nblk = kb * G
// balanced blocks (<= R rows each, whole 32-row units), so every CTA owns exactly kb blocks.
static thread_local int g_cg_last_rows = 0;  // block rows of the last persistent launch

static std::atomic<int> g_cg_xw{[] {
    const char *e = getenv("SPARSEB200_CG_XW");
    return e ? atoi(e) : 1;
}()};

template <class V, class I, int R>
bool cg_persistent_launch_r(const sb_matrix &M, const CgPArgs &proto, bool single, cudaStream_t st, cudaError_t &err) {
    err = cudaSuccess;
    sb_csr A;
    if (M.format == SB_FMT_CSR) {
        A = *(const sb_csr *)M.mat;
    } else if (M.format == SB_FMT_COO) {  // row-pointer-indexed COO: the same CSR arrays
        const sb_coo &C = *(const sb_coo *)M.mat;
        if (!C.plan || !C.plan->row_ptrs || !C.plan->csr_plan) return false;
        A = sb_csr{C.rows, C.cols, C.nnz, C.plan->row_ptrs, C.col_idxs, C.values, C.plan->csr_plan};
    } else {
        return false;
    }
    if (!A.plan || A.plan->kernel != SB_CSR_STREAM || A.rows == 0) return false;
    // single-sync kernel: CTAs per SM from SPARSEB200_CG1_MB (threads per SM = MB R)
    static const int mb_env = getenv("SPARSEB200_CG1_MB") ? atoi(getenv("SPARSEB200_CG1_MB")) : 0;
    const int mb = (mb_env == 3 || mb_env == 4 ? mb_env : 3) * 256 / R;  // 3: 80 registers, 3 stages of 68 KB
    const int sms = device_info().sms;
    const int per_sm = single ? mb : 1024 / R;
    int64_t grid = (int64_t)per_sm * sms;
    const int64_t nb_min = ceil_div(A.rows, R);
    if (grid > nb_min) grid = nb_min;
    if (grid > kMaxGrid) grid = kMaxGrid;
    const int64_t kb = ceil_div(nb_min, grid);
    const int64_t nblk = kb * grid;
    if (nblk > ceil_div(A.rows, 32)) return false;  // tiny systems: fewer units than blocks
    // stage capacity of the balanced blocks (one pass over nblk row pointers)
    unsigned long long *dmax = &proto.ctl->tphase[9];
    if ((err = cudaMemsetAsync(dmax, 0, sizeof(*dmax), st)) != cudaSuccess) return false;
    cg_block_nnz_max_kernel<I><<<(unsigned)std::min<int64_t>(ceil_div(nblk, 256), 1024), 256, 0, st>>>(
        (const I *)A.row_ptrs, A.rows, nblk, ceil_div(A.rows, 32) / nblk, ceil_div(A.rows, 32) % nblk, dmax);
    unsigned long long hmax = 0;
    if ((err = cudaMemcpyAsync(&hmax, dmax, sizeof(hmax), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (err = cudaStreamSynchronize(st)) != cudaSuccess)
        return false;
    if (hmax > (1u << 20)) return false;
    const int cap = (int)((hmax + 63) & ~63ull);
    const size_t smem = single ? 2 * Cg1Layout<V, I>(R, cap > 0 ? cap : 64).stage_bytes() + 16 * kb
                               : 2 * StreamLayout<V, I>(R, cap > 0 ? cap : 64).stage_bytes() + 16 * kb;
    if (smem > 220 * 1024) return false;
    // staged update phase when one block's five operand ranges fit half a stage
    static const int bt_env = getenv("SPARSEB200_CG_BT") ? atoi(getenv("SPARSEB200_CG_BT")) : 1;
    const size_t sb_cap = StreamLayout<V, I>(R, cap > 0 ? cap : 64).stage_bytes();
    const bool bt = bt_env && !proto.xa && 5 * (((size_t)R * sizeof(V) + 15) & ~size_t(15)) <= ((sb_cap / 2) & ~size_t(15));
    // x update in the barrier waits (staged update phase only; sb_set_cg_xw(0) /
    // SPARSEB200_CG_XW=0 turns it off: 128^3 68.4-68.9 -> 66.3-66.9 us per iteration)
    const bool xw = bt && g_cg_xw.load() != 0;
    auto kern = !single ? (proto.prof ? (xw ? cg_persistent_kernel<V, I, R, true, true, true>
                                        : bt ? cg_persistent_kernel<V, I, R, true, true>
                                             : cg_persistent_kernel<V, I, R, true>)
                           : xw ? cg_persistent_kernel<V, I, R, false, true, true>
                           : bt ? cg_persistent_kernel<V, I, R, false, true>
                                : cg_persistent_kernel<V, I, R, false>)
                : mb * R == 768 ? cg1_persistent_kernel<V, I, R, 768 / R> : cg1_persistent_kernel<V, I, R, 1024 / R>;
    ensure_max_smem((const void *)kern);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, R, smem) != cudaSuccess || occ < per_sm) {
        cudaGetLastError();
        return false;
    }
    CgPArgs args = proto;
    args.n = A.rows;
    args.nnz = A.nnz;
    args.rp = A.row_ptrs;
    args.ci = A.col_idxs;
    args.val = A.values;
    args.nnz_cap = cap > 0 ? cap : 64;
    args.nblk = nblk;
    args.bq = ceil_div(A.rows, 32) / nblk;
    args.rem = ceil_div(A.rows, 32) % nblk;
    args.kb = (int)kb;
    void *params[] = {&args};
    err = cudaLaunchCooperativeKernel((const void *)kern, dim3((unsigned)grid), dim3(R), params, smem, st);
    if (err != cudaSuccess) {
        cudaGetLastError();
        err = cudaSuccess;
        return false;  // not co-resident here: graph loop instead
    }
    g_cg_last_rows = R;
    return true;
}

template <class V, class I>
bool cg_persistent_launch(const sb_matrix &M, const CgPArgs &proto, cudaStream_t st, cudaError_t &err) {
    err = cudaSuccess;
    // Small systems (<= 2^20 rows): 512-row blocks (2 CTAs of 512 threads per SM: half the
    // barrier arrivals) where their stage fits; else 256 (cg_modes.py, us per iteration,
    // 256 -> 512 rows: 64^3 15.6 -> 14.5-14.8, 96^3 32.8 -> 32.0-32.3; 128^3 72.2 ->
    // 72.2-72.4 and bench.py 13.80k -> 13.62-13.74k iterations/s).  SPARSEB200_CG_R = 256 /
    // 512 forces one.  Measured and dropped (profiles/README.md, round 2): the residual
    // kept in shared memory (two CTAs per SM: 94 vs 73 us per iteration at 128^3 -- the
    // update pass needs the occupancy for its loads in flight), L2 eviction-priority hints
    // per vector, L2 prefetch of phase-B operands before barrier 1 / of further matrix
    // blocks before barrier 2, and walking the update blocks backwards: all flat or slower.
    static const int r_env = getenv("SPARSEB200_CG_R") ? atoi(getenv("SPARSEB200_CG_R")) : 0;
    const int64_t rows = M.format == SB_FMT_CSR ? ((const sb_csr *)M.mat)->rows
                                                : (M.format == SB_FMT_COO ? ((const sb_coo *)M.mat)->rows : 0);
    const int r = r_env ? r_env : (rows <= (int64_t(1) << 20) ? 512 : 256);
    const bool single = proto.q1 != nullptr;
    if (r == 512 && cg_persistent_launch_r<V, I, 512>(M, proto, single, st, err)) return true;
    if (err != cudaSuccess) return false;
    return cg_persistent_launch_r<V, I, 256>(M, proto, single, st, err);
}

// CG loop shape: 3 = persistent kernel where applicable (default), else the graph loop
// with the fused direction (1) or the three-kernel loop (0).  Measured per iteration on
// B200 (tools/cg_modes.py, fp64 Poisson, us): p=64 25.6 / 22.2 / 14.8, p=96 41.9 / 38.0 /
// 29.6, p=128 79.1 / 73.8 / 72.1, p=160 147 / 134 / 138, p=256 557 / 526 / 554 for
// modes 0 / 1 / 3: the persistent loop wins while its two grid barriers per iteration
// are a large share, the fused graph loop beyond ~24 MB per vector.
static std::atomic<int> g_cg_mode{[] {
    const char *e = getenv("SPARSEB200_CG_FUSED");
    return e ? atoi(e) : 3;
}()};
constexpr size_t kPersistentMaxVectorBytes = 64u << 20;  // round 2 (staged update phase): 160^3 130.9 vs 134, 192^3 222.9 vs 227.5, 256^3 543 vs 544, 320^3 1080 vs 1041 us per iteration (persistent vs graph)
// grid barriers per persistent CG iteration: 2 = the two-barrier kernel (default), 1 = the
// single-sync kernel (SPARSEB200_CG_SYNC=1; measured slower, profiles/README.md round 2)
static std::atomic<int> g_cg_sync{[] {
    const char *e = getenv("SPARSEB200_CG_SYNC");
    return e && atoi(e) == 1 ? 1 : 2;
}()};
static thread_local int g_cg_last_loop = -1;  // loop shape of this thread's last CG solve

// ---------------------------------------------------------------- CG with ILU / IC factors
// z = U^{-1} (L^{-1} r) between the update and the direction: the update kernel stops at
// the criteria (r.r), two triangular sweeps form z, a dot kernel forms r.z and beta
// (solvers.py:207-222 order: x, r, ||r|| check, z = M r, rz_new, beta, p).
template <class V>
struct CgInitNoZ : SkipNone {  // r = b - A x0; b.b, r.r (z follows from the sweeps)
    using value_type = V;
    const V *b, *t;
    V *r;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[2]) const {
        const auto B = ldp<W>(b, i), T = ldp<W>(t, i);
        Pk<V, W> R;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            R.v[w] = axpy_e(-1.0, T.v[w], B.v[w]);
            part[0] = addd(part[0], mulp(B.v[w], B.v[w]));
            part[1] = addd(part[1], mulp(R.v[w], R.v[w]));
        }
        stp<W>(r, i, R);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[2]) const {
        c->bnorm = sqrt(tot[0]);
        c->rnorm = sqrt(tot[1]);
        c->iter = 0;
        if (c->rnorm == 0.0) exact_log(c);
    }
};

template <class V, bool INIT>
struct CgRz : SkipNone {  // r.z -> rz (init: p = z) or beta (loop)
    using value_type = V;
    const V *r, *z;
    V *p;
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[1]) const {
        const auto R = ldp<W>(r, i), Z = ldp<W>(z, i);
#pragma unroll
        for (int w = 0; w < W; ++w) part[0] = addd(part[0], mulp(R.v[w], Z.v[w]));
        if (INIT) stp<W>(p, i, Z);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const {
        if (INIT) {
            c->rz = tot[0];
            return;
        }
        const double rz_new = tot[0];
        if (!isfinite(rz_new) || c->rz == 0.0) {
            breakdown(c, c->iter);
            return;
        }
        c->beta = rz_new / c->rz;
        c->rz = rz_new;
    }
};

template <class V>
struct CgUpdateNoZ : SkipNone {  // x += alpha p; r -= alpha q; r.r -> criteria
    using value_type = V;
    const V *p, *q;
    V *x, *r;
    double alpha;
    __device__ __forceinline__ void prepare(const Ctl *c) { alpha = c->alpha; }
    template <int W>
    __device__ __forceinline__ void elem(int64_t i, double (&part)[1]) const {
        const auto P = ldp<W>(p, i), Q = ldp<W>(q, i);
        auto X = ldp<W>(x, i), R = ldp<W>(r, i);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            X.v[w] = axpy_e(alpha, P.v[w], X.v[w]);
            R.v[w] = axpy_e(-alpha, Q.v[w], R.v[w]);
            part[0] = addd(part[0], mulp(R.v[w], R.v[w]));
        }
        stp<W>(x, i, X);
        stp<W>(r, i, R);
    }
    __device__ __forceinline__ void last(Ctl *c, const double (&tot)[1]) const {
        const int64_t it = c->iter;
        const double rnorm = sqrt(tot[0]);
        c->rnorm = rnorm;
        record(c, it, rnorm);
        int reason = check_criteria(c, it, rnorm, c->bnorm);
        if (reason == STOP_NONE && rnorm == 0.0) reason = STOP_RESIDUAL;
        if (reason != STOP_NONE) finish_with(c, it, reason);
    }
};

// validate both factors once (the reference raises at the first apply)
template <class V, class I>
sb_status tri_precond_check(const sb_tri_precond &m, sb_error *err, cudaStream_t st);

template <class V, class I>
sb_status cg_solve_tri(const SolveArgs &a) {
    sb_error *err = a.err;
    int64_t n = 0;
    sb_status s = check_solve_args<V>(a, n);
    if (s != SB_OK) return s;
    const sb_tri_precond m = *a.tri;
    s = tri_precond_check<V, I>(m, err, a.st);
    if (s != SB_OK) return s;
    const int64_t cap = a.log->history_cap;
    SolverWs w = carve_ws(a.ws, SB_SOLVER_CG, sizeof(V), n, 0, cap);
    V *r = ws_vec<V>(w, 0), *z = ws_vec<V>(w, 1), *p = ws_vec<V>(w, 2), *q = ws_vec<V>(w, 3),
      *t = ws_vec<V>(w, 4);
    const V *b = (const V *)a.b->data;
    V *x = (V *)a.x->data;
    Ctl *ctl = w.ctl;
    double *part = w.partials;
    const sb_matrix M = *a.A;
    const TriWs tw = carve_tri_ws(m.workspace, n);
    Ctl h = initial_ctl(*a.crit, w, cap);
    auto precond = [=](const V *in, cudaStream_t st) -> cudaError_t {  // z = U^{-1} L^{-1} in
        cudaError_t e = launch_trsv<V, I>(*m.l, true, m.l_unit != 0, in, 1, t, 1, tw, ctl, TRI_SKIP_DONE, st);
        if (e != cudaSuccess) return e;
        return launch_trsv<V, I>(*m.u, false, false, t, 1, z, 1, tw, ctl, TRI_SKIP_DONE, st);
    };
    LoopSpec spec;
    spec.key = "cgtri" + std::to_string(sizeof(V)) + std::to_string(sizeof(I)) + "|" + matrix_key(M) +
               ptr_key({b, x, a.ws, w.vecs, w.hist, m.l->row_ptrs, m.l->values, m.u->row_ptrs, m.u->values,
                        m.workspace}) + std::to_string(m.l_unit);
    spec.poll_chunk = 8;
    spec.setup = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(M, x, 1, t, 1, EpiStore<V>{t, 1}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<2>(n, ctl, part, CgInitNoZ<V>{{}, b, t, r}, st);
        if (e != cudaSuccess) return e;
        e = precond(r, st);
        if (e != cudaSuccess) return e;
        return launch_ew<1>(n, ctl, part, CgRz<V, true>{{}, r, z, p}, st);
    };
    spec.body = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(
            M, p, 1, q, 1, EpiSolver<V, 1, CgPqFin>{q, p, nullptr, ctl, part, CgPqFin{}}, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<1>(n, ctl, part, CgUpdateNoZ<V>{{}, p, q, x, r, 0.0}, st);
        if (e != cudaSuccess) return e;
        e = precond(r, st);
        if (e != cudaSuccess) return e;
        e = launch_ew<1>(n, ctl, part, CgRz<V, false>{{}, r, z, nullptr}, st);
        if (e != cudaSuccess) return e;
        return launch_ew<0>(n, ctl, part, CgDirection<V>{{}, z, p, 0.0}, st);
    };
    s = run_loop(spec, ctl, h, a.st, err);
    if (s != SB_OK) return s;
    return finish_log(h, a, w);
}

template <class V, class I>
sb_status cg_solve(const SolveArgs &a) {
    if (a.tri) return cg_solve_tri<V, I>(a);
    sb_error *err = a.err;
    int64_t n = 0;
    sb_status s = check_solve_args<V>(a, n);
    if (s != SB_OK) return s;
    const int64_t cap = a.log->history_cap;
    SolverWs w = carve_ws(a.ws, SB_SOLVER_CG, sizeof(V), n, 0, cap);
    V *r = ws_vec<V>(w, 0), *z = ws_vec<V>(w, 1), *p = ws_vec<V>(w, 2), *q = ws_vec<V>(w, 3),
      *t = ws_vec<V>(w, 4), *q1 = ws_vec<V>(w, 5);
    const V *b = (const V *)a.b->data, *inv = (const V *)a.inv;
    V *x = (V *)a.x->data;
    Ctl *ctl = w.ctl;
    double *part = w.partials;
    const sb_matrix M = *a.A;
    Ctl h = initial_ctl(*a.crit, w, cap);
    const int mode = g_cg_mode.load();
    const bool fused = mode != 0 && matrix_row_owning(M);
    auto setup = [=](cudaStream_t st) -> cudaError_t {
        cudaError_t e = matrix_apply<V, I>(M, x, 1, t, 1, EpiStore<V>{t, 1}, st);
        if (e != cudaSuccess) return e;
        return launch_ew<3>(n, ctl, part, CgInit<V>{{}, b, t, inv, r, z, fused ? nullptr : p}, st);
    };
    static const size_t pmax = getenv("SPARSEB200_CG_PMAX_MB") ? (size_t)atoll(getenv("SPARSEB200_CG_PMAX_MB")) << 20
                                                                 : kPersistentMaxVectorBytes;
    if (mode == 3 && fused && (size_t)n * sizeof(V) <= pmax) {
        // one cooperative launch runs every iteration; p ping-pongs between p and t
        h.cond = 0ull;
        SB_CUDA(cudaMemcpyAsync(ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, a.st));
        SB_CUDA(setup(a.st));
        CgPArgs pa = {};
        pa.inv = inv;
        pa.x = x;
        pa.r = r;
        pa.z = z;
        pa.p0 = p;
        pa.p1 = t;
        pa.q = q;
        pa.ctl = ctl;
        pa.partials = part;
        static const bool prof = getenv("SPARSEB200_CG_PROFILE") != nullptr;
        pa.prof = prof ? reinterpret_cast<unsigned long long *>(part + 4096) : nullptr;  // G <= 1000
        static const int pf = getenv("SPARSEB200_CG_PF") ? atoi(getenv("SPARSEB200_CG_PF")) : 1;
        pa.pf = pf;
        pa.q1 = g_cg_sync.load() == 1 ? q1 : nullptr;  // single-sync kernel (opt-in)
        static const int xa = getenv("SPARSEB200_CG_XA") ? atoi(getenv("SPARSEB200_CG_XA")) : 0;  // 128^3: 75.8 vs 73.1 us, off
        pa.xa = xa;
        cudaError_t le;
        if (cg_persistent_launch<V, I>(M, pa, a.st, le)) {
            g_cg_last_loop = 3;
            SB_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, a.st));
            SB_CUDA(cudaStreamSynchronize(a.st));
            if (prof && h.iter > 0 && pa.q1)
                fprintf(stderr, "[sparseb200] single-sync persistent CG %lld it: phase %.2f | barrier %.2f us/it\n",
                        (long long)h.iter, h.tphase[0] * 1e-3 / h.iter, h.tphase[1] * 1e-3 / h.iter);
            else if (prof && h.iter > 0)
                fprintf(stderr, "[sparseb200] persistent CG %lld it: A %.2f | bar1 %.2f | B %.2f | bar2 %.2f us/it\n",
                        (long long)h.iter, h.tphase[0] * 1e-3 / h.iter, h.tphase[1] * 1e-3 / h.iter,
                        h.tphase[2] * 1e-3 / h.iter, h.tphase[3] * 1e-3 / h.iter);
            if (prof && h.iter > 14 && !pa.q1) {  // per barrier: arrival spread, CTA-0 wait, wake-up
                const int G = (int)h.tphase[4];
                std::vector<unsigned long long> st(20 * (size_t)G);
                SB_CUDA(cudaMemcpy(st.data(), pa.prof, st.size() * 8, cudaMemcpyDeviceToHost));
                if (const char *dump = getenv("SPARSEB200_CG_PROFILE_DUMP")) {  // raw stamps
                    if (FILE *f = fopen(dump, "wb")) {
                        fwrite(st.data(), 8, st.size(), f);
                        fclose(f);
                    }
                }
                for (int e = 0; e < 18 && 10 + e <= 2 * h.iter; ++e) {
                    unsigned long long lo = ~0ull, hi = 0;
                    int slow = 0;
                    for (int i = 0; i < G; ++i) {
                        const unsigned long long t = st[(size_t)e * G + i];
                        if (t < lo) lo = t;
                        if (t > hi) { hi = t; slow = i; }
                    }
                    fprintf(stderr, "[sparseb200]   barrier %d: spread %.2f us (slowest CTA %d), CTA0 waits %.2f, wake %.2f\n",
                            10 + e, (hi - lo) * 1e-3, slow, (hi - st[(size_t)e * G]) * 1e-3,
                            ((long long)st[18 * (size_t)G + e] - (long long)hi) * 1e-3);
                }
            }
            return finish_log(h, a, w);
        }
        SB_CUDA(le);
        // not applicable: fall through to the graph loop (setup is re-run by run_loop)
    }
    LoopSpec spec;
    spec.key = "cg" + std::to_string(sizeof(V)) + std::to_string(sizeof(I)) + "|" + matrix_key(M) +
               ptr_key({a.inv, b, x, a.ws, w.vecs, w.hist, w.small});
    spec.poll_chunk = 8;
    spec.hot_base = r;  // r, z, p, q, t are contiguous in the workspace
    spec.hot_bytes = 5 * w.vec_bytes;
    spec.setup = setup;
    if (fused) {
        // p ping-pongs between p (buf 0) and t (buf 1; free once setup consumed A x0);
        // one body = an odd and an even iteration, so the buffer roles stay fixed
        spec.key += "|fused";
        spec.poll_chunk = 4;
        spec.body = [=](cudaStream_t st) -> cudaError_t {
            for (int h = 0; h < 2; ++h) {
                V *pold = h == 0 ? p : t, *pnew = h == 0 ? t : p;
                cudaError_t e = matrix_apply<V, I>(
                    M, pold, 1, q, 1, EpiCgFused<V>{q, pnew, z, pold, ctl, part, 0.0, 0}, st);
                if (e != cudaSuccess) return e;
                e = launch_ew<2>(n, ctl, part, CgUpdate<V>{{}, pnew, q, inv, x, r, z, 0.0}, st);
                if (e != cudaSuccess) return e;
            }
            return cudaSuccess;
        };
    } else {
        spec.body = [=](cudaStream_t st) -> cudaError_t {
            cudaError_t e = matrix_apply<V, I>(
                M, p, 1, q, 1, EpiSolver<V, 1, CgPqFin>{q, p, nullptr, ctl, part, CgPqFin{}}, st);
            if (e != cudaSuccess) return e;
            e = launch_ew<2>(n, ctl, part, CgUpdate<V>{{}, p, q, inv, x, r, z, 0.0}, st);
            if (e != cudaSuccess) return e;
            return launch_ew<0>(n, ctl, part, CgDirection<V>{{}, z, p, 0.0}, st);
        };
    }
    g_cg_last_loop = fused ? 1 : 0;
    s = run_loop(spec, ctl, h, a.st, err);
    if (s != SB_OK) return s;
    return finish_log(h, a, w);
}


}  // namespace sb

using namespace sb;

extern "C" {

void sb_set_cg_fused(int mode) { g_cg_mode = mode; }
void sb_set_cg_sync(int barriers) { g_cg_sync = barriers == 1 ? 1 : 2; }
void sb_set_cg_xw(int on) { g_cg_xw = on ? 1 : 0; }
int sb_cg_last_loop(void) { return g_cg_last_loop; }
int sb_cg_last_block_rows(void) { return g_cg_last_loop == 3 ? g_cg_last_rows : 0; }

#define SB_DEFS(V, VN, I, IN) \
    sb_status sb_cg_solve_##VN##_##IN(const sb_matrix *a, const void *inv_diag,                    \
                                      const sb_dense *b, sb_dense *x, const sb_criteria *crit,     \
                                      void *workspace, sb_log *log, sb_stream_t stream,            \
                                      sb_error *err) {                                             \
        SB_GUARD_BEGIN                                                                             \
        return cg_solve<V, I>(SolveArgs{a, inv_diag, b, x, crit, 0, workspace, log,                \
                                        as_stream(stream), err});                                  \
        SB_GUARD_END                                                                               \
    }

#define SB_TRI_DEFS(V, VN, I, IN)                                                                  \
    sb_status sb_cg_solve_tri_##VN##_##IN(const sb_matrix *a, const sb_tri_precond *m,              \
                                          const sb_dense *b, sb_dense *x, const sb_criteria *crit,  \
                                          void *workspace, sb_log *log, sb_stream_t stream,         \
                                          sb_error *err) {                                          \
        SB_GUARD_BEGIN                                                                              \
        if (!m || !m->l || !m->u || !m->workspace)                                                  \
            return fail(err, SB_ERR_INVALID_ARGUMENT, "triangular preconditioner: null argument");  \
        SolveArgs sa{a, nullptr, b, x, crit, 0, workspace, log, as_stream(stream), err};            \
        sa.tri = m;                                                                                 \
        return cg_solve<V, I>(sa);                                                                  \
        SB_GUARD_END                                                                                \
    }
SB_TRI_DEFS(float, float, int32_t, i32)
SB_TRI_DEFS(float, float, int64_t, i64)
SB_TRI_DEFS(double, double, int32_t, i32)
SB_TRI_DEFS(double, double, int64_t, i64)

SB_DEFS(float, float, int32_t, i32)
SB_DEFS(float, float, int64_t, i64)
SB_DEFS(double, double, int32_t, i32)
SB_DEFS(double, double, int64_t, i64)

}  // extern "C"
