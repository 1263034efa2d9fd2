// solver_runtime.cu -- the CUDA-graph WHILE loop runner shared by every solver, the
// graph-cache keys, and the library-level solver entry points.
#include <algorithm>
#include <atomic>
#include <cmath>

#include "solver_common.cuh"

namespace sb {

// ================================================================ loop runner
static std::atomic<int> g_graph_mode{1};
bool graph_mode_enabled() { return g_graph_mode.load() != 0; }

// programmatic dependent launch between consecutive solver kernels: opt-in
// (SPARSEB200_PDL=1).  Measured on B200 (128^3 CG, graph loop): 81 -> 90 us per
// iteration for the three-kernel loop, 74.9 -> 76.3 us for the fused loop, so it is
// off by default; switched off for good if a graph with programmatic edges fails.
static std::atomic<int> g_pdl{[] {
    const char *e = getenv("SPARSEB200_PDL");
    return (e && e[0] == '1') ? 1 : 0;
}()};
bool pdl_enabled() { return g_pdl.load() != 0; }

struct GraphEntry {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle handle = 0;
};

static std::mutex g_cache_mu;
static std::map<std::string, GraphEntry> g_cache;

// Keep the Krylov work vectors resident in L2 while the matrix streams through it:
// an access-policy window (hits persist, misses stream) on the capture stream, which
// the captured kernel nodes inherit.  Size of the persisting carve-out from
// SPARSEB200_L2_PERSIST_MB (0 disables).
static void apply_l2_window(cudaStream_t cs, void *base, size_t bytes) {
    static const long mb = [] {
        const char *e = getenv("SPARSEB200_L2_PERSIST_MB");
        return e ? atol(e) : 0L;
    }();
    if (mb <= 0 || !base || !bytes) return;
    int dev = 0, max_persist = 0, max_window = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    size_t carve = std::min<size_t>((size_t)mb << 20, (size_t)max_persist);
    if (carve == 0 || max_window <= 0) return;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve);
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = base;
    v.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, (size_t)max_window);
    v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)carve / (float)v.accessPolicyWindow.num_bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(cs, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaGetLastError();
}

static cudaError_t build_while_graph(const LoopSpec &spec, GraphEntry &out) {
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaGraphCreate(&g, 0);
    if (e != cudaSuccess) return e;
    cudaGraphConditionalHandle h;
    e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        return e;
    }
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &np);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        return e;
    }
    cudaGraph_t body = np.conditional.phGraph_out[0];
    cudaStream_t cs;
    e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        return e;
    }
    apply_l2_window(cs, spec.hot_base, spec.hot_bytes);
    e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
        cudaError_t eb = spec.body(cs);
        cudaGraph_t captured = body;
        e = cudaStreamEndCapture(cs, &captured);
        if (eb != cudaSuccess) e = eb;
    }
    cudaStreamDestroy(cs);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&out.exec, g, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        cudaGetLastError();
        return e;
    }
    out.graph = g;
    out.handle = h;
    return cudaSuccess;
}

sb_status run_loop(const LoopSpec &spec, Ctl *dctl, Ctl &hctl, cudaStream_t st, sb_error *err) {
    GraphEntry entry;
    bool use_graph = graph_mode_enabled();
    if (use_graph) {
        int dev = 0;
        cudaGetDevice(&dev);
        const std::string key = std::to_string(dev) + "|" + spec.key;
        std::lock_guard<std::mutex> lock(g_cache_mu);
        auto it = g_cache.find(key);
        if (it == g_cache.end()) {
            GraphEntry fresh;
            cudaError_t e = build_while_graph(spec, fresh);
            if (e != cudaSuccess && pdl_enabled()) {
                fprintf(stderr, "[sparseb200] graph loop with programmatic launches failed (%s); "
                                "retrying without\n", cudaGetErrorString(e));
                g_pdl = 0;
                e = build_while_graph(spec, fresh);
            }
            if (e != cudaSuccess && spec.local_fallback) {
                // e.g. a collective that cannot be captured into a conditional body: poll
                // this loop, keep graphs for everything else
                fprintf(stderr, "[sparseb200] graph loop unavailable for this solve (%s); polling\n",
                        cudaGetErrorString(e));
                cudaGetLastError();
                use_graph = false;
            } else if (e != cudaSuccess) {
                // conditional nodes unavailable: fall back to host polling for good
                fprintf(stderr, "[sparseb200] graph loop unavailable (%s); using polled launches\n",
                        cudaGetErrorString(e));
                g_graph_mode = 0;
                use_graph = false;
            } else {
                if (g_cache.size() > 64) {  // bound the cache (distinct buffers per solve)
                    for (auto &kv : g_cache) {
                        cudaGraphExecDestroy(kv.second.exec);
                        cudaGraphDestroy(kv.second.graph);
                    }
                    g_cache.clear();
                }
                it = g_cache.emplace(key, fresh).first;
            }
        }
        if (use_graph) entry = it->second;
    }
    hctl.cond = 0ull;  // setup kernels run outside the graph: no handle yet
    SB_CUDA(cudaMemcpyAsync(dctl, &hctl, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    SB_CUDA(spec.setup(st));
    if (use_graph) {
        static thread_local unsigned long long handle_value;
        handle_value = (unsigned long long)entry.handle;
        SB_CUDA(cudaMemcpyAsync(&dctl->cond, &handle_value, sizeof(handle_value),
                                cudaMemcpyHostToDevice, st));
        SB_CUDA(cudaGraphLaunch(entry.exec, st));
    } else {
        static thread_local int *pinned = nullptr;
        static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
        if (!pinned) {
            SB_CUDA(cudaMallocHost(&pinned, 2 * sizeof(int)));
            SB_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
            SB_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        }
        const int chunk = spec.poll_chunk > 0 ? spec.poll_chunk : 8;
        for (int64_t k = 0;; ++k) {
            for (int c = 0; c < chunk; ++c) SB_CUDA(spec.body(st));
            SB_CUDA(cudaMemcpyAsync(&pinned[k & 1], &dctl->done, sizeof(int), cudaMemcpyDeviceToHost, st));
            SB_CUDA(cudaEventRecord(ev[k & 1], st));
            if (k >= 1) {
                SB_CUDA(cudaEventSynchronize(ev[(k - 1) & 1]));
                if (pinned[(k - 1) & 1]) break;
            }
        }
    }
    SB_CUDA(cudaMemcpyAsync(&hctl, dctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
    return SB_OK;
}

std::string ptr_key(std::initializer_list<const void *> ps) {
    std::string s;
    char buf[32];
    for (const void *p : ps) {
        snprintf(buf, sizeof(buf), "%p,", p);
        s += buf;
    }
    return s;
}

std::string matrix_key(const sb_matrix &M) {
    std::string s = std::to_string(M.format) + ":";
    switch (M.format) {
    case SB_FMT_CSR: {
        const sb_csr &A = *(const sb_csr *)M.mat;
        s += ptr_key({A.row_ptrs, A.col_idxs, A.values}) + std::to_string(A.rows) + "," +
             std::to_string(A.nnz);
        if (A.plan)
            s += "|" + std::to_string(A.plan->kernel) + "," + std::to_string(A.plan->block_rows) + "," +
                 std::to_string(A.plan->nnz_cap) + "," + std::to_string(A.plan->num_tiles) +
                 ptr_key({A.plan->tile_rows, A.plan->tile_nnz, A.plan->carry_rows, A.plan->carry_vals});
        break;
    }
    case SB_FMT_COO: {
        const sb_coo &A = *(const sb_coo *)M.mat;
        s += ptr_key({A.row_idxs, A.col_idxs, A.values}) + std::to_string(A.rows) + "," +
             std::to_string(A.nnz);
        if (A.plan) {
            s += ptr_key({A.plan->carry_rows, A.plan->carry_vals, A.plan->row_ptrs}) + std::to_string(A.plan->num_tiles);
            if (A.plan->csr_plan)
                s += "|" + std::to_string(A.plan->csr_plan->kernel) + "," + std::to_string(A.plan->csr_plan->block_rows) +
                     "," + std::to_string(A.plan->csr_plan->nnz_cap) +
                     ptr_key({A.plan->csr_plan->tile_rows, A.plan->csr_plan->carry_rows});
        }
        break;
    }
    case SB_FMT_ELL: {
        const sb_ell &A = *(const sb_ell *)M.mat;
        s += ptr_key({A.col_idxs, A.values}) + std::to_string(A.rows) + "," + std::to_string(A.width) +
             "," + std::to_string(A.stride);
        break;
    }
    case SB_FMT_SELLP: {
        const sb_sellp &A = *(const sb_sellp *)M.mat;
        // max_block_entries picks block vs chunk kernel and sets the staged capacity
        // baked into the captured launch, so it is part of the key
        s += ptr_key({A.slice_lengths, A.slice_sets, A.col_idxs, A.values, A.row_perm, A.piece_plan, A.carry}) +
             std::to_string(A.num_pieces) + "," + std::to_string(A.piece_entries) + "," + std::to_string(A.rows) +
             "," + std::to_string(A.slice_size) + "," + std::to_string(A.num_slices) + "," +
             std::to_string(A.max_block_entries);
        break;
    }
    case SB_FMT_HYBRID: {
        const sb_hybrid &A = *(const sb_hybrid *)M.mat;
        s += ptr_key({A.ell.col_idxs, A.ell.values, A.coo.row_idxs, A.coo.col_idxs, A.coo.values}) +
             std::to_string(A.ell.rows) + "," + std::to_string(A.ell.width) + "," +
             std::to_string(A.ell.stride) + "," + std::to_string(A.coo.nnz);
        if (A.coo.plan) s += ptr_key({A.coo.plan->carry_rows, A.coo.plan->carry_vals});
        break;
    }
    }
    return s;
}

}  // namespace sb

using namespace sb;

extern "C" {

void sb_set_graph_mode(int enabled) { g_graph_mode = enabled ? 1 : 0; }

size_t sb_solver_workspace_bytes(int32_t solver, int32_t value_bytes, int64_t n, int64_t krylov_dim,
                                 int64_t history_cap) {
    return solver_ws_bytes(solver, value_bytes, n, krylov_dim, history_cap);
}

}  // extern "C"
