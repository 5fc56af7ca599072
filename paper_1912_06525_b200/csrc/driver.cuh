// driver.cuh -- host-side iteration driver shared by the CG and LRC solves.
// Launches one solver iteration after another and polls the device count of
// active columns `lag` iterations behind, so the GPU queue never drains.
#pragma once

#include <cstdlib>

#include "blockops.cuh"

namespace kz {

struct PinnedRing {
    int32_t* slots = nullptr;  // [2*kRing]: n_active, err
    static constexpr int kRing = 8;
    PinnedRing() { cudaHostAlloc(&slots, sizeof(int32_t) * 2 * kRing, cudaHostAllocDefault); }
    ~PinnedRing() {
        if (slots) cudaFreeHost(slots);
    }
};

// The shared iteration driver; also used by the LRC Schur solve in lrc.cu
// through a callback that launches one iteration.
// sync_k > 1: iteration sync_k is launched only after iteration sync_k - 1
// has reported (no speculation there) -- for an iteration whose launch
// itself costs block passes even when every column has already stopped
// (the residual-history fold).
template <class LaunchIter>
int run_iterations(SolveState& s, int64_t max_iter, int lag, cudaStream_t st,
                   LaunchIter&& launch_iter, int64_t* iters_run, int64_t sync_k = 0) {
    static thread_local PinnedRing ring;
    if (!ring.slots) return fail(KZ_ECUDA, "pinned host buffer allocation failed");
    constexpr int R = PinnedRing::kRing;
    // host-driven: kernels take the iteration number from their launch
    // arguments, never from the (unmaintained) device counter
    struct Restore {
        SolveState& s;
        int32_t* saved;
        ~Restore() { s.iter_dev = saved; }
    } restore{s, s.iter_dev};
    s.iter_dev = nullptr;
    cudaEvent_t ev[R];
    for (int i = 0; i < R; ++i) KZ_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    int rc = KZ_OK;
    int64_t k = 1;
    for (; k <= max_iter; ++k) {
        const int64_t j = (k == sync_k && lag > 0) ? k - 1 : k - 1 - lag;
        if (j >= 1) {
            if (cudaEventSynchronize(ev[j % R]) != cudaSuccess) {
                rc = fail(KZ_ECUDA, "event sync failed");
                break;
            }
            if (ring.slots[2 * (j % R)] == 0 || ring.slots[2 * (j % R) + 1] != 0) break;
        }
        rc = launch_iter(static_cast<int>(k));
        if (rc) break;
        int32_t* slot = ring.slots + 2 * (k % R);
        if (cudaMemcpyAsync(slot, s.n_active, sizeof(int32_t), cudaMemcpyDeviceToHost, st) ||
            cudaMemcpyAsync(slot + 1, s.err, sizeof(int32_t), cudaMemcpyDeviceToHost, st) ||
            cudaEventRecord(ev[k % R], st)) {
            rc = fail(KZ_ECUDA, "poll copy failed");
            break;
        }
    }
    cudaStreamSynchronize(st);
    for (int i = 0; i < R; ++i) cudaEventDestroy(ev[i]);
    if (iters_run) *iters_run = k - 1;
    return rc;
}

// ---- graph-replayed iteration loop -----------------------------------------
// One solver iteration is captured once into a CUDA graph together with a
// one-thread "tick" kernel that publishes (n_active, err, k) into a mapped
// pinned ring and advances the device iteration counter; the host then
// replays the graph once per iteration and polls the ring `lag` iterations
// behind -- one API call per iteration instead of ~3 launches + 2 copies +
// an event.  Kernels of the loop read the iteration number from
// SolveState::iter_dev (cur_iter), so the captured parameters stay valid.

// Graph capture is impossible on the legacy default stream (torch's default
// current stream): a solve handed that stream runs on a thread-local
// non-blocking side stream ordered after it by events, and the caller's
// stream waits for the side stream when the scope ends.
struct StreamScope {
    cudaStream_t user = nullptr, st = nullptr;
    cudaEvent_t ev = nullptr;
    explicit StreamScope(cudaStream_t u) : user(u), st(u) {
        if (u != nullptr && u != cudaStreamLegacy) return;
        static thread_local cudaStream_t side = nullptr;
        if (!side && cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) side = nullptr;
        if (!side || cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return;
        cudaEventRecord(ev, u);
        cudaStreamWaitEvent(side, ev, 0);
        st = side;
    }
    ~StreamScope() {
        if (st == user) return;
        cudaEventRecord(ev, st);
        cudaStreamWaitEvent(user, ev, 0);
        cudaEventDestroy(ev);
    }
};

// ---- device-driven iteration loop (CUDA graph with a conditional WHILE node) ----
// One solver iteration is captured once into the body of a WHILE node whose
// condition a one-thread tick kernel sets from the device state (columns
// still active, no error, iteration budget left) and which advances the
// device iteration counter; kernels of the loop read the iteration number
// from SolveState::iter_dev (cur_iter).  The instantiated graph is cached per
// thread, keyed by everything the captured kernels see (operator handle id,
// workspace, batch width, beta, tol, max_iter), so a repeated solve costs one
// graph launch for the whole loop: no per-iteration host work or polling.
// Used for solves whose per-iteration work is small (launch-bound: cfg1,
// cfg2); KZ_GRAPHS=0 turns it off, KZ_GRAPHS=1 forces it on.
// per-iteration work ((entries + rows) * columns) up to which a loop runs as
// a graph: CG iterations above ~5e7 take >= ~100 us of device time, where the
// host-driven residual-history loop (6 block passes, sparse first iteration)
// wins over the graph's direction form (cfg2: 2.2 vs 3.7 ms)
constexpr double kGraphWorkCg = 5e7;
constexpr double kGraphWorkLrc = 2e9;
inline int graphs_mode() {
    static const int m = [] {
        const char* e = std::getenv("KZ_GRAPHS");
        return e ? (e[0] == '0' ? 0 : 1) : -1;  // -1: by size
    }();
    return m;
}
inline bool use_graph_loop(double work, double limit) {
    const int m = graphs_mode();
    return m == 1 || (m == -1 && work <= limit);
}

struct GraphKey {
    uint64_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool operator==(const GraphKey& o) const {
        for (int i = 0; i < 8; ++i)
            if (v[i] != o.v[i]) return false;
        return true;
    }
};

static __global__ void iter_set_kernel(int32_t* iter_dev, int v) { *iter_dev = v; }

static __global__ void cond_tick_kernel(SolveState s, cudaGraphConditionalHandle h) {
    const int k = *s.iter_dev;  // the iteration that just ran
    const bool go = *s.n_active > 0 && *s.err == 0 && k < s.max_iter;
    *s.iter_dev = k + 1;
    cudaGraphSetConditional(h, go ? 1u : 0u);
}

struct GraphCache {
    static constexpr int kN = 8;
    struct Entry {
        GraphKey key;
        int dev = -1;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        long long per_iter = 0;
    } e[kN];
    int next = 0;
    ~GraphCache() {
        for (auto& x : e) {
            if (x.exec) cudaGraphExecDestroy(x.exec);
            if (x.graph) cudaGraphDestroy(x.graph);
        }
    }
};

// Runs the whole loop on the device; *per_iter_out = kernels per iteration
// (the caller adds per_iter * iterations to the launch count once it knows
// the iterations).
template <class LaunchIter>
int run_iterations_graph(SolveState& s, cudaStream_t st, LaunchIter&& launch_iter, const GraphKey& key,
                         long long* per_iter_out) {
    static thread_local GraphCache cache;
    if (!s.iter_dev) return fail(KZ_EARG, "graph loop needs the device iteration counter");
    int dev = 0;
    KZ_CUDA(cudaGetDevice(&dev));
    GraphCache::Entry* hit = nullptr;
    for (auto& x : cache.e)
        if (x.exec && x.dev == dev && x.key == key) hit = &x;
    if (!hit) {
        GraphCache::Entry& x = cache.e[cache.next];
        cache.next = (cache.next + 1) % GraphCache::kN;
        if (x.exec) cudaGraphExecDestroy(x.exec);
        if (x.graph) cudaGraphDestroy(x.graph);
        x = GraphCache::Entry();
        KZ_CUDA(cudaGraphCreate(&x.graph, 0));
        cudaGraphConditionalHandle h;
        KZ_CUDA(cudaGraphConditionalHandleCreate(&h, x.graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams p = {};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        KZ_CUDA(cudaGraphAddNode(&node, x.graph, nullptr, 0, &p));
        cudaGraph_t body = p.conditional.phGraph_out[0];
        KZ_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        const long long before = kz_launch_count();
        const int rc = launch_iter(0);
        cond_tick_kernel<<<1, 1, 0, st>>>(s, h);
        x.per_iter = kz_launch_count() - before + 1;
        add_launches(-(x.per_iter - 1));  // captured, not launched: counted per replay
        const cudaError_t ce = cudaStreamEndCapture(st, &body);
        if (rc || ce != cudaSuccess) {
            cudaGraphDestroy(x.graph);
            x = GraphCache::Entry();
            cudaGetLastError();
            return rc ? rc : fail(KZ_ECUDA, std::string("graph capture failed: ") + cudaGetErrorString(ce));
        }
        const cudaError_t ie = cudaGraphInstantiate(&x.exec, x.graph, 0);
        if (ie != cudaSuccess) {
            cudaGraphDestroy(x.graph);
            x = GraphCache::Entry();
            cudaGetLastError();
            return fail(KZ_ECUDA, std::string("graph instantiate failed: ") + cudaGetErrorString(ie));
        }
        x.key = key;
        x.dev = dev;
        hit = &x;
    }
    iter_set_kernel<<<1, 1, 0, st>>>(s.iter_dev, 1);
    note_launch();
    KZ_LAUNCH_CHECK();
    KZ_CUDA(cudaGraphLaunch(hit->exec, st));
    if (per_iter_out) *per_iter_out = hit->per_iter;
    return KZ_OK;
}

}  // namespace kz
