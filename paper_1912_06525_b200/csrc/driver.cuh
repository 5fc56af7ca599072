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

// solves with at most this much per-iteration work ((nnz + n) * columns)
// replay a captured iteration graph (launch overhead dominates below it)
constexpr double kGraphWork = 2e9;
// Opt-in (KZ_GRAPHS=1): measured with tools/timeline.py, capture +
// instantiate costs 0.2-1.2 ms per solve while the loop's launch gaps are
// ~10 us per kernel, so at every BASELINE config the host-driven loop is as
// fast or faster (R-MAT 18, 64 queries: 3.37 vs 4.55 ms span).
inline bool graphs_enabled() {
    static const bool on = std::getenv("KZ_GRAPHS") != nullptr;
    return on;
}

struct MappedRing {
    static constexpr int kRing = 8;
    volatile int32_t* host = nullptr;  // [3*kRing]: n_active, err, iteration stamp
    int32_t* dev = nullptr;
    MappedRing() {
        void* h = nullptr;
        if (cudaHostAlloc(&h, sizeof(int32_t) * 3 * kRing, cudaHostAllocMapped) != cudaSuccess) return;
        void* d = nullptr;
        if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) {
            cudaFreeHost(h);
            return;
        }
        host = static_cast<volatile int32_t*>(h);
        dev = static_cast<int32_t*>(d);
    }
    ~MappedRing() {
        if (host) cudaFreeHost(const_cast<int32_t*>(host));
    }
};

static __global__ void iter_set_kernel(int32_t* iter_dev, int v) { *iter_dev = v; }

static __global__ void iter_tick_kernel(SolveState s, int32_t* ring, int nring) {
    const int k = *s.iter_dev;
    int32_t* slot = ring + 3 * (k % nring);
    slot[0] = *s.n_active;
    slot[1] = *s.err;
    __threadfence_system();
    reinterpret_cast<volatile int32_t*>(slot)[2] = k;
    *s.iter_dev = k + 1;
}

template <class LaunchIter>
int run_iterations_graph(SolveState& s, int64_t max_iter, int lag, cudaStream_t st, LaunchIter&& launch_iter,
                         int64_t* iters_run) {
    static thread_local MappedRing ring;
    if (!ring.host || !s.iter_dev) return run_iterations(s, max_iter, lag, st, launch_iter, iters_run);
    constexpr int R = MappedRing::kRing;
    for (int i = 0; i < 3 * R; ++i) ring.host[i] = -1;
    iter_set_kernel<<<1, 1, 0, st>>>(s.iter_dev, 1);
    KZ_LAUNCH_CHECK();
    note_launch();
    // capture one iteration (+ tick); kernels recorded during capture are
    // counted per replay instead
    const long long before = kz_launch_count();
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    KZ_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int rc = launch_iter(0);
    iter_tick_kernel<<<1, 1, 0, st>>>(s, ring.dev, R);
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    const long long per_iter = kz_launch_count() - before + 1;
    add_launches(-(per_iter - 1));
    if (rc || ce != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return rc ? rc : fail(KZ_ECUDA, std::string("graph capture failed: ") + cudaGetErrorString(ce));
    }
    if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
        cudaGraphDestroy(graph);
        cudaGetLastError();
        return run_iterations(s, max_iter, lag, st, launch_iter, iters_run);  // host-driven fallback
    }
    int64_t k = 1;
    for (; k <= max_iter; ++k) {
        const int64_t j = k - 1 - lag;
        if (j >= 1) {
            volatile int32_t* slot = ring.host + 3 * (j % R);
            long spins = 0;
            while (slot[2] != static_cast<int32_t>(j)) {
                if ((++spins & 0xffff) == 0) {
                    const cudaError_t q = cudaStreamQuery(st);
                    if (q != cudaSuccess && q != cudaErrorNotReady) {
                        rc = fail(KZ_ECUDA, std::string("solve stream failed: ") + cudaGetErrorString(q));
                        break;
                    }
                    if (q == cudaSuccess && slot[2] != static_cast<int32_t>(j)) {
                        rc = fail(KZ_ECUDA, "iteration stamp never arrived");
                        break;
                    }
                }
            }
            if (rc) break;
            if (slot[0] == 0 || slot[1] != 0) break;
        }
        if (cudaGraphLaunch(exec, st) != cudaSuccess) {
            rc = fail(KZ_ECUDA, "graph launch failed");
            break;
        }
        add_launches(per_iter);
    }
    cudaStreamSynchronize(st);
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (iters_run) *iters_run = k - 1;
    return rc;
}

}  // namespace kz
