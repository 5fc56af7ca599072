// driver.cuh -- host-side iteration driver shared by the CG and LRC solves.
// Launches one solver iteration after another and polls the device count of
// active columns `lag` iterations behind, so the GPU queue never drains.
#pragma once

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
template <class LaunchIter>
int run_iterations(SolveState& s, int64_t max_iter, int lag, cudaStream_t st,
                   LaunchIter&& launch_iter, int64_t* iters_run) {
    static thread_local PinnedRing ring;
    if (!ring.slots) return fail(KZ_ECUDA, "pinned host buffer allocation failed");
    constexpr int R = PinnedRing::kRing;
    cudaEvent_t ev[R];
    for (int i = 0; i < R; ++i) KZ_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    int rc = KZ_OK;
    int64_t k = 1;
    for (; k <= max_iter; ++k) {
        const int64_t j = k - 1 - lag;
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

}  // namespace kz
