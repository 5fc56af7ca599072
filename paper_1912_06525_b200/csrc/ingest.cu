// ingest.cu -- graph ingestion on the device: connected components.
//
// Replaces the BFS of connected_components (graph.py:211-229) used by
// largest_connected_component (graph.py:232-261).  Hook + pointer jumping:
// every edge hooks the larger of its two roots under the smaller one with
// atomicMin, then every node jumps to its root; repeat until no hook
// changes anything.  Parent pointers only ever decrease, so the final root
// of a component is its smallest node id -- exactly the label order the
// reference's BFS produces (components numbered by their smallest node), so
// the reference's tie rule ("largest, then the one holding the smallest
// id") is a plain argmax over (size, -label) on the host.
#include <algorithm>

#include "common.cuh"

using namespace kz;

namespace {

__device__ __forceinline__ int32_t find_root(const int32_t* parent, int32_t x) {
    int32_t p = parent[x];
    while (p != x) {
        x = p;
        p = parent[x];
    }
    return x;
}

__global__ void cc_init(int32_t* parent, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        parent[i] = static_cast<int32_t>(i);
}

__global__ void cc_hook(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t nnz,
                        int32_t* parent, int32_t* changed) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t ru = find_root(parent, src[e]);
        const int32_t rv = find_root(parent, dst[e]);
        if (ru != rv) {
            const int32_t hi = max(ru, rv), lo = min(ru, rv);
            if (atomicMin(parent + hi, lo) > lo) *changed = 1;
        }
    }
}

__global__ void cc_jump(int32_t* parent, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        parent[i] = find_root(parent, static_cast<int32_t>(i));
}

}  // namespace

// labels[i] = smallest node id of i's component.  src/dst: device int32[nnz]
// edge endpoints (any orientation, duplicates allowed); labels: device int32[n].
extern "C" int kz_connected_components(int64_t n, int64_t nnz, const int32_t* src, const int32_t* dst,
                                       int32_t* labels, void* stream) {
    clear_error();
    if (n < 1 || nnz < 0 || !labels || (nnz > 0 && (!src || !dst)) || n >= (int64_t(1) << 31))
        return fail(KZ_EARG, "bad connected-components arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t* changed = nullptr;
    int32_t* hchanged = nullptr;
    KZ_CUDA(cudaMalloc(&changed, sizeof(int32_t)));
    KZ_CUDA(cudaHostAlloc(&hchanged, sizeof(int32_t), cudaHostAllocDefault));
    const unsigned gn = static_cast<unsigned>(std::min<int64_t>(4 * max_ctas_per_chunk(), (n + 255) / 256));
    const unsigned ge = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(8 * max_ctas_per_chunk(), (nnz + 255) / 256)));
    cc_init<<<gn, 256, 0, st>>>(labels, n);
    note_launch();
    int rc = KZ_OK;
    for (int it = 0; it < 64; ++it) {
        if (cudaMemsetAsync(changed, 0, sizeof(int32_t), st) != cudaSuccess) { rc = fail(KZ_ECUDA, "memset"); break; }
        if (nnz > 0) {
            cc_hook<<<ge, 256, 0, st>>>(src, dst, nnz, labels, changed);
            note_launch();
        }
        cc_jump<<<gn, 256, 0, st>>>(labels, n);
        note_launch();
        if (cudaMemcpyAsync(hchanged, changed, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            rc = fail(KZ_ECUDA, std::string("components: ") + cudaGetErrorString(cudaGetLastError()));
            break;
        }
        if (!*hchanged) break;
        if (it == 63) rc = fail(KZ_ECUDA, "components did not converge");
    }
    cudaFree(changed);
    cudaFreeHost(hchanged);
    return rc;
}
