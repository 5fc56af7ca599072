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

// ---- from_edges on the device (graph.py:111-148) ---------------------------
// Drop self-loops, symmetrise, deduplicate, sort columns within rows:
//   keys   k = min(u,v)*n + max(u,v) (self-loops -> sentinel n*n)
//   sort   radix sort of the undirected keys (only the ceil(log2(n*n+1))
//          significant bits), unique
//   expand every undirected key into its two directed keys lo*n+hi, hi*n+lo
//   sort   again; row offsets from the row boundaries of the sorted keys
// Everything is integer work: the result is the reference's CSR byte for byte.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

namespace {

__global__ void edge_keys_kernel(const int64_t* __restrict__ u, const int64_t* __restrict__ v, int64_t m,
                                 uint64_t n, uint64_t* __restrict__ keys, int32_t* __restrict__ bad) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t a = u[e], b = v[e];
        if (a < 0 || b < 0 || static_cast<uint64_t>(a) >= n || static_cast<uint64_t>(b) >= n) {
            *bad = 1;
            keys[e] = n * n;
            continue;
        }
        const uint64_t lo = static_cast<uint64_t>(a < b ? a : b), hi = static_cast<uint64_t>(a < b ? b : a);
        keys[e] = a == b ? n * n : lo * n + hi;
    }
}

__global__ void edge_expand_kernel(const uint64_t* __restrict__ uniq, const int64_t* __restrict__ nu, uint64_t n,
                                   uint64_t* __restrict__ out) {
    const int64_t cnt = *nu;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t k = uniq[i];
        if (k == n * n) {  // the sentinel sorts last: the expanded tail is a pair of sentinels
            out[2 * i] = n * n;
            out[2 * i + 1] = n * n;
            continue;
        }
        const uint64_t lo = k / n, hi = k - lo * n;
        out[2 * i] = lo * n + hi;
        out[2 * i + 1] = hi * n + lo;
    }
}

// src/col of the sorted directed keys; off[r] = first position of row r
__global__ void edge_csr_kernel(const uint64_t* __restrict__ keys, int64_t nnz, uint64_t n,
                                int64_t* __restrict__ off, int32_t* __restrict__ col, int32_t* __restrict__ src) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= nnz;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i < nnz ? static_cast<int64_t>(keys[i] / n) : static_cast<int64_t>(n);
        const int64_t rp = i > 0 ? static_cast<int64_t>(keys[i - 1] / n) : -1;
        for (int64_t q = rp + 1; q <= r; ++q) off[q] = i;  // rows rp+1 .. r start at i
        if (i < nnz) {
            col[i] = static_cast<int32_t>(keys[i] - static_cast<uint64_t>(r) * n);
            if (src) src[i] = static_cast<int32_t>(r);
        }
    }
}

struct EdgeWork {
    uint64_t *a, *b;
    int64_t* nsel;
    int32_t* bad;
    void* temp;
    size_t temp_bytes;
};

int carve_edges(int64_t n, int64_t m, void* ws, size_t ws_bytes, EdgeWork& w, size_t* need) {
    const int end_bit = 64 - __builtin_clzll(static_cast<unsigned long long>(n) * n + 1);
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, t1, static_cast<uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                   2 * m, 0, end_bit);
    cub::DeviceSelect::Unique(nullptr, t2, static_cast<uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                              static_cast<int64_t*>(nullptr), m);
    (void)t3;
    Carver cv(ws, ws_bytes);
    w.a = cv.take<uint64_t>(2 * static_cast<size_t>(m) + 1);
    w.b = cv.take<uint64_t>(2 * static_cast<size_t>(m) + 1);
    w.nsel = cv.take<int64_t>(1);
    w.bad = cv.take<int32_t>(1);
    w.temp_bytes = std::max(t1, t2);
    w.temp = cv.take<char>(w.temp_bytes);
    if (need) *need = cv.off + 256;
    return end_bit;
}

}  // namespace

extern "C" size_t kz_edges_to_csr_workspace_bytes(int64_t n, int64_t m) {
    if (n < 1 || m < 0) return 0;
    EdgeWork w;
    size_t need = 0;
    carve_edges(n, std::max<int64_t>(m, 1), nullptr, 0, w, &need);
    return need;
}

extern "C" int kz_edges_to_csr(int64_t n, int64_t m, const int64_t* u, const int64_t* v, int64_t* row_offsets,
                               int32_t* col, int32_t* src, int64_t* nnz_out, void* ws, size_t ws_bytes,
                               void* stream) {
    clear_error();
    if (n < 1 || m < 0 || n >= (int64_t(1) << 31) || !row_offsets || !col || !nnz_out || (m > 0 && (!u || !v)))
        return fail(KZ_EARG, "bad edge-list arguments");
    if (!ws || ws_bytes < kz_edges_to_csr_workspace_bytes(n, m)) return fail(KZ_EARG, "workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t mm = std::max<int64_t>(m, 1);
    EdgeWork w;
    const int end_bit = carve_edges(n, mm, ws, ws_bytes, w, nullptr);
    const uint64_t un = static_cast<uint64_t>(n);
    KZ_CUDA(cudaMemsetAsync(w.bad, 0, sizeof(int32_t), st));
    const unsigned g = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(8 * max_ctas_per_chunk(), (mm + 255) / 256)));
    int64_t uniq = 0;
    if (m > 0) {
        edge_keys_kernel<<<g, 256, 0, st>>>(u, v, m, un, w.a, w.bad);
        note_launch();
        KZ_LAUNCH_CHECK();
        size_t tb = w.temp_bytes;
        KZ_CUDA(cub::DeviceRadixSort::SortKeys(w.temp, tb, w.a, w.b, m, 0, end_bit, st));
        tb = w.temp_bytes;
        KZ_CUDA(cub::DeviceSelect::Unique(w.temp, tb, w.b, w.a, w.nsel, m, st));
        add_launches(8);
        int32_t bad = 0;
        KZ_CUDA(cudaMemcpyAsync(&uniq, w.nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaMemcpyAsync(&bad, w.bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
        if (bad) return fail(KZ_EARG, "edge endpoint out of range");
        edge_expand_kernel<<<g, 256, 0, st>>>(w.a, w.nsel, un, w.b);
        note_launch();
        KZ_LAUNCH_CHECK();
        tb = w.temp_bytes;
        KZ_CUDA(cub::DeviceRadixSort::SortKeys(w.temp, tb, w.b, w.a, 2 * uniq, 0, end_bit, st));
        add_launches(4);
        // the sentinel (self-loops) is the largest key: it is the last unique
        // one when present, and its two expanded copies sort last
        uint64_t last = 0;
        if (uniq > 0) {
            KZ_CUDA(cudaMemcpyAsync(&last, w.b + 2 * uniq - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
            KZ_CUDA(cudaStreamSynchronize(st));
        }
        if (uniq > 0 && last == un * un) --uniq;
    }
    const int64_t nnz = 2 * uniq;
    const unsigned g2 = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(8 * max_ctas_per_chunk(), (nnz + 256) / 256)));
    edge_csr_kernel<<<g2, 256, 0, st>>>(w.a, nnz, un, row_offsets, col, src);
    note_launch();
    KZ_LAUNCH_CHECK();
    *nnz_out = nnz;
    return KZ_OK;
}
