// dsmem_gather.cu -- can distributed shared memory carry part of K1's gathers?
//
// K1 is bound by the L2 -> SM fill path (~18 TB/s for L2-resident 256-byte row
// gathers, tools/l2bw.cu).  A hub slab held in the shared memory of a thread
// block cluster would serve its gathers over the SM-to-SM network instead.
// This measures, for clusters of 4 / 8 / 16 CTAs (one CTA per SM, SLAB_KB of
// rows each): random 256-byte row gathers (8 lanes x 32 bytes, 4 rows in
// flight per lane group, as K1) from (a) the cluster's shared memory only,
// (b) an L2-resident global buffer only, (c) a mix with `dsm_of4` of every 4
// slots served from the cluster -- is the sum faster than L2 alone?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dsmem_gather tools/dsmem_gather.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr int kRowBytes = 256;

__device__ __forceinline__ unsigned lcg(unsigned& s) {
    s = s * 1664525u + 1013904223u;
    return s >> 8;
}

// mode: number of the 4 slots per round that gather from the cluster (0: L2 only, 4: cluster only)
__global__ void __launch_bounds__(kThreads, 1)
    gather_kernel(const double2* __restrict__ grows, unsigned nrows_global, int slab_rows, int rounds, int dsm_of4,
                  double* sink) {
    extern __shared__ __align__(16) double2 slab[];  // [slab_rows][16] double2
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned csize = cluster.num_blocks();
    for (int i = threadIdx.x; i < slab_rows * 16; i += blockDim.x) slab[i] = make_double2(1.0, 2.0);
    cluster.sync();
    const int lane = threadIdx.x & 31, lg = lane & 7, grp = lane >> 3;
    unsigned seed = (blockIdx.x * kThreads + (threadIdx.x >> 3)) * 2654435761u + 12345u + grp;  // per lane group
    double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
    for (int r = 0; r < rounds; ++r) {
        double2 v[4][2];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const unsigned x = lcg(seed);
            if (t < dsm_of4) {
                const unsigned peer = x % csize;
                const unsigned row = (x >> 5) % static_cast<unsigned>(slab_rows);
                const double2* p = cluster.map_shared_rank(slab, peer) + row * 16 + lg * 2;
                v[t][0] = p[0];
                v[t][1] = p[1];
            } else {
                const double2* p = grows + static_cast<size_t>(x % nrows_global) * 16 + lg * 2;
                v[t][0] = __ldg(p);
                v[t][1] = __ldg(p + 1);
            }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            acc0.x += v[t][0].x;
            acc0.y += v[t][0].y;
            acc1.x += v[t][1].x;
            acc1.y += v[t][1].y;
        }
    }
    if (acc0.x + acc1.y == 12345.678) sink[0] = acc0.y + acc1.x;
    cluster.sync();
}

int main(int argc, char** argv) {
    const int slab_kb = argc > 1 ? std::atoi(argv[1]) : 96;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = static_cast<size_t>(slab_kb) << 10;
    const int slab_rows = static_cast<int>(smem / kRowBytes);
    cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const size_t gbytes = 48ull << 20;
    double2* grows;
    cudaMalloc(&grows, gbytes);
    cudaMemset(grows, 0, gbytes);
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int rounds = 4000;
    printf("{\"sms\": %d, \"slab_kb\": %d, \"runs\": [", sms, slab_kb);
    bool first = true;
    const int csizes[] = {1, 4, 8, 16};
    for (int ci = 0; ci < 4; ++ci) {
        const int cs = csizes[ci];
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(cs);
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, gather_kernel, &cfg) != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            continue;
        }
        const int grid = nclusters * cs;
        cfg.gridDim = dim3(grid);
        for (int dsm = 0; dsm <= 4; ++dsm) {
            if (cs == 1 && dsm != 0 && dsm != 4) continue;
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                cudaError_t e = cudaLaunchKernelEx(&cfg, gather_kernel, (const double2*)grows,
                                                   (unsigned)(gbytes / kRowBytes), slab_rows, rounds, dsm, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
                    best = -1.0f;
                    break;
                }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep > 0 && ms < best) best = ms;
            }
            const double bytes = double(grid) * (kThreads / 8) * rounds * 4.0 * kRowBytes;
            printf("%s{\"cluster\": %d, \"ctas\": %d, \"dsm_slots_of_4\": %d, \"ms\": %.3f, \"gathered_gbs\": %.1f, "
                   "\"dsm_gbs\": %.1f, \"l2_gbs\": %.1f}",
                   first ? "" : ", ", cs, grid, dsm, best, bytes / (best * 1e-3) / 1e9,
                   bytes * dsm / 4.0 / (best * 1e-3) / 1e9, bytes * (4 - dsm) / 4.0 / (best * 1e-3) / 1e9);
            first = false;
        }
    }
    printf("]}\n");
    return 0;
}
