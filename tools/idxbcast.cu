// idxbcast.cu -- does loading the neighbour indices as broadcast int4s (every
// lane of a row group reads the same 16 bytes) instead of one index per lane
// + shuffles speed up K1-style 256-byte row gathers (8 lanes x 32-byte loads,
// 4 groups per warp, 4 rows per group per round)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/idxbcast tools/idxbcast.cu && build/idxbcast
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// shuffle form (the shipped K1 scheme): lanes lg < 4 load one index each
template <int MODE>
__global__ void __launch_bounds__(256, 5) gath(const double* __restrict__ rows, const int* __restrict__ idx, size_t nidx,
                                               double* sink) {
    const int lane = threadIdx.x & 31, lg = lane & 7, grp = lane >> 3;
    const size_t warp = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const size_t nwarps = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
    double acc[4] = {0, 0, 0, 0};
    const double* Xl = rows + lg * 4;
    if (MODE == 0) {
        size_t base = warp * 16;
        int nj = base + grp * 4 + (lg & 3) < nidx ? __ldcs(idx + base + grp * 4 + (lg & 3)) : 0;
        for (; base < nidx; base += nwarps * 16) {
            const int j = nj;
            const size_t nb = base + nwarps * 16 + grp * 4 + (lg & 3);
            nj = nb < nidx ? __ldcs(idx + nb) : 0;
            double v[4][4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int jt = __shfl_sync(0xffffffffu, j, grp * 8 + t);
                ld4(Xl + static_cast<size_t>(jt) * 32, v[t]);
            }
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] += v[t][q];
        }
    } else {
        size_t base = warp * 16;
        int4 nj = base < nidx ? __ldcs(reinterpret_cast<const int4*>(idx + base + grp * 4)) : make_int4(0, 0, 0, 0);
        for (; base < nidx; base += nwarps * 16) {
            const int4 j = nj;
            const size_t nb = base + nwarps * 16;
            if (MODE == 1) nj = nb < nidx ? __ldcs(reinterpret_cast<const int4*>(idx + nb + grp * 4)) : make_int4(0, 0, 0, 0);
            double v[4][4];
            ld4(Xl + static_cast<size_t>(j.x) * 32, v[0]);
            ld4(Xl + static_cast<size_t>(j.y) * 32, v[1]);
            ld4(Xl + static_cast<size_t>(j.z) * 32, v[2]);
            ld4(Xl + static_cast<size_t>(j.w) * 32, v[3]);
            if (MODE == 2) nj = nb < nidx ? __ldcs(reinterpret_cast<const int4*>(idx + nb + grp * 4)) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] += v[t][q];
        }
    }
    if (acc[0] == 12345.678) sink[0] = acc[1] + acc[2] + acc[3];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t ws_mb[] = {48, 612};
    printf("[");
    for (int si = 0; si < 2; ++si) {
        const size_t nrows = (ws_mb[si] << 20) / 256;
        double* rows;
        cudaMalloc(&rows, nrows * 256);
        cudaMemset(rows, 0, nrows * 256);
        const size_t nidx = 64ull << 20;
        std::vector<int> h(nidx);
        unsigned long long s = 88172645463325252ull;
        for (size_t i = 0; i < nidx; ++i) {
            s ^= s << 13;
            s ^= s >> 7;
            s ^= s << 17;
            h[i] = static_cast<int>(s % nrows);
        }
        int* idx;
        cudaMalloc(&idx, nidx * 4);
        cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
        const double gb = nidx * 256.0 / 1e9;
        float ms[3];
        for (int rep = 0; rep < 2; ++rep)
            for (int m = 0; m < 3; ++m) {
                cudaEventRecord(e0);
                if (m == 0) gath<0><<<sms * 5, 256>>>(rows, idx, nidx, sink);
                if (m == 1) gath<1><<<sms * 5, 256>>>(rows, idx, nidx, sink);
                if (m == 2) gath<2><<<sms * 5, 256>>>(rows, idx, nidx, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms[m], e0, e1);
            }
        printf("%s{\"working_set_mb\": %zu, \"shfl_tbs\": %.2f, \"int4_prefetch_tbs\": %.2f, \"int4_late_tbs\": %.2f}",
               si ? ",\n " : "", ws_mb[si], gb / ms[0], gb / ms[1], gb / ms[2]);
        cudaFree(rows);
        cudaFree(idx);
    }
    printf("]\n");
    return 0;
}
