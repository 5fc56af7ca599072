// l2bw.cu -- measured L2 read throughput of this GPU: the roofline of the K1
// gather (rows of an L2-resident block read with 16-byte loads, like K1's).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/l2bw tools/l2bw.cu && build/l2bw
//
// Every warp streams 16-byte loads over a buffer of `mb` MB (default 48 MB,
// well inside the 126 MB L2) many times; prints GB/s of bytes delivered to
// the SMs for a sweep of buffer sizes (the 4 GB case is HBM-bound) and, with
// random row order, for 256-byte rows gathered by index like K1 does.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

__global__ void stream_kernel(const double2* __restrict__ buf, size_t n16, int reps, double* sink) {
    double2 acc = make_double2(0.0, 0.0);
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
            const double2 v = __ldg(buf + i);
            acc.x += v.x;
            acc.y += v.y;
        }
    if (acc.x == 12345.678) sink[0] = acc.y;
}

// K1-like gather: 16 lanes read one 256-byte row chosen by idx; 8 rows in flight per lane group
__global__ void gather_kernel(const double2* __restrict__ rows, const int* __restrict__ idx, size_t nidx,
                              double* sink) {
    const int lane = threadIdx.x & 31, lg = lane & 15, grp = lane >> 4;
    const size_t warp = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const size_t nwarps = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
    double2 acc = make_double2(0.0, 0.0);
    for (size_t base = warp * 16; base < nidx; base += nwarps * 16) {
        double2 v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const size_t k = base + grp * 8 + t;
            const int j = k < nidx ? __ldg(idx + k) : 0;
            v[t] = __ldg(rows + static_cast<size_t>(j) * 16 + lg);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            acc.x += v[t].x;
            acc.y += v[t].y;
        }
    }
    if (acc.x == 12345.678) sink[0] = acc.y;
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{\"sms\": %d, \"stream\": [", sms);
    const size_t sizes_mb[] = {16, 48, 96, 4096};
    for (int si = 0; si < 4; ++si) {
        const size_t bytes = sizes_mb[si] << 20;
        double2* buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 0, bytes);
        const size_t n16 = bytes / 16;
        const int reps = static_cast<int>(std::max<size_t>(1, (64ull << 30) / bytes));
        const int grid = sms * 8;
        stream_kernel<<<grid, 256>>>(buf, n16, 1, sink);
        cudaEventRecord(e0);
        stream_kernel<<<grid, 256>>>(buf, n16, reps, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s{\"mb\": %zu, \"gbs\": %.1f}", si ? ", " : "", sizes_mb[si], bytes * double(reps) / (ms * 1e-3) / 1e9);
        cudaFree(buf);
    }
    printf("], \"gather256\": [");
    // rows: 256-byte rows, working set sizes; random indices
    const size_t ws_mb[] = {48, 96, 612};
    for (int si = 0; si < 3; ++si) {
        const size_t nrows = (ws_mb[si] << 20) / 256;
        double2* rows;
        cudaMalloc(&rows, nrows * 256);
        cudaMemset(rows, 0, nrows * 256);
        const size_t nidx = 64ull << 20;
        std::vector<int> h(nidx);
        unsigned long long s = 88172645463325252ull;
        for (size_t i = 0; i < nidx; ++i) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            h[i] = static_cast<int>(s % nrows);
        }
        int* idx;
        cudaMalloc(&idx, nidx * 4);
        cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
        const int grid = sms * 5;
        gather_kernel<<<grid, 256>>>(rows, idx, nidx, sink);
        cudaEventRecord(e0);
        gather_kernel<<<grid, 256>>>(rows, idx, nidx, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s{\"working_set_mb\": %zu, \"gathered_gbs\": %.1f}", si ? ", " : "", ws_mb[si],
               nidx * 256.0 / (ms * 1e-3) / 1e9);
        cudaFree(rows);
        cudaFree(idx);
    }
    printf("]}\n");
    return 0;
}
