// dmma_rate.cu -- fp64 tensor-core issue rate by mma.sync shape on this GPU:
// m8n8k4 (what dense.cuh / lowrank.cuh use) against m16n8k4 / m16n8k8 /
// m16n8k16, register operands only (no memory traffic), 16 warps per SM with
// 4 independent accumulator chains each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dmma_rate tools/dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void __launch_bounds__(512, 1) rate_kernel(int iters, double* sink) {
    double c[4][4];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) b[i] = 0.5 + threadIdx.x * 1e-4 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            if constexpr (SHAPE == 0) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[ch][0]), "+d"(c[ch][1]) : "d"(a[ch]), "d"(b[ch]));
            } else if constexpr (SHAPE == 1) {
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c[ch][0]), "+d"(c[ch][1]), "+d"(c[ch][2]), "+d"(c[ch][3])
                             : "d"(a[ch]), "d"(a[ch + 4]), "d"(b[ch]));
            } else if constexpr (SHAPE == 2) {
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c[ch][0]), "+d"(c[ch][1]), "+d"(c[ch][2]), "+d"(c[ch][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[ch]), "d"(b[(ch + 1) & 3]));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c[ch][0]), "+d"(c[ch][1]), "+d"(c[ch][2]), "+d"(c[ch][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
            }
        }
    }
    double s = 0.0;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) s += c[i][j];
    if (s == 1234.5) sink[0] = s;
}

template <int SHAPE>
void run(const char* name, double flops_per_mma, int sms) {
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    rate_kernel<SHAPE><<<sms, 512>>>(100, sink);
    cudaEventRecord(e0);
    rate_kernel<SHAPE><<<sms, 512>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = double(sms) * 16 * 4 * iters;
    printf("{\"shape\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f, \"err\": \"%s\"}\n", name, ms,
           mmas * flops_per_mma / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("m8n8k4", 2.0 * 8 * 8 * 4, sms);
    run<1>("m16n8k4", 2.0 * 16 * 8 * 4, sms);
    run<2>("m16n8k8", 2.0 * 16 * 8 * 8, sms);
    run<3>("m16n8k16", 2.0 * 16 * 8 * 16, sms);
    return 0;
}
