// tmagather.cu -- can TMA bulk copies (cp.async.bulk, one 256-byte row per
// lane) gather K1's rows faster than register-staged 16-byte loads?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmagather tools/tmagather.cu && build/tmagather
//
// Same random 256-byte-row index streams as tools/l2bw.cu (48 / 96 / 612 MB
// working sets).  ldg: 16 lanes per row, 8 rows in flight per lane group (the
// K1 scheme).  tma<W,S>: W warps per CTA, each with an S-stage smem ring of
// 32 rows; lane t bulk-copies row idx[k+t] into slot t, completion on the
// stage's mbarrier; the warp sums the rows from shared memory (lane = column).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

__global__ void ldg_gather(const double2* __restrict__ rows, const int* __restrict__ idx, size_t nidx,
                           double* sink) {
    const int lane = threadIdx.x & 31, lg = lane & 15, grp = lane >> 4;
    const size_t warp = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const size_t nwarps = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
    double2 acc = make_double2(0.0, 0.0);
    size_t base = warp * 16;
    int nj = base + grp * 8 + (lg & 7) < nidx ? __ldg(idx + base + grp * 8 + (lg & 7)) : 0;
    for (; base < nidx; base += nwarps * 16) {
        const int j = nj;
        const size_t nb = base + nwarps * 16 + grp * 8 + (lg & 7);
        nj = nb < nidx ? __ldg(idx + nb) : 0;
        double2 v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int jt = __shfl_sync(0xffffffffu, j, grp * 16 + t);
            v[t] = __ldg(rows + static_cast<size_t>(jt) * 16 + lg);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            acc.x += v[t].x;
            acc.y += v[t].y;
        }
    }
    if (acc.x == 12345.678) sink[0] = acc.y;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <int W, int S>
__global__ void __launch_bounds__(W * 32, 1) tma_gather(const double* __restrict__ rows, const int* __restrict__ idx,
                                                       size_t nidx, double* sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[W][S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* ring = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp) * S * 32 * 32;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const size_t gw = static_cast<size_t>(blockIdx.x) * W + warp;
    const size_t nw = static_cast<size_t>(gridDim.x) * W;
    const size_t nbatch = (nidx + 31) / 32;
    auto issue = [&](size_t k, int s) {
        const size_t bi = gw + k * nw;
        if (bi >= nbatch) return;
        const size_t pos = bi * 32 + lane;
        const int nv = static_cast<int>((nidx - bi * 32) < 32 ? (nidx - bi * 32) : 32);
        if (lane == 0) mbar_expect(&bars[warp][s], nv * 256u);
        __syncwarp();
        if (lane < nv) {
            const int j = __ldg(idx + pos);
            bulk_g2s(ring + (static_cast<size_t>(s) * 32 + lane) * 32, rows + static_cast<size_t>(j) * 32, 256u,
                     &bars[warp][s]);
        }
    };
    for (int s = 0; s < S; ++s) issue(s, s);
    double acc = 0.0;
    for (size_t k = 0;; ++k) {
        const size_t bi = gw + k * nw;
        if (bi >= nbatch) break;
        const int s = static_cast<int>(k % S);
        mbar_wait(&bars[warp][s], static_cast<uint32_t>((k / S) & 1));
        const int nv = static_cast<int>((nidx - bi * 32) < 32 ? (nidx - bi * 32) : 32);
        const double* st = ring + static_cast<size_t>(s) * 32 * 32;
#pragma unroll 8
        for (int t = 0; t < nv; ++t) acc += st[t * 32 + lane];
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + S, s);
    }
    if (acc == 12345.678) sink[0] = acc;
}

// Mixed: warps < NL gather with 16-byte LDGs (K1 scheme), the others with
// per-row TMA bulk copies into a 1-stage smem ring; all pull 512-row batches
// from one atomic queue, so the two paths run concurrently to the end.
template <int NW, int NL>
__global__ void __launch_bounds__(NW * 32, 1) mixed_gather(const double* __restrict__ rows, const int* __restrict__ idx,
                                                          size_t nidx, int* queue, double* sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[NW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr size_t kBatch = 512;
    const size_t nbatch = (nidx + kBatch - 1) / kBatch;
    double acc = 0.0;
    if (warp < NL) {
        const int lg = lane & 15, grp = lane >> 4;
        const double2* r2 = reinterpret_cast<const double2*>(rows);
        double2 a2 = make_double2(0.0, 0.0);
        while (true) {
            int bi = 0;
            if (lane == 0) bi = atomicAdd(queue, 1);
            bi = __shfl_sync(0xffffffffu, bi, 0);
            if (static_cast<size_t>(bi) >= nbatch) break;
            const size_t b0 = static_cast<size_t>(bi) * kBatch;
            const size_t b1 = b0 + kBatch < nidx ? b0 + kBatch : nidx;
            for (size_t base = b0; base < b1; base += 16) {
                const size_t k = base + grp * 8 + (lg & 7);
                const int j = k < b1 ? __ldg(idx + k) : 0;
                double2 v[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int jt = __shfl_sync(0xffffffffu, j, grp * 16 + t);
                    v[t] = __ldg(r2 + static_cast<size_t>(jt) * 16 + lg);
                }
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    a2.x += v[t].x;
                    a2.y += v[t].y;
                }
            }
        }
        acc = a2.x + a2.y;
    } else {
        double* ring = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp - NL) * 32 * 32;
        if (lane == 0) mbar_init(&bars[warp], 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        uint32_t phase = 0;
        while (true) {
            int bi = 0;
            if (lane == 0) bi = atomicAdd(queue, 1);
            bi = __shfl_sync(0xffffffffu, bi, 0);
            if (static_cast<size_t>(bi) >= nbatch) break;
            const size_t b0 = static_cast<size_t>(bi) * kBatch;
            const size_t b1 = b0 + kBatch < nidx ? b0 + kBatch : nidx;
            for (size_t base = b0; base < b1; base += 32) {
                const int nv = static_cast<int>(b1 - base < 32 ? b1 - base : 32);
                if (lane == 0) mbar_expect(&bars[warp], nv * 256u);
                __syncwarp();
                if (lane < nv)
                    bulk_g2s(ring + static_cast<size_t>(lane) * 32, rows + static_cast<size_t>(__ldg(idx + base + lane)) * 32,
                             256u, &bars[warp]);
                mbar_wait(&bars[warp], phase);
                phase ^= 1;
                for (int t = 0; t < nv; ++t) acc += ring[t * 32 + lane];
                __syncwarp();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
        }
    }
    if (acc == 12345.678) sink[0] = acc;
}

template <int NW, int NL>
float run_mixed(const double* rows, const int* idx, size_t nidx, double* sink, int sms) {
    const size_t smem = static_cast<size_t>(NW - NL) * 32 * 256 + 16;
    cudaFuncSetAttribute(mixed_gather<NW, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int* q;
    cudaMalloc(&q, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemset(q, 0, 4);
    mixed_gather<NW, NL><<<sms, NW * 32, smem>>>(rows, idx, nidx, q, sink);
    cudaMemset(q, 0, 4);
    cudaEventRecord(e0);
    mixed_gather<NW, NL><<<sms, NW * 32, smem>>>(rows, idx, nidx, q, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        exit(1);
    }
    cudaFree(q);
    return ms;
}

template <int W, int S>
float run_tma(const double* rows, const int* idx, size_t nidx, double* sink, int sms) {
    const size_t smem = static_cast<size_t>(W) * S * 32 * 256;
    cudaFuncSetAttribute(tma_gather<W, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    tma_gather<W, S><<<sms, W * 32, smem>>>(rows, idx, nidx, sink);
    cudaEventRecord(e0);
    tma_gather<W, S><<<sms, W * 32, smem>>>(rows, idx, nidx, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        exit(1);
    }
    return ms;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t ws_mb[] = {48, 96, 612};
    printf("[");
    for (int si = 0; si < 3; ++si) {
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
        ldg_gather<<<sms * 5, 256>>>(reinterpret_cast<const double2*>(rows), idx, nidx, sink);
        cudaEventRecord(e0);
        ldg_gather<<<sms * 5, 256>>>(reinterpret_cast<const double2*>(rows), idx, nidx, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s{\"working_set_mb\": %zu, \"ldg_tbs\": %.2f", si ? ",\n " : "", ws_mb[si], gb / ms);
        printf(", \"tma_w8_s3\": %.2f", gb / run_tma<8, 3>(rows, idx, nidx, sink, sms));
        printf(", \"tma_w4_s6\": %.2f", gb / run_tma<4, 6>(rows, idx, nidx, sink, sms));
        printf(", \"tma_w12_s2\": %.2f", gb / run_tma<12, 2>(rows, idx, nidx, sink, sms));
        printf(", \"tma_w16_s1\": %.2f", gb / run_tma<16, 1>(rows, idx, nidx, sink, sms));
        printf(", \"tma_w6_s4\": %.2f", gb / run_tma<6, 4>(rows, idx, nidx, sink, sms));
        printf(", \"mixed_32w_ldg32\": %.2f", gb / run_mixed<32, 32>(rows, idx, nidx, sink, sms));
        printf(", \"mixed_32w_ldg24_tma8\": %.2f", gb / run_mixed<32, 24>(rows, idx, nidx, sink, sms));
        printf(", \"mixed_32w_ldg16_tma16\": %.2f", gb / run_mixed<32, 16>(rows, idx, nidx, sink, sms));
        printf(", \"mixed_32w_ldg28_tma4\": %.2f}", gb / run_mixed<32, 28>(rows, idx, nidx, sink, sms));
        fflush(stdout);
        cudaFree(rows);
        cudaFree(idx);
    }
    printf("]\n");
    return 0;
}
