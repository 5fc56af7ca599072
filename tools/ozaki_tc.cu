// ozaki_tc.cu -- fp64-accurate tall-skinny GEMM C = A Y (A: n x 128, Y: 128 x b)
// on the int8 tcgen05 tensor cores by Ozaki splitting, checked against a
// host fp64 product and timed at the headline shape (n = 2.39 M, b = 256).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ozaki_tc tools/ozaki_tc.cu && build/ozaki_tc
//
// Each row of A (column of Y) is scaled by a power of two into (-128, 128)
// and cut into S int8 slices of 7 bits; slice products of the same level
// d = p + q are summed exactly in int32 TMEM accumulators by
// tcgen05.mma.kind::i8 (M 128, N 64, K 32); the epilogue combines the levels
// in fp64 and undoes the scaling.  Error ~ 2^-(7S) of |A_i||Y_j|.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cuda_runtime.h>
#include <random>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);         \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

constexpr int K = 128;      // inner dimension (rank)
constexpr int TM = 128;     // rows per tile
constexpr int TN = 64;      // columns per group

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO: 8-row groups 1 KB apart
    d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
    return d;
}

// kind::i8, D s32, A/B signed int8, both K-major, M = 128, N = 64
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((TN >> 3) << 17) | ((TM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// Persistent, warp-specialised: warps 0-3 epilogue (TMEM lane quarter w),
// warp 4 producer (cp.async of the A / Y slices, lane 0 issues the MMAs).
// Column groups of TN2 = 32 columns; two TMEM accumulator buffers of
// S levels x 32 columns, two Y buffers, one A buffer per tile.
constexpr int TN2 = 32;
template <int S>
__global__ void __launch_bounds__(288, 1)
    oz_gemm_ws(const int8_t* __restrict__ As, const int8_t* __restrict__ Ys, const int* __restrict__ eA,
               const int* __restrict__ fY, double* __restrict__ C, int n, int b, int64_t ldc, int mode = 0) {
    constexpr uint32_t kIdesc32 = (2u << 4) | (1u << 7) | (1u << 10) | ((TN2 >> 3) << 17) | ((TM >> 4) << 24);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t accfull[2], accempty[2];
    __shared__ uint32_t tmem_base_s;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;                                 // S x [128][128 B]
    uint8_t* sY = base + S * TM * K;                    // 3 x S x [32][128 B]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int j = 0; j < 2; ++j) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&accfull[j])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su32(&accempty[j])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    const int ntiles = (n + TM - 1) / TM, ncg = b / TN2;
    if (warp == 8) {
        // ---------------- producer ----------------
        // Y slices of column-group use u go to stage u % 3 and are issued two
        // uses ahead; stage (u+2) % 3 was read by MMA(u-1), so its reload
        // waits for that MMA's commit.  A is reloaded per tile once the
        // tile's last MMAs completed.
        const int total = ((ntiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                           static_cast<int>(gridDim.x)) * ncg;
        auto load_y = [&](int u) {
            if (u < total) {
                const int cg = u % ncg;
                uint8_t* yb = sY + (u % 3) * S * TN2 * K;
                for (int c = lane; c < S * TN2 * 8; c += 32) {
                    const int s = c / (TN2 * 8), r = (c / 8) % TN2, ch = c % 8;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     su32(yb + s * TN2 * K + r * 128 + ((ch ^ (r & 7)) * 16))),
                                 "l"(Ys + ((static_cast<size_t>(s) * b + cg * TN2 + r) * K + ch * 16)));
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        auto load_a = [&](int tile) {
            const int row0 = tile * TM;
            for (int c = lane; c < S * TM * 8; c += 32) {
                const int s = c / (TM * 8), r = (c / 8) % TM, ch = c % 8;
                const int rr = row0 + r < n ? row0 + r : n - 1;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 su32(sA + s * TM * K + r * 128 + ((ch ^ (r & 7)) * 16))),
                             "l"(As + ((static_cast<size_t>(s) * n + rr) * K + ch * 16)));
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        // prologue: A of the first tile, Y of uses 0 and 1
        load_a(blockIdx.x);
        load_y(0);
        load_y(1);
        int u = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            if (u > 0) {
                // new tile: A free once the previous tile's MMAs are done
                mbar_wait(su32(&accfull[(u - 1) & 1]), ((u - 1) >> 1) & 1);
                load_a(tile);
            }
            for (int cg = 0; cg < ncg; ++cg, ++u) {
                // Y(u) (and A) landed: all groups but the newest (Y(u+1)) -- or,
                // right after a reload of A, all of them
                if (cg == 0 && u > 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
                else asm volatile("cp.async.wait_group 1;" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                const int j = u & 1;
                if (u >= 2) mbar_wait(su32(&accempty[j]), ((u - 2) >> 1) & 1);
                const uint8_t* yb = sY + (u % 3) * S * TN2 * K;
                if (lane == 0) {
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t acc = tmem + j * (S * TN2);
                    const uint64_t da0 = sw128_desc(su32(sA)), db0 = sw128_desc(su32(yb));
                    for (int d = 0; d < (mode != 2 ? S : 0); ++d)
                        for (int p = 0; p <= d; ++p) {
                            const int q = d - p;
#pragma unroll
                            for (int kk = 0; kk < K / 32; ++kk) {
                                const uint64_t da = da0 + static_cast<uint64_t>((p * TM * K + kk * 32) >> 4);
                                const uint64_t db = db0 + static_cast<uint64_t>((q * TN2 * K + kk * 32) >> 4);
                                asm volatile(
                                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(
                                        acc + d * TN2),
                                    "l"(da), "l"(db), "r"(kIdesc32), "r"((p > 0 || kk > 0) ? 1u : 0u), "r"(0), "r"(0),
                                    "r"(0), "r"(0));
                            }
                        }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     su32(&accfull[j]))
                                 : "memory");
                }
                __syncwarp();
                // stage (u+2) % 3 was read by MMA(u-1)
                if (u >= 1) mbar_wait(su32(&accfull[(u - 1) & 1]), ((u - 1) >> 1) & 1);
                load_y(u + 2);
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else {
        // ---------------- epilogue (warps 0-7) ----------------
        // warp w reads TMEM lane quarter w % 4, columns 16 * (w / 4) .. +15
        const int quarter = warp & 3, half = warp >> 2;
        uint32_t use = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int row = tile * TM + quarter * 32 + lane;
            const double rs = row < n ? __longlong_as_double(static_cast<long long>(1023 - eA[row]) << 52) : 0.0;
            for (int cg = 0; cg < ncg; ++cg, ++use) {
                const int j = use & 1;
                mbar_wait(su32(&accfull[j]), (use >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                long long hi[16], lo[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) hi[c] = lo[c] = 0;
#pragma unroll
                for (int d = 0; d < S; ++d) {
                    uint32_t v[16];
                    const uint32_t addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + j * (S * TN2) + d * TN2 + half * 16;
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                          "=r"(v[14]), "=r"(v[15])
                        : "r"(addr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (d < 3) {
#pragma unroll
                        for (int c = 0; c < 16; ++c) hi[c] = hi[c] * 128 + static_cast<int32_t>(v[c]);
                    } else {
#pragma unroll
                        for (int c = 0; c < 16; ++c) lo[c] = lo[c] * 128 + static_cast<int32_t>(v[c]);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&accempty[j])) : "memory");
                if (row < n && mode != 1) {
                    const double shi = 1.0 / 16384.0, slo = ldexp(1.0, -7 * (S - 1));
                    double out[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const int col = cg * TN2 + half * 16 + c;
                        const double cs = __longlong_as_double(static_cast<long long>(1023 - fY[col]) << 52);
                        out[c] = fma(static_cast<double>(hi[c]), shi, static_cast<double>(lo[c]) * slo) * rs * cs;
                    }
                    double* dst = C + static_cast<size_t>(row) * ldc + cg * TN2 + half * 16;
#pragma unroll
                    for (int c = 0; c < 16; c += 2) *reinterpret_cast<double2*>(dst + c) = make_double2(out[c], out[c + 1]);
                }
            }
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// row-wise power-of-two scaling into (-128, 128) and S slices of 7 bits
static void slice_rows(const std::vector<double>& M, int rows, int S, std::vector<int8_t>& out, std::vector<int>& ex) {
    out.assign(static_cast<size_t>(S) * rows * K, 0);
    ex.assign(rows, 0);
    for (int i = 0; i < rows; ++i) {
        double mx = 0;
        for (int k = 0; k < K; ++k) mx = std::max(mx, std::fabs(M[static_cast<size_t>(i) * K + k]));
        int e = 0;
        if (mx > 0) e = 6 - static_cast<int>(std::floor(std::log2(mx)));
        while (mx > 0 && std::ldexp(mx, e) >= 128.0) --e;
        ex[i] = e;
        for (int k = 0; k < K; ++k) {
            double a = std::ldexp(M[static_cast<size_t>(i) * K + k], e);
            for (int s = 0; s < S; ++s) {
                const double t = std::trunc(a);
                out[(static_cast<size_t>(s) * rows + i) * K + k] = static_cast<int8_t>(t);
                a = (a - t) * 128.0;
            }
        }
    }
}

int main(int argc, char** argv) {
    constexpr int S = 7;
    const int n_check = 4096, b = 256;
    const int n_big = argc > 1 ? atoi(argv[1]) : 2394845;
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::uniform_real_distribution<double> ud(-20.0, 5.0);
    std::vector<double> A(static_cast<size_t>(n_check) * K), Yt(static_cast<size_t>(b) * K);  // Yt: [b][K]
    for (int i = 0; i < n_check; ++i) {
        const double rs = std::ldexp(1.0, static_cast<int>(ud(rng)));
        for (int k = 0; k < K; ++k) A[static_cast<size_t>(i) * K + k] = rs * nd(rng) * (k % 17 == 3 ? 1e-6 : 1.0);
    }
    for (int j = 0; j < b; ++j)
        for (int k = 0; k < K; ++k) Yt[static_cast<size_t>(j) * K + k] = nd(rng) * std::ldexp(1.0, j % 9);
    std::vector<int8_t> As, Ys;
    std::vector<int> eA, fY;
    slice_rows(A, n_check, S, As, eA);
    slice_rows(Yt, b, S, Ys, fY);
    int8_t *dA, *dY;
    int *deA, *dfY;
    double* dC;
    CK(cudaMalloc(&dA, As.size()));
    CK(cudaMalloc(&dY, Ys.size()));
    CK(cudaMalloc(&deA, 4 * eA.size()));
    CK(cudaMalloc(&dfY, 4 * fY.size()));
    CK(cudaMalloc(&dC, sizeof(double) * n_check * b));
    CK(cudaMemcpy(dA, As.data(), As.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dY, Ys.data(), Ys.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(deA, eA.data(), 4 * eA.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dfY, fY.data(), 4 * fY.size(), cudaMemcpyHostToDevice));
    const size_t smem = 1024 + static_cast<size_t>(S) * (TM + 3 * TN2) * K;
    CK(cudaFuncSetAttribute(oz_gemm_ws<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    oz_gemm_ws<S><<<std::min(sms, (n_check + TM - 1) / TM), 288, smem>>>(dA, dY, deA, dfY, dC, n_check, b, b);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<double> Cg(static_cast<size_t>(n_check) * b);
    CK(cudaMemcpy(Cg.data(), dC, sizeof(double) * Cg.size(), cudaMemcpyDeviceToHost));
    double worst = 0.0;
    for (int i = 0; i < n_check; ++i)
        for (int j = 0; j < b; ++j) {
            long double s = 0, na = 0, ny = 0;
            for (int k = 0; k < K; ++k) {
                const long double a = A[static_cast<size_t>(i) * K + k], y = Yt[static_cast<size_t>(j) * K + k];
                s += a * y;
                na += a * a;
                ny += y * y;
            }
            const double err = static_cast<double>(std::fabs(static_cast<long double>(Cg[static_cast<size_t>(i) * b + j]) - s) /
                                                   std::sqrt(na * ny));
            worst = std::max(worst, err);
        }
    printf("{\"slices\": %d, \"max_err_rel_to_norms\": %.3e", S, worst);
    // timing at the headline shape (slices random: timing only)
    int8_t* dAb;
    double* dCb;
    int* deAb;
    CK(cudaMalloc(&dAb, static_cast<size_t>(S) * n_big * K));
    CK(cudaMalloc(&dCb, sizeof(double) * static_cast<size_t>(n_big) * b));
    CK(cudaMalloc(&deAb, 4 * static_cast<size_t>(n_big)));
    CK(cudaMemset(dAb, 1, static_cast<size_t>(S) * n_big * K));
    CK(cudaMemset(deAb, 0, 4 * static_cast<size_t>(n_big)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms;
    oz_gemm_ws<S><<<grid, 288, smem>>>(dAb, dY, deAb, dfY, dCb, n_big, b, b);
    CK(cudaGetLastError());
    float mode_ms[3];
    for (int mode = 2; mode >= 0; --mode) {
        cudaEventRecord(e0);
        oz_gemm_ws<S><<<grid, 288, smem>>>(dAb, dY, deAb, dfY, dCb, n_big, b, b, mode);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&mode_ms[mode], e0, e1);
    }
    const float ms = mode_ms[0];
    printf(", \"ms_no_store\": %.3f, \"ms_no_mma\": %.3f", mode_ms[1], mode_ms[2]);
    const double flops = 2.0 * n_big * K * b;
    printf(", \"n\": %d, \"b\": %d, \"ms\": %.3f, \"fp64_equiv_tflops\": %.2f}\n", n_big, b, ms, flops / ms / 1e9);
    return 0;
}
