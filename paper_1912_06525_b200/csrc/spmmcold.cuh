// spmmcold.cuh -- EXPERIMENT (not in the product build; make EXTRA=-DKZ_EXPERIMENTS=1):
// a cold-column pass for a split K1 on large operators.  Measured at R-MAT 22
// (profiles/r02_k1_coldpass_proto.jsonl): the pass gathers at ~6.6 TB/s and
// main + cold is slower than the unsplit K1 (19.6-22 ms vs 18.8 ms), because
// static slot ownership needs slab lockstep, per-(group, slab) loads are uneven
// (max/mean 1.8), and with 5 accumulator slots per lane group the shared-memory
// carve-out leaves 28 KB of L1 for the gathers in flight.  Kept for the record.
//
// K1 gathers one 8*C-byte row of Xg per stored entry.  At R-MAT 22 a C = 32
// chunk of Xg is 612 MB: the ~130k highest-degree columns (33 MB) take 74% of
// the gathers and stay in L2, but the remaining "cold" columns are fetched
// from DRAM ~13 times each per chunk (67 of K1's 72 GB of DRAM traffic per
// launch, profiles/r02_spmm_cfg3.ncu-rep).  The split operator (built in numpy by
// tools/k1_coldpass_proto.py) moves the cold entries of the rows that hold most of them
// into this pass, which walks the cold columns slab by slab (a slab of Xg
// rows fits in L2), every lane group of the grid in step:
//
//   * a lane group (G = C/VEC lanes) owns up to `slots` partial rows
//     ("virtual rows": a row's cold entries, or one round-robin piece of a
//     hub row's) for the whole launch; their accumulators are thread-private
//     words of shared memory, so there is no inter-warp protocol at all;
//   * the group's entries are stored in processing order: [slab][group], each
//     entry (slot << 27 | column); a slot's running sum lives in registers
//     and is folded into its accumulator when the stream changes slot;
//   * warps may run at most one slab ahead of the slowest warp (counter per
//     (chunk, slab), spin-wait): the L2 working set is two slabs.  The wait
//     needs every CTA resident, so the kernel is launched cooperatively;
//   * at the end of a chunk the accumulators are streamed to
//     P[chunk][group*slots + slot][C]; the main K1 pass reads them as extra
//     gathered columns (index cols + group*slots + slot).
//
// Summation order is fixed (entry order within a slot, slabs in order), so
// the result is run-to-run deterministic.
#pragma once

#include "spmm.cuh"

namespace kz {

constexpr int kColdSlotBits = 27;  // entry = slot << 27 | column  (cols < 2^27)
constexpr uint32_t kColdColMask = (1u << kColdSlotBits) - 1u;
constexpr uint32_t kColdInvalid = 0xffffffffu;
#ifndef KZ_COLD_SLOTS
#define KZ_COLD_SLOTS 5
#endif
constexpr int kColdSlots = KZ_COLD_SLOTS;  // partial rows per lane group (8*C bytes of shared memory each)

struct ColdArgs {
    const uint32_t* __restrict__ ent;     // packed entries, [slab][group] segments
    const int32_t* __restrict__ segoff;   // [nslabs*ng + 1]
    const uint8_t* __restrict__ nslot;    // [ng] slots in use per group
    int32_t ng, nslabs, nchunks;
    int32_t cols;
    const double* Xg;
    int64_t ldxg;
    double* P;                            // [nchunks][ng*slots][C]
    int32_t* done;                        // [nchunks*nslabs] CTAs finished per (chunk, slab)
    const int32_t* chunk_active;
    const int32_t* n_active;              // CG/PCG: columns still running (0: leave at once)
    int32_t throttle;                     // 1: slab lockstep (0: experiments only)
};

template <int C>
__global__ void __launch_bounds__(kThreads, kSpmmMinBlocks) spmm_cold_kernel(ColdArgs a) {
    using K = Cfg<C>;
    constexpr int VEC = K::VEC;
    static_assert(VEC == 4 && K::G == 8, "cold pass is built for C = 32 (32-byte gathers)");
    constexpr int R = 4;
    extern __shared__ double s_acc[];  // [groups per CTA][slots][C]
    __shared__ int s_arr[2];           // warps of this CTA that finished slab p (parity p & 1)
    if (threadIdx.x < 2) s_arr[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gw = lane / K::G, lg = lane % K::G, gbase = gw * K::G;
    const unsigned gmask = ((1u << K::G) - 1u) << gbase;
    const int gic = (threadIdx.x / 32) * K::NGW + gw;  // lane group within the CTA
    const int g = blockIdx.x * (kThreads / K::G) + gic;
    double* my = s_acc + static_cast<size_t>(gic) * kColdSlots * C + lg * VEC;
    if (a.n_active && *reinterpret_cast<volatile const int32_t*>(a.n_active) == 0) return;
    const int my_slots = a.nslot[g];

    for (int chunk = 0; chunk < a.nchunks; ++chunk) {
        if (a.chunk_active && !a.chunk_active[chunk]) continue;
#pragma unroll
        for (int s = 0; s < kColdSlots; ++s)
#pragma unroll
            for (int q = 0; q < VEC; ++q) my[s * C + q] = 0.0;
        int cur = -1;
        double acc[VEC];
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
        const double* __restrict__ Xl = a.Xg + static_cast<size_t>(chunk) * a.ldxg + lg * VEC;
        int32_t* done = a.done + chunk * a.nslabs;

        for (int p = 0; p < a.nslabs; ++p) {
            // at most one slab ahead of the slowest CTA: thread 0 polls the
            // arrival count of slab p-2 (one poller per CTA keeps the counter's
            // L2 slice out of the way of the arrivals), the barrier releases
            // the CTA and separates its arrivals for slabs p-1 and p+1
            if (a.throttle) {
                if (p >= 2 && threadIdx.x == 0) {
#if KZ_CHECKED
                    long long spins = 0;
#endif
                    while (*reinterpret_cast<volatile int32_t*>(done + p - 2) < static_cast<int32_t>(gridDim.x)) {
                        __nanosleep(256);
                        KZ_DCHECK(++spins < (1ll << 26));
                    }
                }
                __syncthreads();
            }
            const int k = p * a.ng + g;
            const int beg = a.segoff[k], end = a.segoff[k + 1];
            uint32_t ne = (lg < R && beg + lg < end) ? __ldcs(a.ent + beg + lg) : kColdInvalid;
#pragma unroll 1
            for (int base = beg; base < end; base += R) {
                const uint32_t e = ne;
                const int pos = base + R + lg;
                ne = (lg < R && pos < end) ? __ldcs(a.ent + pos) : kColdInvalid;
                double v[R][VEC];
                uint32_t et[R];
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    et[t] = __shfl_sync(gmask, e, gbase + t);
                    const uint32_t j = et[t] == kColdInvalid ? 0u : (et[t] & kColdColMask);
                    KZ_DCHECK(static_cast<int>(j) < a.cols);
                    ld_nc<VEC>(Xl + static_cast<size_t>(j) * C, v[t]);
                }
#pragma unroll
                for (int t = 0; t < R; ++t) {
                    if (et[t] != kColdInvalid) {
                        const int s = static_cast<int>(et[t] >> kColdSlotBits);
                        if (s != cur) {
                            KZ_DCHECK(s < my_slots);
                            if (cur >= 0) {
#pragma unroll
                                for (int q = 0; q < VEC; ++q) my[cur * C + q] += acc[q];
                            }
                            cur = s;
#pragma unroll
                            for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
                        }
#pragma unroll
                        for (int q = 0; q < VEC; ++q) acc[q] = __dadd_rn(acc[q], v[t][q]);
                    }
                }
            }
            __syncwarp();
            // the CTA's last warp out of slab p reports the CTA
            if (a.throttle && lane == 0 && atomicAdd(&s_arr[p & 1], 1) == kWarps - 1) {
                s_arr[p & 1] = 0;
                atomicAdd(done + p, 1);
            }
        }
        if (cur >= 0) {
#pragma unroll
            for (int q = 0; q < VEC; ++q) my[cur * C + q] += acc[q];
        }
        double* Pc = a.P + (static_cast<size_t>(chunk) * a.ng + g) * kColdSlots * C + lg * VEC;
        for (int s = 0; s < my_slots; ++s) {
            double o[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) o[q] = my[s * C + q];
            st_stream<VEC>(Pc + static_cast<size_t>(s) * C, o);
        }
    }
}

inline size_t cold_smem_bytes(int C) { return static_cast<size_t>(kThreads / Cfg<32>::G) * kColdSlots * C * sizeof(double); }

// resident CTAs per SM of the cold pass (its grid is fixed when the split is
// built: every lane group owns its slots for the whole launch)
inline int cold_ctas_per_sm() {
    int occ = 0;
    cudaFuncSetAttribute(spmm_cold_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(cold_smem_bytes(32)));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_cold_kernel<32>, kThreads, cold_smem_bytes(32)) !=
        cudaSuccess)
        return 0;
    return std::min(occ, kSpmmMinBlocks);
}

inline int launch_spmm_cold(ColdArgs a, int grid, cudaStream_t st) {
    void* params[] = {&a};
    cudaFuncSetAttribute(spmm_cold_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(cold_smem_bytes(32)));
    cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(spmm_cold_kernel<32>), dim3(grid),
                                                dim3(kThreads), params, cold_smem_bytes(32), st);
    if (e != cudaSuccess) return fail(KZ_ECUDA, std::string("cold pass launch: ") + cudaGetErrorString(e));
    note_launch();
    return KZ_OK;
}

}  // namespace kz
