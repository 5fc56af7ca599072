// spmm.cuh -- K1: binary-pattern CSR SpMM with fused epilogue and column dots.
//
//   Y = s0*Z + (s1*Xs + s2*(A Xg))         (per row, per column of the block)
//   dots[j] = sum_i D[i,j] * Y[i,j]        (optional, deterministic)
//
// Replaces the reference's operator applications: KatzIndex.apply_m_permuted
// (index.py:86-91: x - alpha*A x through factor reassembly), the coupling
// products m12 @ v / m12.T @ u (solver.py:110,115,178), the interior solve
// M11^-1 (factor.py:89-106, as a weighted operator) and the rhs column
// (index.py:93-101).  A is a binary pattern (no stored values, int32 column
// indices), so the only per-nonzero traffic is 4 bytes of index plus a
// gathered C-wide row segment of Xg.
//
// Layout: blocks are chunked node-major [b/C][rows][C] (the C doubles of one
// row are contiguous, 8*C bytes), so a gathered neighbour is one coalesced
// segment read by G = C/VEC lanes with 16-byte loads.  The grid is
// chunk-major, so the L2 working set is one chunk of Xg, not the block.
//
// Schedule (built once per operator on the host, graph.cu): the rows are cut
// into warp tasks in row order --
//   S  a run of short rows (deg <= kMedDeg), one lane group per row;
//   M  one medium row, its neighbours split over the warp's lane groups;
//   L  one kSegLen-long segment of a long row (power-law hubs); the warp that
//      runs a row's last segment waits for the others and combines the
//      partial sums in segment order (stream-K style fix-up).
// Optional column blocking (graph.cu SchedOpts, KZ_K1_SLICE_MB, off by
// default): rows above a degree threshold are also cut by column block and
// their segments run block-major so the gathered X slice stays in L2.
// Measured at R-MAT 22 (profiles/r01_k1_colblock_sweep.jsonl): slower at
// every slice size -- the per-segment fix-up costs more than the L2 hits save.
// Each CTA owns a contiguous task range and its warps pull tasks dynamically
// (no intra-CTA tail); every task's dot partial lands in its own shared slot
// and slots are summed in task order, then CTAs in CTA order by the last CTA
// of the chunk, so the column dots are run-to-run deterministic.  Short and
// medium rows sum their neighbours in CSR order with explicit _rn adds, so
// they are bit-identical to scipy's csr_matvec.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace kz {
#ifndef KZ_K1_MEDDEG
#define KZ_K1_MEDDEG 32
#endif
#ifndef KZ_K1_SEGLEN
#define KZ_K1_SEGLEN 4096
#endif
#ifndef KZ_K1_GROUPCOST
#define KZ_K1_GROUPCOST 4096.0
#endif
constexpr int kMedDeg = KZ_K1_MEDDEG;    // rows with deg <= kMedDeg are "short"
constexpr int kSegLen = KZ_K1_SEGLEN;    // rows with deg > kSegLen are split into segments
#ifndef KZ_K1_GROUPTASKS
#define KZ_K1_GROUPTASKS 8
#endif
constexpr int kGroupTasks = KZ_K1_GROUPTASKS;   // max tasks a warp dequeues at once (one dot slot)
constexpr double kGroupCost = KZ_K1_GROUPCOST;  // max neighbour-equivalents per work unit
constexpr int kSuperGroups = 256; // max groups reduced together by their last finisher
#ifndef KZ_K1_MINBLOCKS
#define KZ_K1_MINBLOCKS 5  // resident CTAs per SM the register budget is sized for
#endif
constexpr int kSpmmMinBlocks = KZ_K1_MINBLOCKS;
constexpr double kColBlockSliceMB = 0.0;  // column-block slice of a C = 32 chunk (0: off)
constexpr int64_t kColBlockMinDeg = 128;  // rows above this degree are column-blocked
}  // namespace kz

struct kz_graph {
    int64_t rows = 0, cols = 0, nnz = 0;
    int32_t* rowptr = nullptr;  // device int32[rows+1]
    int32_t* colidx = nullptr;  // device int32[nnz]
    double* vals = nullptr;     // optional fp64 values (weighted operator, e.g. M11^-1)
    int32_t ntasks = 0;
    int4* tasks = nullptr;      // {a, b, type, k}: S {r0, r1}, M {row}, L {row, lidx, seg k}
    int32_t ngroups = 0;        // warp work units (consecutive task ranges)
    int32_t* group_first = nullptr;  // [ngroups+1]
    int32_t nlong = 0;              // rows with deg > kSegLen
    int32_t nseg = 0;               // their segments
    int32_t* long_seg0 = nullptr;   // [nlong+1] first segment slot of each long row
    int2* seg_range = nullptr;      // [nseg] CSR position range [x, y) of each segment
    int32_t nblocks = 1;            // column blocks of the long-row phases (1: unblocked)
    int32_t max_deg = 0;
    uint64_t uid = 0;               // process-unique id (keys cached solve graphs)
};

namespace kz {

enum TaskType : int { TASK_S = 0, TASK_M = 1, TASK_L = 2 };

#ifndef KZ_K1_VEC32
#define KZ_K1_VEC32 4  // doubles per lane of a gathered row for C >= 32 (2: 16-byte, 4: 32-byte loads)
#endif
#ifndef KZ_K1_VEC16
#define KZ_K1_VEC16 2  // doubles per lane of a gathered row for C = 16 (experiments: 4 = 32-byte loads)
#endif
#ifndef KZ_K1_SMEM_DOT
#define KZ_K1_SMEM_DOT 1  // 1: column-dot accumulators in shared memory instead of registers
#endif
#ifndef KZ_K1_PRED
#define KZ_K1_PRED 0   // 1: tail slots of a gather round are predicated off instead of clamped
#endif
#ifndef KZ_K1_R32
#define KZ_K1_R32 0    // neighbours per round for C >= 32 (0: default rule)
#endif

template <int C>
struct Cfg {
    // doubles per lane of a gathered row: 16-byte loads, or 32-byte
    // (LDG.256, sm_100) loads for wide chunks
    static constexpr int VEC = (C >= 32) ? KZ_K1_VEC32 : (C >= 16 ? KZ_K1_VEC16 : (C >= 2 ? 2 : 1));
    static constexpr int SVEC = (C >= 2) ? 2 : 1;  // doubles per lane of the streaming kernels
    static constexpr int G = C / VEC;             // lanes per row group
    static constexpr int NGW = 32 / G;            // row groups per warp
    // neighbours gathered per round: 8 with 16-byte loads, 4 with 32-byte loads (4 for
    // narrow groups) -- R*VEC doubles of gather registers per lane either way
    static constexpr int R = (C >= 32 && KZ_K1_R32 > 0) ? KZ_K1_R32 : ((G >= 8) ? (VEC == 4 ? 4 : 8) : (G >= 4 ? G : 4));
    static constexpr int PER = (R >= G) ? R / G : 1;  // indices loaded per lane per round
    static constexpr bool PART = R < G;               // only lanes lg < R load indices
};

template <int VEC>
__device__ __forceinline__ void ld_nc(const double* p, double (&v)[VEC]);
template <>
__device__ __forceinline__ void ld_nc<4>(const double* p, double (&v)[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p));
}
template <>
__device__ __forceinline__ void ld_nc<2>(const double* p, double (&v)[2]) {
    double2 t = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = t.x;
    v[1] = t.y;
}
template <>
__device__ __forceinline__ void ld_nc<1>(const double* p, double (&v)[1]) {
    v[0] = __ldg(p);
}
#ifndef KZ_K1_L2HINT
#define KZ_K1_L2HINT 0  // experiments: per-row L2 eviction priority (1: hub last / tail first, 2: hub last / tail normal)
#endif
// gather with an L2 cache-policy operand (createpolicy), chosen per row
__device__ __forceinline__ void ld_nc_hint4(const double* p, double (&v)[4], uint64_t pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p), "l"(pol));
}
#ifndef KZ_K1_L1HINT
#define KZ_K1_L1HINT 0  // experiments: per-row L1 policy (1: hub evict_last / tail no_allocate, 2: hub evict_last / tail evict_first)
#endif
// gather with an L1 eviction priority chosen per row: the hottest hub rows
// stay in L1, the tail rows pass through without displacing them
__device__ __forceinline__ void ld_nc_l1hint4(const double* p, double (&v)[4], bool hub) {
    if (hub) {
        asm volatile("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(p));
    } else {
#if KZ_K1_L1HINT == 2
        asm volatile("ld.global.nc.L1::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
#else
        asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
#endif
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(p));
    }
}
// Predicated gather: lanes with !pred issue no memory request and read 0.
template <int VEC>
__device__ __forceinline__ void ld_nc_pred(const double* p, double (&v)[VEC], bool pred) {
    const int pr = pred;
    if constexpr (VEC == 4) {
        asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
            "mov.f64 %0, 0d0000000000000000;\n\tmov.f64 %1, 0d0000000000000000;\n\t"
            "mov.f64 %2, 0d0000000000000000;\n\tmov.f64 %3, 0d0000000000000000;\n\t"
            "@q ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n\t}"
            : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
            : "l"(p), "r"(pr));
    } else if constexpr (VEC == 2) {
        asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
            "mov.f64 %0, 0d0000000000000000;\n\tmov.f64 %1, 0d0000000000000000;\n\t"
            "@q ld.global.nc.v2.f64 {%0,%1}, [%2];\n\t}"
            : "=d"(v[0]), "=d"(v[1])
            : "l"(p), "r"(pr));
    } else {
        asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
            "mov.f64 %0, 0d0000000000000000;\n\t"
            "@q ld.global.nc.f64 %0, [%1];\n\t}"
            : "=d"(v[0])
            : "l"(p), "r"(pr));
    }
}
template <int VEC>
__device__ __forceinline__ void ld_plain(const double* p, double (&v)[VEC]) {
    if constexpr (VEC == 4) {
        asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(p)
                     : "memory");
    } else if constexpr (VEC == 2) {
        double2 t = *reinterpret_cast<const double2*>(p);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = *p;
    }
}
template <int VEC>
__device__ __forceinline__ void st_plain(double* p, const double (&v)[VEC]) {
    if constexpr (VEC == 4) {
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                     : "memory");
    } else if constexpr (VEC == 2) {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    } else {
        *p = v[0];
    }
}

// streaming (evict-first) store: the output block must not push gathered
// rows out of L2 (column indices are read with __ldcs for the same reason)
template <int VEC>
__device__ __forceinline__ void st_stream(double* p, const double (&v)[VEC]) {
    if constexpr (VEC == 4) {
        asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                     : "memory");
    } else if constexpr (VEC == 2) {
        __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
    } else {
        __stcs(p, v[0]);
    }
}

// Sum Xg rows of neighbours col[beg..end) into acc, R neighbours per round,
// rounds `stride` apart.  All lanes of a group share the neighbour; lane lg
// owns columns lg*VEC .. lg*VEC+VEC-1 of the chunk.  W: weighted operator.
// .cg (L2-only) loads of data other CTAs wrote in the same launch
template <int VEC>
__device__ __forceinline__ void ld_cg_vec(const double* p, double (&v)[VEC]) {
    if constexpr (VEC == 4) {
        asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(p));
    } else if constexpr (VEC == 2) {
        const double2 t = __ldcg(reinterpret_cast<const double2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = __ldcg(p);
    }
}

// CO: the gathered block is written within the same launch (the fused small
// CG loop): coherent L1-cached loads instead of the non-coherent path; the
// kernel's gpu-scope fences before each grid barrier invalidate L1 (CCTL.IVALL)
template <int C, bool W = false, bool CO = false>
__device__ __forceinline__ void gather_rows(const int32_t* __restrict__ col, int beg, int end,
                                            int stride, const double* __restrict__ Xc, int lg,
                                            int gbase, unsigned gmask,
                                            double (&acc)[Cfg<C>::VEC],
                                            const double* __restrict__ vals = nullptr,
                                            int hub_rows = 0, uint64_t pol_hub = 0, uint64_t pol_tail = 0,
                                            int ncols = 0x7fffffff) {
    using K = Cfg<C>;
    // Software pipeline: the column indices of round k+1 are loaded while the
    // R gathers of round k are in flight.  Tail slots gather a clamped valid
    // row (index 0, always cache-hot) instead of predicating the load, so the
    // compiler keeps all R loads outstanding; their sums are skipped.
    int idx[K::PER], nidx[K::PER];
    double wv[K::PER], nwv[K::PER];
#pragma unroll
    for (int m = 0; m < K::PER; ++m) {
        const int pos = beg + lg + K::G * m;
        const bool ok = pos < end && (!K::PART || lg < K::R);
        nidx[m] = ok ? __ldcs(col + pos) : 0;
        if constexpr (W) nwv[m] = ok ? __ldg(vals + pos) : 0.0;
    }
    const double* __restrict__ Xl = Xc + lg * K::VEC;
#pragma unroll 1
    for (int base = beg; base < end; base += stride) {
#pragma unroll
        for (int m = 0; m < K::PER; ++m) {
            idx[m] = nidx[m];
            if constexpr (W) wv[m] = nwv[m];
            const int pos = base + stride + lg + K::G * m;
            const bool ok = pos < end && (!K::PART || lg < K::R);
            nidx[m] = ok ? __ldcs(col + pos) : 0;
            if constexpr (W) nwv[m] = ok ? __ldg(vals + pos) : 0.0;
        }
        double v[K::R][K::VEC];
        double w[K::R];
#pragma unroll
        for (int t = 0; t < K::R; ++t) {
            int j;
            if constexpr (K::G == 1) {
                j = idx[t];
                if constexpr (W) w[t] = wv[t];
            } else {
                j = __shfl_sync(gmask, idx[t / K::G], gbase + (t % K::G));
                if constexpr (W) w[t] = __shfl_sync(gmask, wv[t / K::G], gbase + (t % K::G));
            }
            KZ_DCHECK(j >= 0 && j < ncols);
#if KZ_K1_PRED
            ld_nc_pred<K::VEC>(Xl + static_cast<size_t>(j) * C, v[t], t < end - base);
#elif KZ_K1_L2HINT
            if constexpr (K::VEC == 4)
                ld_nc_hint4(Xl + static_cast<size_t>(j) * C, v[t], j < hub_rows ? pol_hub : pol_tail);
            else
                ld_nc<K::VEC>(Xl + static_cast<size_t>(j) * C, v[t]);
#elif KZ_K1_L1HINT
            if constexpr (K::VEC == 4 && !CO)
                ld_nc_l1hint4(Xl + static_cast<size_t>(j) * C, v[t], j < hub_rows);
            else if constexpr (CO)
                ld_plain<K::VEC>(Xl + static_cast<size_t>(j) * C, v[t]);
            else
                ld_nc<K::VEC>(Xl + static_cast<size_t>(j) * C, v[t]);
#else
            if constexpr (CO)
                ld_plain<K::VEC>(Xl + static_cast<size_t>(j) * C, v[t]);
            else
                ld_nc<K::VEC>(Xl + static_cast<size_t>(j) * C, v[t]);
#endif
        }
        const int nvalid = end - base;  // slots t < nvalid hold real neighbours
#pragma unroll
        for (int t = 0; t < K::R; ++t)
            if (t < nvalid) {
#pragma unroll
                for (int q = 0; q < K::VEC; ++q) {
                    if constexpr (W)
                        acc[q] = fma(w[t], v[t][q], acc[q]);
                    else
                        acc[q] = __dadd_rn(acc[q], v[t][q]);
                }
            }
    }
}

// What the last CTA of a chunk does with the reduced column dots.
struct DotHook {
    int mode = 0;               // 0: dots_out[col] = v ; 1: CG/PCG step length
    int b = 0;                  // real (unpadded) columns
    double* dots_out = nullptr;
    // mode 1 state (see cg.cu)
    const double* rs = nullptr;  // r.r (CG) or r.z (PCG)
    double* alpha = nullptr;
    int32_t* active = nullptr;
    int32_t* xstamp = nullptr;
    int32_t* chunk_xstamp = nullptr;
    int32_t* status = nullptr;
    int32_t* err = nullptr;
    int32_t* n_active = nullptr;
    int32_t iter = 0;
    const int32_t* iter_dev = nullptr;  // device iteration number (graph replay); overrides iter
};

struct SpmmArgs {
    int32_t rows, cols;
    const int32_t* __restrict__ rowptr;
    const int32_t* __restrict__ colidx;
    const int4* __restrict__ tasks;
    const int32_t* __restrict__ group_first;
    const int32_t* __restrict__ long_seg0;
    const int2* __restrict__ seg_range;
    int32_t ntasks, nlong, nseg;
    int32_t ngroups;    // task groups (kGroupTasks consecutive tasks) per chunk
    int32_t nsuper;     // super groups per chunk
    int32_t super_size; // groups per super group (spmm_super_size)
    int32_t nchunks;
    int32_t chunk0;     // first chunk of this launch (0 unless the SpMM is launched chunk by chunk)
    int32_t nwarps;     // warps of the (persistent) launch
    const double* Xg;
    const double* Xs;
    const double* Z;
    double* Y;
    const double* D;
    // chunk strides (elements) of each operand; 0 = dense default (rows*C or cols*C)
    int64_t ldxg, ldxs, ldz, ldy, ldd;
    const double* vals;  // weighted operator values (nullptr: binary pattern)
    double s0, s1, s2;
    const double* s0v;   // per-column s0 (device [nchunks*C]); overrides s0 when set
    int32_t hub_rows;    // KZ_K1_L2HINT experiments: rows [0, hub_rows) get the hub L2 policy
    double* partial;   // [nchunks][nseg][C] long-row segment sums
    int32_t* rowcnt;   // [nchunks][nlong] finished-segment counters
    double* gslot;     // [nchunks][ngroups][C] group dot partials
    double* sslot;     // [nchunks][nsuper][C] super-group dot partials
    int32_t* scnt;     // [nchunks][nsuper] finished groups per super group
    int32_t* ccnt;     // [nchunks] finished super groups per chunk
    int32_t* queue;    // [2] work-queue head, exited warps
    const int32_t* chunk_active;  // optional per-chunk skip flags
    int32_t want_dot;
    DotHook hook;
};

// Fixed-order reduction of `nparts` per-CTA partials [nparts][C] of one chunk,
// executed by one CTA; returns the value for column threadIdx.x (< C).
template <int C>
__device__ __forceinline__ double reduce_partials(const double* part, int nparts, double* sm) {
    constexpr int TPC = kThreads / C;
    const int c = threadIdx.x % C, t = threadIdx.x / C;
    double s = 0.0;
    for (int q = t; q < nparts; q += TPC) s += __ldcg(part + static_cast<size_t>(q) * C + c);
    sm[t * C + c] = s;
    __syncthreads();
    double tot = 0.0;
    if (threadIdx.x < C) {
        for (int q = 0; q < TPC; ++q) tot += sm[q * C + threadIdx.x];
    }
    __syncthreads();
    return tot;
}

__device__ __forceinline__ void apply_dot_hook(const DotHook& h, int col, double v, int chunk) {
    if (h.mode == 0) {
        if (h.dots_out) h.dots_out[col] = v;
        return;
    }
    // mode 1: step length a = rs / (p.q) for columns active this iteration
    // (solver.py:83-87 for cg, 139-143 for lrc_pcg)
    if (col < h.b && h.active[col]) {
        if (h.dots_out) h.dots_out[col] = v;
        if (v <= 0.0) {
            h.status[col] = KZ_ENOTSPD;
            h.active[col] = 0;
            atomicExch(h.err, 1);
            atomicSub(h.n_active, 1);
        } else {
            h.alpha[col] = h.rs[col] / v;
            h.xstamp[col] = h.iter_dev ? *h.iter_dev : h.iter;
        }
    }
}

// Fixed-order sum over `cnt` partials of width C (stride C), one warp; lane
// c < C returns column c.  8 independent accumulators keep loads in flight;
// the combination order is fixed, so the result is deterministic.
template <int C>
__device__ __forceinline__ double warp_fixed_sum(const double* part, int cnt, int lane) {
    constexpr int LPC = (32 / C) < 8 ? (32 / C) : 8;  // lanes per column (<= 8)
    const int c = lane % C, sub = lane / C;
    double s = 0.0;
    if (sub < LPC) {
        // 8 independent loads per round: the reduction is a latency chain on
        // the tail of the launch (and the whole cost for small operators)
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        int q = sub;
        for (; q + 7 * LPC < cnt; q += 8 * LPC) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + static_cast<size_t>(q + u * LPC) * C + c);
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] += v[u] + v[u + 4];
        }
        for (; q < cnt; q += LPC) a[0] += __ldcg(part + static_cast<size_t>(q) * C + c);
        s = (a[0] + a[1]) + (a[2] + a[3]);
    }
#pragma unroll
    for (int off = C; off < C * LPC; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
}

// Persistent, warp-granular K1.  Every warp pulls groups of kGroupTasks
// consecutive tasks from one chunk-major queue (so the L2 working set stays
// about one chunk), runs them, and publishes the group's dot partial into
// its fixed slot.  The warp that completes a super group reduces its slots in
// order; the warp that completes a chunk's last super group reduces those
// and runs the CG/PCG hook.  No block-wide barrier anywhere.
template <int C, bool W>
__global__ void __launch_bounds__(kThreads, kSpmmMinBlocks) spmm_kernel(SpmmArgs a) {
    using K = Cfg<C>;
    constexpr int VEC = K::VEC;
    constexpr bool SD = (KZ_K1_SMEM_DOT != 0) && (C >= 32 || VEC == 4);
    __shared__ double s_dacc[SD ? VEC * kThreads : 1];
    const int lane = threadIdx.x & 31;
    const int gw = lane / K::G, lg = lane % K::G, gbase = gw * K::G;
    const unsigned gmask = (K::G == 32) ? 0xffffffffu : (((1u << K::G) - 1u) << gbase);
    const int total = a.ngroups * a.nchunks;
    // the solve loop issues one iteration ahead of its stop poll: when every
    // column has already stopped, leave at once instead of draining the
    // queue through masked chunks (the queue and counters stay armed; a
    // warp that skips still counts itself out below, so the last warp
    // re-arms the queue either way)
    int idle_l = 0;  // read by one lane: the loop below is warp-synchronous
    if (lane == 0)
        idle_l = a.hook.mode == 1 && a.hook.n_active &&
                 *reinterpret_cast<volatile const int32_t*>(a.hook.n_active) == 0;
    const bool idle = __shfl_sync(0xffffffffu, idle_l, 0) != 0;
    uint64_t pol_hub = 0, pol_tail = 0;
#if KZ_K1_L2HINT
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_hub));
    if (KZ_K1_L2HINT == 1)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_tail));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_tail));
#endif

    while (!idle) {
        int g = 0;
        if (lane == 0) g = atomicAdd(a.queue, 1);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= total) break;
        const int cq = g / a.ngroups, gl = g - cq * a.ngroups;
        const int chunk = a.chunk0 + cq;  // chunk0 > 0: per-chunk launches (KZ_K1_L2WINDOW_ROWS experiment)
        if (a.chunk_active && !a.chunk_active[chunk]) continue;
        const double* __restrict__ Xc = a.Xg + static_cast<size_t>(chunk) * a.ldxg;
        // wide chunks (32-byte gathers): the column-dot accumulators live in
        // shared memory (one slot per thread), not in registers across the
        // gather loop; narrow chunks keep them in registers
        double dacc_r[VEC];
        if constexpr (SD) {
#pragma unroll
            for (int q = 0; q < VEC; ++q) s_dacc[q * kThreads + threadIdx.x] = 0.0;
        } else {
#pragma unroll
            for (int q = 0; q < VEC; ++q) dacc_r[q] = 0.0;
        }

        auto epilogue = [&](int row, const double (&acc)[VEC]) {
            const size_t roff = static_cast<size_t>(row) * C + lg * VEC;
            double y[VEC];
            if (a.Xs) {
                double xs[VEC];
                ld_plain<VEC>(a.Xs + static_cast<size_t>(chunk) * a.ldxs + roff, xs);
#pragma unroll
                for (int q = 0; q < VEC; ++q)
                    y[q] = __dadd_rn(__dmul_rn(a.s1, xs[q]), __dmul_rn(a.s2, acc[q]));
            } else {
#pragma unroll
                for (int q = 0; q < VEC; ++q) y[q] = __dmul_rn(a.s2, acc[q]);
            }
            if (a.Z) {
                double z[VEC];
                ld_plain<VEC>(a.Z + static_cast<size_t>(chunk) * a.ldz + roff, z);
                if (a.s0v) {
                    const double* sv = a.s0v + chunk * C + lg * VEC;
#pragma unroll
                    for (int q = 0; q < VEC; ++q) y[q] = __dadd_rn(__dmul_rn(sv[q], z[q]), y[q]);
                } else {
#pragma unroll
                    for (int q = 0; q < VEC; ++q) y[q] = __dadd_rn(__dmul_rn(a.s0, z[q]), y[q]);
                }
            }
            st_stream<VEC>(a.Y + static_cast<size_t>(chunk) * a.ldy + roff, y);
            if (a.want_dot) {
                double d[VEC];
                ld_plain<VEC>(a.D ? a.D + static_cast<size_t>(chunk) * a.ldd + roff
                                  : a.Xs + static_cast<size_t>(chunk) * a.ldxs + roff, d);
#pragma unroll
                for (int q = 0; q < VEC; ++q) {
                    if constexpr (SD) {
                        double& da = s_dacc[q * kThreads + threadIdx.x];
                        da = fma(d[q], y[q], da);
                    } else {
                        dacc_r[q] = fma(d[q], y[q], dacc_r[q]);
                    }
                }
            }
        };
        auto warp_sum = [&](double (&v)[VEC]) {
#pragma unroll
            for (int off = K::G; off < 32; off <<= 1)
#pragma unroll
                for (int q = 0; q < VEC; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
        };

        const int t_end = a.group_first[gl + 1];
        for (int t = a.group_first[gl]; t < t_end; ++t) {
            const int4 task = a.tasks[t];
            KZ_DCHECK(task.x >= 0 && task.x < a.rows);
            if (task.z == TASK_S) {
                KZ_DCHECK(task.y <= a.rows);
                for (int row = task.x + gw; row < task.y; row += K::NGW) {
                    double acc[VEC];
#pragma unroll
                    for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
                    gather_rows<C, W>(a.colidx, a.rowptr[row], a.rowptr[row + 1], K::R, Xc, lg, gbase,
                                      gmask, acc, a.vals, a.hub_rows, pol_hub, pol_tail, a.cols);
                    epilogue(row, acc);
                }
            } else if (task.z == TASK_M) {
                const int row = task.x;
                double acc[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
                gather_rows<C, W>(a.colidx, a.rowptr[row] + gw * K::R, a.rowptr[row + 1], K::NGW * K::R,
                                  Xc, lg, gbase, gmask, acc, a.vals, a.hub_rows, pol_hub, pol_tail, a.cols);
                warp_sum(acc);
                if (gw == 0) epilogue(row, acc);
            } else {
                // long-row segment k of long row lidx
                const int row = task.x, lidx = task.y, k = task.w;
                const int s0 = a.long_seg0[lidx], nseg = a.long_seg0[lidx + 1] - s0;
                const int2 sr = a.seg_range[s0 + k];
                const int beg = sr.x, end = sr.y;
                KZ_DCHECK(k < nseg && beg >= a.rowptr[row] && end <= a.rowptr[row + 1]);
                double acc[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
                gather_rows<C, W>(a.colidx, beg + gw * K::R, end, K::NGW * K::R, Xc, lg, gbase, gmask,
                                  acc, a.vals, a.hub_rows, pol_hub, pol_tail, a.cols);
                warp_sum(acc);
                double* pbase = a.partial + static_cast<size_t>(chunk) * a.nseg * C;
                int* cnt = a.rowcnt + static_cast<size_t>(chunk) * a.nlong + lidx;
                if (k < nseg - 1) {
                    if (lane < K::G) {
                        st_plain<VEC>(pbase + static_cast<size_t>(s0 + k) * C + lg * VEC, acc);
                        __threadfence();
                    }
                    __syncwarp();
                    if (lane == 0) atomicAdd(cnt, 1);
                } else {
                    // last segment: the others were dequeued earlier by running
                    // warps; wait for them and combine in segment order
                    if (lane == 0) {
#if KZ_CHECKED
                        long long spins = 0;
                        while (atomicAdd(cnt, 0) < nseg - 1) {
                            __nanosleep(64);
                            KZ_DCHECK(++spins < (1ll << 26));  // a lost segment would hang here
                        }
#else
                        while (atomicAdd(cnt, 0) < nseg - 1) __nanosleep(64);
#endif
                        __threadfence();
                    }
                    __syncwarp();
                    double tot[VEC];
#pragma unroll
                    for (int q = 0; q < VEC; ++q) tot[q] = 0.0;
                    for (int s = 0; s < nseg - 1; ++s) {
                        const double* src = pbase + static_cast<size_t>(s0 + s) * C + lg * VEC;
#pragma unroll
                        for (int q = 0; q < VEC; ++q) tot[q] += __ldcg(src + q);
                    }
#pragma unroll
                    for (int q = 0; q < VEC; ++q) tot[q] += acc[q];
                    if (gw == 0) epilogue(row, tot);
                    __syncwarp();
                    if (lane == 0) *cnt = 0;  // re-arm for the next launch
                }
            }
        }
        if (!a.want_dot) continue;

        // ---- deterministic dot reduction: group -> super group -> chunk ----
        double dacc[VEC];
#pragma unroll
        for (int q = 0; q < VEC; ++q) dacc[q] = SD ? s_dacc[q * kThreads + threadIdx.x] : dacc_r[q];
        warp_sum(dacc);
        double* gs = a.gslot + (static_cast<size_t>(chunk) * a.ngroups + gl) * C;
        if (lane < K::G) {
            st_plain<VEC>(gs + lg * VEC, dacc);
            __threadfence();
        }
        __syncwarp();
        const int sg = gl / a.super_size;
        const int sg_groups = min(a.super_size, a.ngroups - sg * a.super_size);
        int last = 0;
        if (lane == 0)
            last = atomicAdd(a.scnt + static_cast<size_t>(chunk) * a.nsuper + sg, 1) == sg_groups - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence();
        const double sv = warp_fixed_sum<C>(a.gslot + (static_cast<size_t>(chunk) * a.ngroups + sg * a.super_size) * C,
                                            sg_groups, lane);
        if (lane < C) {
            a.sslot[(static_cast<size_t>(chunk) * a.nsuper + sg) * C + lane] = sv;
            __threadfence();
        }
        __syncwarp();
        int clast = 0;
        if (lane == 0) {
            a.scnt[static_cast<size_t>(chunk) * a.nsuper + sg] = 0;
            clast = atomicAdd(a.ccnt + chunk, 1) == a.nsuper - 1;
        }
        clast = __shfl_sync(0xffffffffu, clast, 0);
        if (!clast) continue;
        __threadfence();
        const double v = warp_fixed_sum<C>(a.sslot + static_cast<size_t>(chunk) * a.nsuper * C, a.nsuper, lane);
        if (lane < C) apply_dot_hook(a.hook, chunk * C + lane, v, chunk);
        __syncwarp();
        if (lane == 0) {
            a.ccnt[chunk] = 0;
            if (a.hook.mode == 1 && a.hook.chunk_xstamp)
                a.hook.chunk_xstamp[chunk] = a.hook.iter_dev ? *a.hook.iter_dev : a.hook.iter;
        }
    }
    // the last warp out re-arms the queue for the next launch
    if (lane == 0 && atomicAdd(a.queue + 1, 1) == a.nwarps - 1) {
        a.queue[0] = 0;
        a.queue[1] = 0;
    }
}

// Scratch needed by one SpMM launch over `nchunks` chunks of width C.
struct SpmmScratch {
    double* partial = nullptr;
    int32_t* rowcnt = nullptr;
    double* gslot = nullptr;
    double* sslot = nullptr;
    int32_t* scnt = nullptr;
    int32_t* ccnt = nullptr;
    int32_t* queue = nullptr;
    int64_t nlong_cap = 0, nsuper_cap = 0;
};

// Groups per super group: ~sqrt(ngroups) balances the two serial reductions
// at the end of a chunk (super group, then chunk); small operators would
// otherwise wait ~20 us on one warp summing 256 slots.
inline int spmm_super_size(int64_t ngroups) {
    int64_t s = static_cast<int64_t>(std::ceil(std::sqrt(static_cast<double>(std::max<int64_t>(ngroups, 1)))));
    return static_cast<int>(std::min<int64_t>(kSuperGroups, std::max<int64_t>(16, s)));
}
inline int64_t spmm_supers(int64_t ngroups) {
    const int64_t s = spmm_super_size(ngroups);
    return (ngroups + s - 1) / s;
}

// sizes for the largest of several operators (LRC reuses one scratch)
struct SpmmDims {
    int64_t nseg = 0, nlong = 0, ngroups = 0, nsuper = 0;
    void add(const kz_graph* g) {
        if (!g) return;
        nseg = std::max<int64_t>(nseg, g->nseg);
        nlong = std::max<int64_t>(nlong, g->nlong);
        ngroups = std::max<int64_t>(ngroups, g->ngroups);
        nsuper = std::max<int64_t>(nsuper, spmm_supers(g->ngroups));
    }
};

inline void carve_spmm_scratch(Carver& cv, const SpmmDims& d, int nchunks, int C, SpmmScratch& s) {
    s.partial = cv.take<double>(static_cast<size_t>(nchunks) * d.nseg * C + 1);
    s.gslot = cv.take<double>(static_cast<size_t>(nchunks) * d.ngroups * C + 1);
    s.sslot = cv.take<double>(static_cast<size_t>(nchunks) * d.nsuper * C + 1);
    s.rowcnt = cv.take<int32_t>(static_cast<size_t>(nchunks) * d.nlong + 1);
    s.scnt = cv.take<int32_t>(static_cast<size_t>(nchunks) * d.nsuper + 1);
    s.ccnt = cv.take<int32_t>(nchunks + 1);
    s.queue = cv.take<int32_t>(2);
    s.nlong_cap = d.nlong;
    s.nsuper_cap = d.nsuper;
}
inline void carve_spmm_scratch(Carver& cv, const kz_graph* g, int nchunks, int C, SpmmScratch& s) {
    SpmmDims d;
    d.add(g);
    carve_spmm_scratch(cv, d, nchunks, C, s);
}

// counters are re-armed by the kernels themselves; zero them once per call
inline int zero_spmm_counters(const SpmmDims& d, int nchunks, const SpmmScratch& s, cudaStream_t st) {
    const char* b0 = reinterpret_cast<const char*>(s.rowcnt);
    const char* b1 = reinterpret_cast<const char*>(s.queue + 2);
    KZ_CUDA(zero_span(const_cast<char*>(b0), const_cast<char*>(b1), st));
    (void)d;
    (void)nchunks;
    return KZ_OK;
}
inline int zero_spmm_counters(const kz_graph* g, int nchunks, const SpmmScratch& s, cudaStream_t st) {
    SpmmDims d;
    d.add(g);
    return zero_spmm_counters(d, nchunks, s, st);
}

inline SpmmArgs make_spmm_args(const kz_graph* g, const SpmmScratch& s) {
    SpmmArgs a{};
    a.rows = static_cast<int32_t>(g->rows);
    a.cols = static_cast<int32_t>(g->cols);
    a.rowptr = g->rowptr;
    a.colidx = g->colidx;
    a.tasks = g->tasks;
    a.long_seg0 = g->long_seg0;
    a.seg_range = g->seg_range;
    a.ntasks = g->ntasks;
    a.nlong = g->nlong;
    a.nseg = g->nseg;
    a.group_first = g->group_first;
    a.ngroups = g->ngroups;
    a.nsuper = static_cast<int32_t>(spmm_supers(g->ngroups));
    a.super_size = spmm_super_size(g->ngroups);
    a.partial = s.partial;
    a.rowcnt = s.rowcnt;
    a.gslot = s.gslot;
    a.sslot = s.sslot;
    a.scnt = s.scnt;
    a.ccnt = s.ccnt;
    a.queue = s.queue;
    return a;
}

inline int launch_spmm(const kz_graph* g, int C, int nchunks, SpmmArgs a, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(a.ngroups) * nchunks;
    if (total == 0) return KZ_OK;
    // persistent grid: at most one resident wave, at most one warp per group
    static const int ctas_per_sm = [] {
        const char* e = std::getenv("KZ_K1_CTAS");  // experiments: fewer resident CTAs per SM
        const int v = e ? std::atoi(e) : kSpmmMinBlocks;
        return v >= 1 && v <= kSpmmMinBlocks ? v : kSpmmMinBlocks;
    }();
    const int64_t cap = static_cast<int64_t>(num_sms()) * ctas_per_sm;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cap, (total + kWarps - 1) / kWarps)));
    a.nchunks = nchunks;
    a.nwarps = static_cast<int32_t>(grid) * kWarps;
    if (a.ldxg == 0) a.ldxg = g->cols * C;
    if (a.ldxs == 0) a.ldxs = g->rows * C;
    if (a.ldz == 0) a.ldz = g->rows * C;
    if (a.ldy == 0) a.ldy = g->rows * C;
    if (a.ldd == 0) a.ldd = g->rows * C;
    a.vals = g->vals;
    const bool w = g->vals != nullptr;
#if KZ_K1_L2HINT || KZ_K1_L1HINT
    static const int hub_rows_env = [] {
        const char* e = std::getenv("KZ_K1_HUBROWS");
        return e ? std::atoi(e) : 131072;
    }();
    a.hub_rows = hub_rows_env;
#endif
    cudaEvent_t tev = nullptr;
    if (k1_timing_on()) k1_timing_begin(st, &tev);
    // experiments: KZ_K1_CARVEOUT = preferred shared-memory carveout (percent)
    static const int carveout = [] {
        const char* e = std::getenv("KZ_K1_CARVEOUT");
        return e ? std::atoi(e) : -1;
    }();
    // experiment: one launch per chunk with an L2 persisting
    // access-policy window over the chunk's first KZ_K1_L2WINDOW_ROWS rows of Xg
    // (the hub rows in the degree-class order); KZ_K1_L2WINDOW_MB = set-aside size
    static const int win_rows = [] {
        const char* e = std::getenv("KZ_K1_L2WINDOW_ROWS");
        return e ? std::atoi(e) : 0;
    }();
    if (win_rows > 0 && C == 32 && !w && nchunks > 1 && a.chunk0 == 0 && !tev) {
        static const bool set_aside = [] {
            const char* e = std::getenv("KZ_K1_L2WINDOW_MB");
            const size_t mb = e ? std::atoi(e) : 40;
            return cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, mb << 20) == cudaSuccess;
        }();
        (void)set_aside;
        static const float hit_ratio = [] {
            const char* e = std::getenv("KZ_K1_L2WINDOW_HIT");
            return e ? static_cast<float>(std::atof(e)) : 1.0f;
        }();
        for (int c = 0; c < nchunks; ++c) {
            cudaStreamAttrValue attr{};
            attr.accessPolicyWindow.base_ptr = const_cast<double*>(a.Xg) + static_cast<size_t>(c) * a.ldxg;
            attr.accessPolicyWindow.num_bytes = static_cast<size_t>(std::min<int64_t>(win_rows, g->cols)) * C * sizeof(double);
            attr.accessPolicyWindow.hitRatio = hit_ratio;
            attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr);
            SpmmArgs ac = a;
            ac.chunk0 = c;
            ac.nchunks = 1;
            const int64_t tot1 = a.ngroups;
            const unsigned grid1 = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cap, (tot1 + kWarps - 1) / kWarps)));
            ac.nwarps = static_cast<int32_t>(grid1) * kWarps;
            spmm_kernel<32, false><<<grid1, kThreads, 0, st>>>(ac);
            note_launch();
        }
        cudaStreamAttrValue off{};
        off.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &off);
        KZ_LAUNCH_CHECK();
        return KZ_OK;
    }
#define KZ_SPMM_CASE(CC)                                                                  \
    case CC:                                                                              \
        if (carveout >= 0) {                                                              \
            cudaFuncSetAttribute(spmm_kernel<CC, true>,                                   \
                                 cudaFuncAttributePreferredSharedMemoryCarveout, carveout); \
            cudaFuncSetAttribute(spmm_kernel<CC, false>,                                  \
                                 cudaFuncAttributePreferredSharedMemoryCarveout, carveout); \
        }                                                                                 \
        if (w) spmm_kernel<CC, true><<<grid, kThreads, 0, st>>>(a);                        \
        else spmm_kernel<CC, false><<<grid, kThreads, 0, st>>>(a);                         \
        break;
    switch (C) {
        KZ_SPMM_CASE(1)
        KZ_SPMM_CASE(2)
        KZ_SPMM_CASE(4)
        KZ_SPMM_CASE(8)
        KZ_SPMM_CASE(16)
        KZ_SPMM_CASE(32)
        KZ_SPMM_CASE(64)
        default:
            if (tev) cudaEventDestroy(tev);
            return fail(KZ_EARG, "unsupported chunk width");
    }
#undef KZ_SPMM_CASE
    if (tev) k1_timing_end(st, tev);
    note_launch();
    KZ_LAUNCH_CHECK();
    return KZ_OK;
}

}  // namespace kz
