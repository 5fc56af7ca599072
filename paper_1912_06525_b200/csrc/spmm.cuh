// spmm.cuh -- K1: binary-pattern CSR SpMM with fused epilogue and column dots.
//
//   Y = s0*Z + (s1*Xs + s2*(A Xg))         (per row, per column of the block)
//   dots[j] = sum_i D[i,j] * Y[i,j]        (optional, deterministic)
//
// Replaces the reference's operator applications: KatzIndex.apply_m_permuted
// (index.py:86-91: x - alpha*A x through factor reassembly), the coupling
// products m12 @ v / m12.T @ u (solver.py:110,115,178) and the rhs column
// (index.py:93-101).  A is a binary pattern (no stored values, int32 column
// indices), so the only per-nonzero traffic is 4 bytes of index plus a
// gathered C-wide row segment of Xg.
//
// Layout: blocks are chunked node-major [b/C][rows][C] (C doubles of one row
// are contiguous, 16*C bytes... i.e. 8*C bytes), so one gathered neighbour is a
// coalesced 8*C-byte segment read by G = C/VEC lanes with 16-byte vector
// loads.  The grid is chunk-major, so at any moment the L2 working set is
// one chunk of Xg (rows*8*C bytes) rather than the whole block.
//
// Power-law degree skew: rows with deg <= seg ("short") are handled by one
// lane group each, in CSR order, so their sum is bit-identical to scipy's
// csr_matvec.  Longer rows are cut into seg-long segments processed by whole
// warps in dedicated CTAs (launched first in each chunk); their partial sums
// are combined in a fixed order by the CTA that owns the row's range, which
// waits on a per-row completion counter (stream-K style fix-up).  All dot
// partials are reduced in a fixed order by the last CTA of the chunk, so the
// result is run-to-run deterministic.
#pragma once

#include "common.cuh"

struct kz_graph {
    int64_t rows = 0, cols = 0, nnz = 0;
    int32_t* rowptr = nullptr;  // device int32[rows+1]
    int32_t* colidx = nullptr;  // device int32[nnz]
    int32_t seg = 512;          // long-row segment length
    int32_t nlong = 0;          // rows with degree > seg
    int32_t nitems = 0;         // seg-long segments of the long rows
    int32_t* long_rows = nullptr;   // [nlong] sorted row ids
    int32_t* long_first = nullptr;  // [nlong+1] first segment of each long row
    int32_t* item_lrow = nullptr;   // [nitems] owning long-row index
    int32_t nshort = 0;             // row-range CTAs per chunk
    int32_t* cta_rows = nullptr;    // [nshort+1] row ranges (cost balanced)
    int32_t* cta_long = nullptr;    // [nshort+1] long-row index ranges per CTA
    int32_t nlongcta = 0;           // segment CTAs per chunk
    int32_t max_deg = 0;
};

namespace kz {

template <int C>
struct Cfg {
    static constexpr int VEC = (C >= 2) ? 2 : 1;  // doubles per lane (16-byte loads)
    static constexpr int G = C / VEC;             // lanes per row group
    static constexpr int NGW = 32 / G;            // row groups per warp
    static constexpr int R = (G >= 4) ? G : 4;    // neighbours gathered per round
    static constexpr int PER = R / G;             // column indices loaded per lane per round
};

template <int VEC>
__device__ __forceinline__ void ld_nc(const double* p, double (&v)[VEC]);
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
template <int VEC>
__device__ __forceinline__ void ld_plain(const double* p, double (&v)[VEC]) {
    if constexpr (VEC == 2) {
        double2 t = *reinterpret_cast<const double2*>(p);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = *p;
    }
}
template <int VEC>
__device__ __forceinline__ void st_plain(double* p, const double (&v)[VEC]) {
    if constexpr (VEC == 2) {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    } else {
        *p = v[0];
    }
}

// Sum Xg rows of neighbours col[beg..end) into acc, R neighbours per round,
// rounds `stride` apart.  All lanes of a group share the neighbour; lane lg
// owns columns lg*VEC .. lg*VEC+VEC-1 of the chunk.
template <int C>
__device__ __forceinline__ void gather_rows(const int32_t* __restrict__ col, int beg, int end,
                                            int stride, const double* __restrict__ Xc, int lg,
                                            int gbase, unsigned gmask,
                                            double (&acc)[Cfg<C>::VEC]) {
    using K = Cfg<C>;
    for (int base = beg; base < end; base += stride) {
        int idx[K::PER];
#pragma unroll
        for (int m = 0; m < K::PER; ++m) {
            const int pos = base + lg + K::G * m;
            idx[m] = (pos < end) ? __ldg(col + pos) : -1;
        }
        double v[K::R][K::VEC];
        int jj[K::R];
#pragma unroll
        for (int t = 0; t < K::R; ++t) {
            int j;
            if constexpr (K::G == 1)
                j = idx[t];
            else
                j = __shfl_sync(gmask, idx[t / K::G], gbase + (t % K::G));
            jj[t] = j;
            if (j >= 0)
                ld_nc<K::VEC>(Xc + static_cast<size_t>(j) * C + lg * K::VEC, v[t]);
        }
#pragma unroll
        for (int t = 0; t < K::R; ++t)
            if (jj[t] >= 0) {
#pragma unroll
                for (int q = 0; q < K::VEC; ++q) acc[q] = __dadd_rn(acc[q], v[t][q]);
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
};

struct SpmmArgs {
    int32_t rows, cols;
    const int32_t* __restrict__ rowptr;
    const int32_t* __restrict__ colidx;
    int32_t seg, nlong, nitems, nshort, nlongcta;
    const int32_t* long_rows;
    const int32_t* long_first;
    const int32_t* item_lrow;
    const int32_t* cta_rows;
    const int32_t* cta_long;
    const double* Xg;
    const double* Xs;
    const double* Z;
    double* Y;
    const double* D;
    double s0, s1, s2;
    double* partial;
    int32_t* rowcnt;
    double* dotcta;
    int32_t* chunkcnt;
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
            h.xstamp[col] = h.iter;
        }
    }
}

template <int C>
__global__ void __launch_bounds__(kThreads) spmm_kernel(SpmmArgs a) {
    using K = Cfg<C>;
    constexpr int VEC = K::VEC;
    const int per_chunk = a.nlongcta + a.nshort;
    const int chunk = blockIdx.x / per_chunk;
    const int local = blockIdx.x - chunk * per_chunk;
    if (a.chunk_active && !a.chunk_active[chunk]) return;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = lane / K::G, lg = lane % K::G, gbase = gw * K::G;
    const unsigned gmask = (K::G == 32) ? 0xffffffffu : (((1u << K::G) - 1u) << gbase);
    const double* __restrict__ Xc = a.Xg + static_cast<size_t>(chunk) * a.cols * C;

    if (local < a.nlongcta) {
        // ---- long-row segments: one warp per segment, partial sums out ----
        const int nw_total = a.nlongcta * kWarps;
        for (int it = local * kWarps + warp; it < a.nitems; it += nw_total) {
            const int lr = a.item_lrow[it];
            const int row = a.long_rows[lr];
            const int k = it - a.long_first[lr];
            const int beg = a.rowptr[row] + k * a.seg;
            const int end = min(beg + a.seg, a.rowptr[row + 1]);
            double acc[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
            gather_rows<C>(a.colidx, beg + gw * K::R, end, K::NGW * K::R, Xc, lg, gbase, gmask,
                           acc);
#pragma unroll
            for (int off = K::G; off < 32; off <<= 1)
#pragma unroll
                for (int q = 0; q < VEC; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
            if (lane < K::G) {
                st_plain<VEC>(a.partial + (static_cast<size_t>(chunk) * a.nitems + it) * C +
                                  lg * VEC,
                              acc);
                __threadfence();
            }
            __syncwarp();
            if (lane == 0) atomicAdd(a.rowcnt + static_cast<size_t>(chunk) * a.nlong + lr, 1);
        }
        return;
    }

    // ---- row-range CTA: short rows by lane groups, then owned long rows ----
    const int p = local - a.nlongcta;
    const int rb = a.cta_rows[p], re = a.cta_rows[p + 1];
    const int ngroups = kWarps * K::NGW;
    const int gid = warp * K::NGW + gw;
    double dacc[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) dacc[q] = 0.0;

    auto epilogue = [&](int row, const double (&acc)[VEC]) {
        const size_t off = (static_cast<size_t>(chunk) * a.rows + row) * C + lg * VEC;
        double y[VEC];
        if (a.Xs) {
            double xs[VEC];
            ld_plain<VEC>(a.Xs + off, xs);
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                y[q] = __dadd_rn(__dmul_rn(a.s1, xs[q]), __dmul_rn(a.s2, acc[q]));
        } else {
#pragma unroll
            for (int q = 0; q < VEC; ++q) y[q] = __dmul_rn(a.s2, acc[q]);
        }
        if (a.Z) {
            double z[VEC];
            ld_plain<VEC>(a.Z + off, z);
#pragma unroll
            for (int q = 0; q < VEC; ++q) y[q] = __dadd_rn(__dmul_rn(a.s0, z[q]), y[q]);
        }
        st_plain<VEC>(a.Y + off, y);
        if (a.want_dot) {
            double d[VEC];
            ld_plain<VEC>((a.D ? a.D : a.Xs) + off, d);
#pragma unroll
            for (int q = 0; q < VEC; ++q) dacc[q] = fma(d[q], y[q], dacc[q]);
        }
    };

    for (int row = rb + gid; row < re; row += ngroups) {
        const int beg = a.rowptr[row], end = a.rowptr[row + 1];
        if (end - beg > a.seg) continue;  // long row: finished below
        double acc[VEC];
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
        gather_rows<C>(a.colidx, beg, end, K::R, Xc, lg, gbase, gmask, acc);
        epilogue(row, acc);
    }

    // long rows whose range this CTA owns: wait for their segments, combine
    // the partials in segment order, run the epilogue
    const int l0 = a.cta_long[p], l1 = a.cta_long[p + 1];
    for (int lr = l0 + warp; lr < l1; lr += kWarps) {
        const int row = a.long_rows[lr];
        const int f = a.long_first[lr], nseg = a.long_first[lr + 1] - f;
        int* cnt = a.rowcnt + static_cast<size_t>(chunk) * a.nlong + lr;
        if (lane == 0) {
            while (atomicAdd(cnt, 0) < nseg) __nanosleep(100);
            __threadfence();
        }
        __syncwarp();
        double acc[VEC];
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
        for (int s = gw; s < nseg; s += K::NGW) {
            const double* src =
                a.partial + (static_cast<size_t>(chunk) * a.nitems + f + s) * C + lg * VEC;
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] += __ldcg(src + q);
        }
#pragma unroll
        for (int off = K::G; off < 32; off <<= 1)
#pragma unroll
            for (int q = 0; q < VEC; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
        if (gw == 0) epilogue(row, acc);
        __syncwarp();
        if (lane == 0) *cnt = 0;  // re-arm for the next launch
    }

    if (!a.want_dot) return;

    // ---- deterministic column dots: warp -> CTA -> chunk ----
#pragma unroll
    for (int off = K::G; off < 32; off <<= 1)
#pragma unroll
        for (int q = 0; q < VEC; ++q) dacc[q] += __shfl_xor_sync(0xffffffffu, dacc[q], off);
    __shared__ double sm[kThreads];
    __shared__ int is_last;
    if (lane < K::G) {
#pragma unroll
        for (int q = 0; q < VEC; ++q) sm[warp * C + lg * VEC + q] = dacc[q];
    }
    __syncthreads();
    if (threadIdx.x < C) {
        double s = 0.0;
        for (int w = 0; w < kWarps; ++w) s += sm[w * C + threadIdx.x];
        a.dotcta[(static_cast<size_t>(chunk) * a.nshort + p) * C + threadIdx.x] = s;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int old = atomicAdd(a.chunkcnt + chunk, 1);
        is_last = (old == a.nshort - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const double v =
        reduce_partials<C>(a.dotcta + static_cast<size_t>(chunk) * a.nshort * C, a.nshort, sm);
    if (threadIdx.x < C) apply_dot_hook(a.hook, chunk * C + threadIdx.x, v, chunk);
    if (threadIdx.x == 0) {
        a.chunkcnt[chunk] = 0;
        if (a.hook.mode == 1 && a.hook.chunk_xstamp) a.hook.chunk_xstamp[chunk] = a.hook.iter;
    }
}

// Scratch needed by one SpMM launch over `nchunks` chunks of width C.
struct SpmmScratch {
    double* partial = nullptr;
    int32_t* rowcnt = nullptr;
    double* dotcta = nullptr;
    int32_t* chunkcnt = nullptr;
};

inline void carve_spmm_scratch(Carver& cv, const kz_graph* g, int nchunks, int C, SpmmScratch& s) {
    s.partial = cv.take<double>(static_cast<size_t>(nchunks) * g->nitems * C + 1);
    s.rowcnt = cv.take<int32_t>(static_cast<size_t>(nchunks) * g->nlong + 1);
    s.dotcta = cv.take<double>(static_cast<size_t>(nchunks) * g->nshort * C + 1);
    s.chunkcnt = cv.take<int32_t>(nchunks + 1);
}

inline int zero_spmm_counters(const kz_graph* g, int nchunks, const SpmmScratch& s,
                              cudaStream_t st) {
    KZ_CUDA(cudaMemsetAsync(s.rowcnt, 0, sizeof(int32_t) * (static_cast<size_t>(nchunks) * g->nlong + 1), st));
    KZ_CUDA(cudaMemsetAsync(s.chunkcnt, 0, sizeof(int32_t) * (nchunks + 1), st));
    return KZ_OK;
}

inline SpmmArgs make_spmm_args(const kz_graph* g, const SpmmScratch& s) {
    SpmmArgs a{};
    a.rows = static_cast<int32_t>(g->rows);
    a.cols = static_cast<int32_t>(g->cols);
    a.rowptr = g->rowptr;
    a.colidx = g->colidx;
    a.seg = g->seg;
    a.nlong = g->nlong;
    a.nitems = g->nitems;
    a.nshort = g->nshort;
    a.nlongcta = g->nlongcta;
    a.long_rows = g->long_rows;
    a.long_first = g->long_first;
    a.item_lrow = g->item_lrow;
    a.cta_rows = g->cta_rows;
    a.cta_long = g->cta_long;
    a.partial = s.partial;
    a.rowcnt = s.rowcnt;
    a.dotcta = s.dotcta;
    a.chunkcnt = s.chunkcnt;
    return a;
}

inline int launch_spmm(const kz_graph* g, int C, int nchunks, const SpmmArgs& a,
                       cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(nchunks) * (g->nlongcta + g->nshort);
    switch (C) {
        case 1: spmm_kernel<1><<<grid, kThreads, 0, st>>>(a); ::kz::note_launch(); break;
        case 2: spmm_kernel<2><<<grid, kThreads, 0, st>>>(a); ::kz::note_launch(); break;
        case 4: spmm_kernel<4><<<grid, kThreads, 0, st>>>(a); ::kz::note_launch(); break;
        case 8: spmm_kernel<8><<<grid, kThreads, 0, st>>>(a); ::kz::note_launch(); break;
        case 16: spmm_kernel<16><<<grid, kThreads, 0, st>>>(a); ::kz::note_launch(); break;
        case 32: spmm_kernel<32><<<grid, kThreads, 0, st>>>(a); ::kz::note_launch(); break;
        default: return fail(KZ_EARG, "unsupported chunk width");
    }
    KZ_LAUNCH_CHECK();
    return KZ_OK;
}

}  // namespace kz
