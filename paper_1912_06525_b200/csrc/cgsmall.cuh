// cgsmall.cuh -- a whole small batched CG solve in ONE cooperative kernel.
// At cfg1 sizes (n ~ 10^4, 16 columns) the vector blocks sit in L2 and every
// separate kernel, memset and copy of the host- or graph-driven loop costs
// more in launch, tail and cross-CTA-reduction latency than in work; here the
// right-hand side, the CG iterations, the output store and the reports are
// one launch with three grid barriers per iteration.
//
// Per iteration, exactly the reference recurrence of cg() (solver.py:78-95)
// for every column:
//   1  q = p - beta*A p over a merge-path share of (rows + entries) per warp
//      (K1's pipelined row gathers, L1-cached: the hub rows every warp
//      gathers stay on the SM; each grid barrier is preceded by a gpu-scope
//      fence, which invalidates L1); a row split
//      across warps leaves its earlier parts as carries, published with a
//      per-(warp, chunk) iteration stamp, and the warp owning the row's end
//      adds them in warp order; p.q partials per CTA
//   2  every CTA reduces the CTA partials in a fixed order, a = rs/pq
//      (non-positive curvature: the column errs and the solve stops),
//      r -= a*q over its share, r.r partials per CTA
//   3  every CTA reduces r.r, applies the stop test / budget, b = rs'/rs,
//      then x += a*p and p = r + b*p over its share
// Every CTA derives the same per-column scalars from the same partials in
// the same order (no broadcast step), so results are run-to-run
// deterministic; CTA 0 publishes the per-column state and the reports.
// With `init` the kernel also forms r0 = p0 = beta*A e_q (index.py:93-101),
// ||b|| and the start state (solver.py:71-77) itself, and with `scores` it
// stores clamp(x) through perm (solver.py:223-225).
#pragma once

#include <cooperative_groups.h>

#include <mutex>
#include <utility>
#include <vector>

#include "blockops.cuh"

namespace kz {

constexpr int kSmallCgThreads = 256;
constexpr int kSmallCgMaxCols = 256;                   // columns (bpad) the fused loop handles
constexpr size_t kSmallCgElems = size_t(1) << 22;      // block size (doubles) up to which it is used
constexpr int64_t kSmallCgMaxNnz = int64_t(1) << 24;   // ... and operator entries
constexpr int kSmallCgWarps = kSmallCgThreads / 32;
#ifndef KZ_SMALL_CTAS
#define KZ_SMALL_CTAS 1  // resident CTAs per SM (more: longer barriers and reductions, measured slower)
#endif
constexpr int kSmallCgCtasPerSm = KZ_SMALL_CTAS;
constexpr int32_t kSmallCgWarpRow = 32;  // rows longer than this are gathered by the whole warp
// (entries + rows) * columns up to which the fused loop is used: its 8 warps
// per SM hide less gather latency than K1's 40, so above ~10^7 (R-MAT 16 at
// 64 columns: 1.2e8) the host-driven loop is faster (2.8 vs ~1.5 ms)
constexpr double kSmallCgMaxWork = 1e7;

struct SmallCgArgs {
    int32_t rows, nchunks, b, bpad;
    const int32_t* rowptr;
    const int32_t* colidx;
    double beta;
    double *x, *r, *p, *q;  // chunked blocks [nchunks][rows][C]
    double* part;           // [2][gridDim.x][bpad] CTA partials (two phases in flight)
    double* carry;          // [nwarps][bpad] split-row partials published by each warp
    int32_t* stamp;         // [nwarps][nchunks] iteration whose carry is published
    SolveState s;
    // init: r0 = p0 = beta*A e_q from qpos, x0 = 0, the start state
    int init;
    const int64_t* qpos;    // device [b]
    // output (scores != NULL): scores[j][perm ? perm[i] : i] = clamp(x_j[i]); reports[j]
    double* scores;
    const int64_t* perm;
    int clamp;
    kz_report* reports;     // device [b]
};

// the row holding merged position pos (row i starts at rowptr[i] + i): the
// largest i with rowptr[i] + i <= pos
__device__ __forceinline__ int32_t merge_row(const int32_t* rowptr, int32_t n, int64_t pos) {
    int32_t lo = 0, hi = n;
    while (lo < hi) {
        const int32_t mid = (lo + hi + 1) >> 1;
        if (static_cast<int64_t>(rowptr[mid]) + mid <= pos) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// the warp whose merge-path share [total*w/nw, total*(w+1)/nw) holds pos
__device__ __forceinline__ int warp_of(int64_t pos, int64_t total, int nw) {
    int w = static_cast<int>(pos * nw / total);
    while (w + 1 < nw && total * (w + 1) / nw <= pos) ++w;
    while (w > 0 && total * w / nw > pos) --w;
    return w;
}

#ifdef KZ_SMALL_DEBUG
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define KZ_PT(k) \
    if (blockIdx.x == 0 && threadIdx.x == 0) ph[k] += gtimer() - t0, t0 = gtimer();
__device__ unsigned long long g_slowest_warp;  // (phase-1 ns << 20) | warp of the slowest warp, last iteration
__device__ unsigned int g_wt[8192];            // per-warp phase-1 ns, last iteration
__device__ unsigned int g_wt2[8192];           // per-warp ns until the end of the gathers (before the CTA partial)
#else
#define KZ_PT(k)
#endif

template <int C>
__global__ void __launch_bounds__(kSmallCgThreads, kSmallCgCtasPerSm) cg_small_kernel(SmallCgArgs a) {
#ifdef KZ_SMALL_DEBUG
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t0 = gtimer();
#endif
    namespace cgr = cooperative_groups;
    cgr::grid_group grid = cgr::this_grid();
    using K = Cfg<C>;
    constexpr int VEC = K::VEC;
    __shared__ double s_red[kSmallCgThreads];
    __shared__ double s_red2[kSmallCgWarps * 32];  // [warp][C] group-0 column partials
    __shared__ double s_a[kSmallCgMaxCols], s_b[kSmallCgMaxCols], s_rs[kSmallCgMaxCols];
    __shared__ int s_on[kSmallCgMaxCols], s_act[kSmallCgMaxCols], s_chunk[kSmallCgMaxCols];
    __shared__ int s_any, s_err;
    const SolveState& s = a.s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * kSmallCgWarps + warp, nw = gridDim.x * kSmallCgWarps;
    const int64_t ld = static_cast<int64_t>(a.rows) * C;
    const int nch = a.nchunks, bpad = a.bpad;
    const int lg = lane % K::G, grp = lane / K::G, gbase = grp * K::G;
    const unsigned gmask = (K::G == 32) ? 0xffffffffu : (((1u << K::G) - 1u) << gbase);
    // merge-path share [S, E) of this warp; rows rs0 .. rs1 intersect it
    const int64_t total = static_cast<int64_t>(a.rowptr[a.rows]) + a.rows;
    const int64_t S = total * gw / nw, E = total * (gw + 1) / nw;
    const bool has = S < E;
    const int32_t rs0 = has ? merge_row(a.rowptr, a.rows, S) : 0;
    const int32_t rs1 = has ? merge_row(a.rowptr, a.rows, E - 1) : -1;
    auto row_start = [&](int32_t i) { return static_cast<int64_t>(a.rowptr[i]) + i; };
    auto row_endpos = [&](int32_t i) { return static_cast<int64_t>(a.rowptr[i + 1]) + i; };  // the row-end item
    const bool first_split = has && row_start(rs0) < S && row_endpos(rs0) < E;  // owns the end of a split row
    const int w0 = first_split ? warp_of(row_start(rs0), total, nw) : gw;    // ... whose start is in warp w0
    double* carry_last = a.carry;
    // element share of this CTA inside each chunk: rows [e0, e1)
    const int32_t e0 = static_cast<int32_t>(static_cast<int64_t>(a.rows) * blockIdx.x / gridDim.x);
    const int32_t e1 = static_cast<int32_t>(static_cast<int64_t>(a.rows) * (blockIdx.x + 1) / gridDim.x);
    double* partA = a.part;
    double* partB = a.part + static_cast<size_t>(gridDim.x) * bpad;

    if (a.init) {
        // ---- r0 = p0 = beta*A e_q, x0 = 0; ||b||; the start state ----
        for (int ch = 0; ch < nch; ++ch)
            for (int64_t e = static_cast<int64_t>(e0) * C + threadIdx.x; e < static_cast<int64_t>(e1) * C;
                 e += kSmallCgThreads) {
                const size_t o = static_cast<size_t>(ch) * ld + e;
                a.x[o] = 0.0;
                a.r[o] = 0.0;
                a.p[o] = 0.0;
            }
    }
    // carry stamps of an earlier solve on this workspace must not match
    for (int i = blockIdx.x * kSmallCgThreads + threadIdx.x; i < nw * nch; i += gridDim.x * kSmallCgThreads)
        a.stamp[i] = 0;
    __threadfence();
    grid.sync();
    if (a.init) {
        for (int j = blockIdx.x; j < bpad; j += gridDim.x) {
            const int ch = j / C, c = j % C;
            if (j < a.b) {
                const int64_t q = a.qpos[j];
                const int32_t beg = a.rowptr[q], end = a.rowptr[q + 1];
                for (int32_t e = beg + threadIdx.x; e < end; e += kSmallCgThreads) {
                    const size_t o = static_cast<size_t>(ch) * ld + static_cast<size_t>(a.colidx[e]) * C + c;
                    a.r[o] = a.beta;
                    a.p[o] = a.beta;
                }
            }
            if (threadIdx.x == 0) {
                // ||b||^2 = sum over N(q) of beta^2, in CSR order (solver.py:71)
                double bn2 = 0.0;
                if (j < a.b) {
                    const int32_t deg = a.rowptr[a.qpos[j] + 1] - a.rowptr[a.qpos[j]];
                    for (int32_t k = 0; k < deg; ++k) bn2 = fma(a.beta, a.beta, bn2);
                }
                s.bnorm2[j] = bn2;
                const double bn = sqrt(bn2);
                s.thresh[j] = s.tol * bn;
                s.rnorm[j] = bn;
                s.rs[j] = bn2;
                s.iters[j] = 0;
                s.status[j] = 0;
                const bool act = j < a.b && bn > s.thresh[j];
                s.active[j] = act ? 1 : 0;
                s.converged[j] = act ? 0 : 1;
            }
        }
        __threadfence();
        grid.sync();
    }
    for (int c = threadIdx.x; c < bpad; c += kSmallCgThreads) {
        s_act[c] = c < a.b ? __ldcg(s.active + c) : 0;
        s_rs[c] = __ldcg(s.rs + c);
    }
    __syncthreads();
    auto chunk_flags = [&]() {
        // phase 3's x / p update still reads s_chunk: no thread may rewrite the
        // flags before every warp of the CTA has left that loop (without this
        // barrier a fast warp could clear a chunk's flag -- its last column
        // just converged -- while slower warps had not started that chunk, and
        // their rows of x missed the final update; found by tools/fuzz_parity.py)
        __syncthreads();
        if (threadIdx.x < nch) {
            int any = 0;
            for (int c = 0; c < C; ++c) any |= s_act[threadIdx.x * C + c];
            s_chunk[threadIdx.x] = any;
        }
        if (threadIdx.x == 0) {
            int any = 0;
            for (int c = 0; c < bpad; ++c) any |= s_act[c];
            s_any = any;
        }
        __syncthreads();
    };
    // per-thread values of one chunk (thread t holds column t % C) -> CTA partial
    auto cta_partial = [&](double v, int chunk, double* part) {
        s_red[threadIdx.x] = v;
        __syncthreads();
        if (threadIdx.x < C) {
            double t = 0.0;
            for (int k = threadIdx.x; k < kSmallCgThreads; k += C) t += s_red[k];
            part[static_cast<size_t>(blockIdx.x) * bpad + chunk * C + threadIdx.x] = t;
        }
        __syncthreads();
    };
    // every CTA: the column totals of the CTA partials, in a fixed order
    // (TPC threads per column sum strided subsets -- all loads issued
    // before the adds -- then a fixed tree)
    auto reduce_cols = [&](const double* part, double* out) {
        int TPC = 1;
        while (TPC * 2 * bpad <= kSmallCgThreads) TPC *= 2;
        const int G = static_cast<int>(gridDim.x);
        for (int base = 0; base < bpad; base += kSmallCgThreads / TPC) {
            const int c = base + static_cast<int>(threadIdx.x) / TPC, sub = threadIdx.x % TPC;
            double t = 0.0;
            if (c < bpad) {
                for (int k0 = sub; k0 < G; k0 += 8 * TPC) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int k = k0 + u * TPC;
                        v[u] = k < G ? __ldcg(part + static_cast<size_t>(k) * bpad + c) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) t += v[u];
                }
            }
            s_red[threadIdx.x] = t;
            __syncthreads();
            for (int w = TPC / 2; w > 0; w >>= 1) {
                if (sub < w) s_red[threadIdx.x] += s_red[threadIdx.x + w];
                __syncthreads();
            }
            if (sub == 0 && c < bpad) out[c] = s_red[threadIdx.x];
            __syncthreads();
        }
    };
    chunk_flags();
    int64_t it = 0;
    for (;;) {
        if (!s_any || it >= s.max_iter) break;
        ++it;
        KZ_PT(0);
#ifdef KZ_SMALL_DEBUG
        const unsigned long long w_t0 = gtimer();
        if (gw == 0 && lane == 0) g_slowest_warp = 0;
#endif
        // ---- phase 1: q = p - beta*A p over the merge-path share, p.q partials.
        // Rows wholly inside the share run one per lane group (K1's short-row
        // gather: R neighbours in flight, next indices prefetched); the split
        // pieces at either end run across the whole warp.
        for (int ch = 0; ch < nch; ++ch) {
            double dot[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) dot[v] = 0.0;
            if (s_chunk[ch] && has) {
                const double* pc = a.p + static_cast<size_t>(ch) * ld;
                double* qc = a.q + static_cast<size_t>(ch) * ld;
                const bool start0 = row_start(rs0) >= S;
                const int32_t in0 = start0 ? rs0 : rs0 + 1;
                const int32_t in1 = row_endpos(rs1) < E ? rs1 : rs1 - 1;
                auto finish = [&](int32_t i, const double (&acc)[VEC]) {  // q_i and its p.q term
                    double pv[VEC], qv[VEC];
                    ld_plain<VEC>(pc + static_cast<size_t>(i) * C + lg * VEC, pv);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) {
                        qv[v] = __dadd_rn(pv[v], __dmul_rn(-a.beta, acc[v]));
                        dot[v] = fma(pv[v], qv[v], dot[v]);
                    }
                    st_plain<VEC>(qc + static_cast<size_t>(i) * C + lg * VEC, qv);
                };
                // whole-warp gather of entries [beg, end), summed over the lane groups
                auto piece = [&](int32_t beg, int32_t end, double (&acc)[VEC]) {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
                    gather_rows<C, false, true>(a.colidx, beg + grp * K::R, end, K::NGW * K::R, pc, lg, gbase, gmask,
                                                acc);
#pragma unroll
                    for (int off = K::G; off < 32; off <<= 1)
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);
                };
                // rows inside the share: long ones across the whole warp (one
                // lane group would take deg/R dependent rounds), short ones one
                // per lane group
                for (int32_t i = in0; i <= in1; ++i) {
                    if (a.rowptr[i + 1] - a.rowptr[i] <= kSmallCgWarpRow) continue;
                    double acc[VEC];
                    piece(a.rowptr[i], a.rowptr[i + 1], acc);
                    if (grp == 0) finish(i, acc);
                }
                // one lane group per row.  Rows of at most SR entries take one
                // gather round each; a group works on U of them at once (all
                // their row bounds, indices, gathers and p loads in flight
                // together -- the latency chain of a short row is rowptr ->
                // index -> gather, and this kernel has only 8 warps per SM to
                // hide it).  Longer rows (<= kSmallCgWarpRow) use K1's
                // pipelined gather.
                constexpr int SR = K::R < K::G ? K::R : K::G;  // entries one round covers
                constexpr int U = 4;
                for (int32_t i0 = in0 + grp; i0 <= in1; i0 += U * K::NGW) {
                    int32_t beg[U], deg[U], idx[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int32_t i = i0 + u * K::NGW;
                        beg[u] = i <= in1 ? __ldg(a.rowptr + i) : 0;
                        deg[u] = i <= in1 ? __ldg(a.rowptr + i + 1) - beg[u] : 0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) idx[u] = (deg[u] <= SR && lg < deg[u]) ? __ldg(a.colidx + beg[u] + lg) : 0;
                    double pv[U][VEC], vv[U][SR][VEC];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int32_t i = i0 + u * K::NGW;
                        if (deg[u] <= SR && i <= in1) {
                            ld_plain<VEC>(pc + static_cast<size_t>(i) * C + lg * VEC, pv[u]);
#pragma unroll
                            for (int t = 0; t < SR; ++t) {
                                const int32_t j = __shfl_sync(gmask, idx[u], gbase + t);
                                if (t < deg[u]) ld_plain<VEC>(pc + static_cast<size_t>(j) * C + lg * VEC, vv[u][t]);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int32_t i = i0 + u * K::NGW;
                        if (i > in1 || deg[u] > kSmallCgWarpRow) continue;
                        double acc[VEC];
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
                        if (deg[u] <= SR) {
#pragma unroll
                            for (int t = 0; t < SR; ++t)
                                if (t < deg[u]) {
#pragma unroll
                                    for (int v = 0; v < VEC; ++v) acc[v] += vv[u][t][v];
                                }
                            double qv[VEC];
#pragma unroll
                            for (int v = 0; v < VEC; ++v) {
                                qv[v] = __dadd_rn(pv[u][v], __dmul_rn(-a.beta, acc[v]));
                                dot[v] = fma(pv[u][v], qv[v], dot[v]);
                            }
                            st_plain<VEC>(qc + static_cast<size_t>(i) * C + lg * VEC, qv);
                        } else {
                            gather_rows<C, false, true>(a.colidx, beg[u], beg[u] + deg[u], K::R, pc, lg, gbase, gmask,
                                                        acc);
                            finish(i, acc);
                        }
                    }
                }
                auto publish = [&](const double (&acc)[VEC]) {  // carry_last + stamp
                    if (grp == 0) st_plain<VEC>(carry_last + static_cast<size_t>(gw) * bpad + ch * C + lg * VEC, acc);
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) atomicExch(a.stamp + static_cast<size_t>(gw) * nch + ch, static_cast<int32_t>(it));
                };
                double tail[VEC];  // this warp's part of a split row it owns the end of
#pragma unroll
                for (int v = 0; v < VEC; ++v) tail[v] = 0.0;
                if (!start0) {
                    double acc[VEC];
                    piece(static_cast<int32_t>(S - rs0),
                          static_cast<int32_t>(min(static_cast<int64_t>(a.rowptr[rs0 + 1]), E - rs0)), acc);
                    if (first_split) {
#pragma unroll
                        for (int v = 0; v < VEC; ++v) tail[v] = acc[v];
                    } else {
                        publish(acc);  // a middle piece: the row continues
                    }
                }
                if (row_endpos(rs1) >= E && (rs1 > rs0 || start0)) {
                    double acc[VEC];
                    piece(a.rowptr[rs1], static_cast<int32_t>(E - rs1), acc);  // the head of a row that continues
                    publish(acc);
                }
                if (first_split) {
                    // the earlier parts of row rs0 (warps w0 .. gw-1): every lane
                    // waits for the stamps of its warps in parallel, then lane
                    // group g sums warps w0+g, w0+g+NGW, ... and a fixed
                    // butterfly over the groups combines them.  Every warp
                    // publishes before it waits, so this cannot deadlock.
                    for (int w = w0 + lane; w < gw; w += 32) {
                        if (total * (w + 1) / nw <= total * w / nw) continue;  // an empty share holds no part
                        volatile int32_t* f = a.stamp + static_cast<size_t>(w) * nch + ch;
#if KZ_CHECKED
                        long long spins = 0;
                        while (*f != static_cast<int32_t>(it)) KZ_DCHECK(++spins < (1ll << 28));
#else
                        while (*f != static_cast<int32_t>(it)) {
                        }
#endif
                    }
                    __syncwarp();
                    __threadfence();
                    double acc[VEC];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
                    for (int w = w0 + grp; w < gw; w += K::NGW) {
                        if (total * (w + 1) / nw <= total * w / nw) continue;
                        double t[VEC];
                        ld_cg_vec<VEC>(carry_last + static_cast<size_t>(w) * bpad + ch * C + lg * VEC, t);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] += t[v];
                    }
#pragma unroll
                    for (int off = K::G; off < 32; off <<= 1)
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] += tail[v];
                    if (grp == 0) finish(rs0, acc);
                }
            }
#ifdef KZ_SMALL_DEBUG
            if (lane == 0 && gw < 8192) g_wt2[gw] = static_cast<unsigned int>(gtimer() - w_t0);
#endif
            // warp p.q partial (butterfly over the lane groups) -> CTA partial, warps in order
#pragma unroll
            for (int off = K::G; off < 32; off <<= 1)
#pragma unroll
                for (int v = 0; v < VEC; ++v) dot[v] += __shfl_xor_sync(0xffffffffu, dot[v], off);
            if (grp == 0) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) s_red2[warp * C + lg * VEC + v] = dot[v];
            }
            __syncthreads();
            if (threadIdx.x < C) {
                double t = 0.0;
                for (int w = 0; w < kSmallCgWarps; ++w) t += s_red2[w * C + threadIdx.x];
                partA[static_cast<size_t>(blockIdx.x) * bpad + ch * C + threadIdx.x] = t;
            }
            __syncthreads();
        }
        KZ_PT(1);
#ifdef KZ_SMALL_DEBUG
        if (lane == 0) atomicMax(&g_slowest_warp, ((gtimer() - w_t0) << 20) | static_cast<unsigned long long>(gw));
        if (lane == 0 && gw < 8192) g_wt[gw] = static_cast<unsigned int>(gtimer() - w_t0);
#endif
        __threadfence();
        grid.sync();
        KZ_PT(2);
        // ---- phase 2: a = rs / pq, r -= a*q, r.r partials
        reduce_cols(partA, s_a);  // s_a := pq
        if (threadIdx.x == 0) s_err = 0;
        __syncthreads();
        for (int c = threadIdx.x; c < bpad; c += kSmallCgThreads) {
            const double pq = s_a[c];
            int on = s_act[c];
            if (on && pq <= 0.0) {  // solver.py:84-85
                on = 0;
                s_act[c] = 0;
                atomicExch(&s_err, 1);
                if (blockIdx.x == 0) {
                    s.status[c] = KZ_ENOTSPD;
                    s.active[c] = 0;
                }
            }
            s_on[c] = on;
            s_a[c] = on ? s_rs[c] / pq : 0.0;
        }
        __syncthreads();
        if (s_err) {
            if (blockIdx.x == 0 && threadIdx.x == 0) *s.err = 1;
            break;
        }
        for (int ch = 0; ch < nch; ++ch) {
            const int cc = ch * C + threadIdx.x % C;
            double rr = 0.0;
            if (s_chunk[ch]) {
                double* rc = a.r + static_cast<size_t>(ch) * ld;
                const double* qc = a.q + static_cast<size_t>(ch) * ld;
                const double av = s_a[cc];
                const bool on = s_on[cc] != 0;
                for (int64_t e = static_cast<int64_t>(e0) * C + threadIdx.x; e < static_cast<int64_t>(e1) * C;
                     e += kSmallCgThreads) {
                    double rv = __ldcg(rc + e);
                    if (on) {
                        rv = __dsub_rn(rv, __dmul_rn(av, __ldcg(qc + e)));
                        rc[e] = rv;
                    }
                    rr = fma(rv, rv, rr);
                }
            }
            cta_partial(rr, ch, partB);
        }
        KZ_PT(3);
        __threadfence();
        grid.sync();
        KZ_PT(4);
        // ---- phase 3: stop test, b = rs'/rs, x += a*p, p = r + b*p
        reduce_cols(partB, s_b);  // s_b := r.r
        for (int c = threadIdx.x; c < bpad; c += kSmallCgThreads) {
            double bc = 0.0;
            if (s_on[c]) {  // solver.py:89-95
                const double v = s_b[c];
                const double rn = sqrt(v);
                if (blockIdx.x == 0) {
                    s.iters[c] = it;
                    s.rnorm[c] = rn;
                }
                if (rn <= s.thresh[c]) {
                    s_act[c] = 0;
                    if (blockIdx.x == 0) {
                        s.converged[c] = 1;
                        s.active[c] = 0;
                    }
                } else if (it >= s.max_iter) {
                    s_act[c] = 0;
                    if (blockIdx.x == 0) s.active[c] = 0;
                } else {
                    bc = v / s_rs[c];
                    s_rs[c] = v;
                }
            }
            s_b[c] = bc;
        }
        __syncthreads();
        for (int ch = 0; ch < nch; ++ch) {
            if (!s_chunk[ch]) continue;
            const int cc = ch * C + threadIdx.x % C;
            const bool ox = s_on[cc] != 0, op = ox && s_act[cc];
            if (!ox) continue;
            double* xc = a.x + static_cast<size_t>(ch) * ld;
            double* pc = a.p + static_cast<size_t>(ch) * ld;
            const double* rc = a.r + static_cast<size_t>(ch) * ld;
            const double av = s_a[cc], bv = s_b[cc];
            for (int64_t e = static_cast<int64_t>(e0) * C + threadIdx.x; e < static_cast<int64_t>(e1) * C;
                 e += kSmallCgThreads) {
                const double pv = __ldcg(pc + e);
                xc[e] = __dadd_rn(__ldcg(xc + e), __dmul_rn(av, pv));
                if (op) pc[e] = __dadd_rn(__ldcg(rc + e), __dmul_rn(bv, pv));
            }
        }
        chunk_flags();
        KZ_PT(5);
        __threadfence();
        grid.sync();
        KZ_PT(6);
    }
#ifdef KZ_SMALL_DEBUG
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long sw = g_slowest_warp;
        const int w = static_cast<int>(sw & 0xfffff);
        const int64_t Sw = total * w / nw, Ew = total * (w + 1) / nw;
        const int32_t r0w = merge_row(a.rowptr, a.rows, Sw), r1w = merge_row(a.rowptr, a.rows, Ew - 1);
        printf("slowest warp %d: %.2f us, rows %d..%d (deg %d .. %d), split start %d\n", w, (sw >> 20) / 1e3, r0w, r1w,
               a.rowptr[r0w + 1] - a.rowptr[r0w], a.rowptr[r1w + 1] - a.rowptr[r1w],
               (int)(static_cast<int64_t>(a.rowptr[r0w]) + r0w < Sw));
        for (int ww = 0; ww < nw && ww < 8192; ++ww) {
            if (g_wt[ww] < 10000) continue;  // only the slow ones (> 10 us)
            const int64_t S2 = total * ww / nw, E2 = total * (ww + 1) / nw;
            const int32_t a0 = merge_row(a.rowptr, a.rows, S2), a1 = merge_row(a.rowptr, a.rows, E2 - 1);
            printf("  warp %d: gathers %.2f us, phase %.2f us, rows %d..%d degs %d %d inner %d\n", ww, g_wt2[ww] / 1e3,
                   g_wt[ww] / 1e3, a0, a1, a.rowptr[a0 + 1] - a.rowptr[a0], a.rowptr[a1 + 1] - a.rowptr[a1], a1 - a0 + 1);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("small cg: %lld it, us per it: top %.2f ph1 %.2f sync %.2f ph2 %.2f sync %.2f ph3 %.2f sync %.2f\n",
               (long long)it, ph[0] / 1e3 / it, ph[1] / 1e3 / it, ph[2] / 1e3 / it, ph[3] / 1e3 / it, ph[4] / 1e3 / it,
               ph[5] / 1e3 / it, ph[6] / 1e3 / it);
#endif
    if (blockIdx.x == 0 && threadIdx.x == 0) *s.n_active = 0;
    if (a.scores) {
        // ---- output: clamp(x) through perm; the packed reports ----
        __threadfence();
        grid.sync();
        for (int ch = 0; ch < nch; ++ch)
            for (int64_t e = static_cast<int64_t>(e0) * C + threadIdx.x; e < static_cast<int64_t>(e1) * C;
                 e += kSmallCgThreads) {
                const int c = static_cast<int>(e % C), j = ch * C + c;
                if (j >= a.b) continue;
                const int64_t i = e / C;
                double v = __ldcg(a.x + static_cast<size_t>(ch) * ld + e);
                if (a.clamp) v = v > 0.0 ? v : 0.0;
                a.scores[static_cast<size_t>(j) * a.rows + (a.perm ? a.perm[i] : i)] = v;
            }
        if (blockIdx.x == 0)
            for (int j = threadIdx.x; j < a.b; j += kSmallCgThreads) {
                kz_report rp;
                rp.iterations = __ldcg(s.iters + j);
                rp.converged = __ldcg(s.converged + j);
                rp.status = __ldcg(s.status + j);
                rp.final_residual_norm = __ldcg(s.rnorm + j);
                rp.rhs_norm = sqrt(__ldcg(s.bnorm2 + j));
                a.reports[j] = rp;
            }
    }
}

// Grid of the fused loop (at most one CTA per SM), or 0 when it does not apply.
inline int small_cg_grid(int64_t rows, int64_t nnz, int C, int bpad, const void* kernel) {
    if (bpad > kSmallCgMaxCols || (kSmallCgThreads % C) != 0 || nnz > kSmallCgMaxNnz ||
        static_cast<size_t>(rows) * bpad > kSmallCgElems ||
        static_cast<double>(nnz + rows) * bpad > kSmallCgMaxWork)
        return 0;
    // occupancy of each kernel instantiation, queried once per device
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, int>> occ;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = -1;
    {
        std::lock_guard<std::mutex> lock(mu);
        for (const auto& e : occ)
            if (e.first.first == kernel && e.first.second == dev) per_sm = e.second;
        if (per_sm < 0) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSmallCgThreads, 0) != cudaSuccess) {
                cudaGetLastError();
                per_sm = 0;
            }
            occ.push_back({{kernel, dev}, per_sm});
        }
    }
    if (per_sm < 1) return 0;
    // gathers are latency-bound: as many resident warps as the registers
    // allow (the merge-path shares stay >= ~16 items per warp)
    const int64_t want = std::max<int64_t>(1, (nnz + rows) / (16 * kSmallCgWarps));
    return static_cast<int>(std::min<int64_t>(static_cast<int64_t>(num_sms()) * std::min(per_sm, kSmallCgCtasPerSm), want));
}

}  // namespace kz
