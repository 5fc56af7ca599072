// lowrank.cuh -- the eigen-of-A low-rank start of the north-star LRC variant
// (not in the reference, parity only against the exact
// solution).
//
// Index: U = n x r Ritz vectors of A (top r, device Lanczos), AU = A U (one
// K1 SpMM of the r-column block), W = (I - beta U'AU)^-1 (r x r).  For a
// query q the Galerkin start on span(U) is
//     x0 = U y,   y = W U' b = beta * W (AU)[q, :]'      (b = beta A e_q)
// and its exact residual needs no SpMM:
//     r0 = b - (I - beta A) U y = b - x0 + beta * (AU) y.
// CG then runs from (x0, r0) with the stop test ||r|| <= tol ||b|| -- the same
// iterates as CG on M d = r0 from zero.  The two tall-skinny products
// U y and (AU) y (n x r times r x b) are one fused DMMA pass.
//
// Walk start (a2u = A^2 U given): the first term of the Katz series
// x = sum_k beta^k A^k e_q is put into the start exactly and the Galerkin
// step is taken on the remainder,
//     x0 = beta A e_q + U y,   y = beta^2 W (A^2 U)[q, :]'
//     r0 = beta^2 A^2 e_q - U y + beta (AU) y,
// where (A^2 e_q)_i = |N(i) ∩ N(q)| is an integer count (the 2-walks from q),
// pushed from the neighbours of q with integer atomics -- order-free, so
// deterministic -- at a cost of sum_{t in N(q)} deg(t) increments per query
// (R-MAT 22: 45 M for 256 queries, vs 33 G gathered values for one SpMM).
// The remainder's residual starts where plain Galerkin's first CG step
// would leave it: one CG iteration fewer (R-MAT 22: 5 -> 4).
#pragma once

#include "spmm.cuh"

struct kz_eigen {
    int64_t n = 0, r = 0, ldr = 0;  // ldr: row stride of u / au (>= r, multiple of 4, zero padded)
    double beta = 0.0;
    const kz_graph* op = nullptr;   // A in the solve order
    const double* u = nullptr;      // device n x ldr row-major
    const double* au = nullptr;     // device n x ldr row-major
    const double* w = nullptr;      // device r x r row-major, symmetric
    const double* a2u = nullptr;    // optional device n x ldr row-major, A^2 U (walk start)
    const double* a3u = nullptr;    // optional device n x ldr row-major, A^3 U (two-term walk start)
    const double* a4u = nullptr;    // optional device n x ldr row-major, A^4 U (three-term walk start)
};

namespace kz {

// y[j] (chunked [nch][ldr][C]) = beta * W (AU)[q_j, :]' (walk start:
// beta^2 * W (A^2 U)[q_j, :]'); padded columns and rows r..ldr-1 are zero.
// One thread per (k, j); fixed summation order.
template <int C>
__global__ void lowrank_coef_kernel(kz_eigen h, const int64_t* __restrict__ qpos, int b, double* __restrict__ y) {
    const int j = blockIdx.y;
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= h.ldr) return;
    double s = 0.0;
    if (j < b && k < h.r) {
        const double* __restrict__ aurow =
            (h.a4u ? h.a4u : h.a3u ? h.a3u : h.a2u ? h.a2u : h.au) + qpos[j] * h.ldr;
        const double* __restrict__ wrow = h.w + k * h.r;
        for (int64_t i = 0; i < h.r; ++i) s = fma(wrow[i], __ldg(aurow + i), s);
        const double b2 = __dmul_rn(h.beta, h.beta);
        s *= h.a4u ? __dmul_rn(b2, b2) : h.a3u ? __dmul_rn(b2, h.beta) : h.a2u ? b2 : h.beta;
    }
    y[static_cast<size_t>(j / C) * h.ldr * C + static_cast<size_t>(k) * C + (j % C)] = s;
}

constexpr int kLrWarps = 8;
#ifndef KZ_LR_MT
#define KZ_LR_MT 1
#endif
constexpr int kLrMT = KZ_LR_MT;                    // m-fragments (8 rows) per warp (2 spills)
constexpr int kLrRows = 8 * kLrMT * kLrWarps;      // rows per tile
#ifndef KZ_LR_AHEAD
#define KZ_LR_AHEAD 4
#endif
#ifndef KZ_LR_MINBLOCKS
#define KZ_LR_MINBLOCKS 2
#endif
constexpr int kLrAhead = KZ_LR_AHEAD;              // k-steps of A fragments in flight

__device__ __forceinline__ void lr_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// For the NC = 8*NT columns j0 .. j0+NC-1 (the column group; columns >= jmax
// are padding and are neither read nor written):
//   x = U y ;  r = p = beta * (AU y) - x    (the rhs b = beta A e_q is added
//   afterwards by eigen_add_rhs_kernel, so r is written, never read)
// walk start (cnt != nullptr): r = p = beta * (AU y) - x + beta^2 * cnt with
// cnt the int32 2-walk counts in the block layout; b goes onto x instead.
// y's group columns are staged in shared memory once per CTA ([ldr][NC+8],
// bank padded); each warp owns 16 rows of a 128-row tile and streams its U
// and AU fragments from HBM kLrAhead k-steps ahead.  Persistent over tiles.
// XO (two-term walk start): only x = U y + beta^2 * cnt; the residual comes
// from one K1 SpMM on x instead of the (AU) y product.
template <int C, int NT, bool XO = false>
__global__ void __launch_bounds__(32 * kLrWarps, KZ_LR_MINBLOCKS)
    lowrank_init_kernel(kz_eigen h, const double* __restrict__ y, double* __restrict__ x, double* __restrict__ r,
                        double* __restrict__ p, int64_t ldv, int j0, int jmax,
                        const int32_t* __restrict__ cnt = nullptr, double* __restrict__ cnt_out = nullptr) {
    constexpr int NC = 8 * NT;
    constexpr int YLD = NC + 8;
    extern __shared__ __align__(16) double ys[];
    const int64_t ldr = h.ldr;
    for (int e = threadIdx.x; e < ldr * NC; e += blockDim.x) {
        const int k = e / NC, jj = e % NC;
        const int j = j0 + jj;
        ys[k * YLD + jj] = j < jmax ? y[static_cast<size_t>(j / C) * ldr * C + static_cast<size_t>(k) * C + (j % C)] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fk = lane & 3;
    const int64_t ntiles = (h.n + kLrRows - 1) / kLrRows;
    const int nsteps = static_cast<int>(ldr / 4);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t rw = tile * kLrRows + warp * (8 * kLrMT);
        double ua[kLrMT][NT][2], wa[kLrMT][NT][2];
#pragma unroll
        for (int m = 0; m < kLrMT; ++m)
#pragma unroll
            for (int n = 0; n < NT; ++n) ua[m][n][0] = ua[m][n][1] = wa[m][n][0] = wa[m][n][1] = 0.0;
        const double* up[kLrMT];
        const double* wp[kLrMT];
#pragma unroll
        for (int m = 0; m < kLrMT; ++m) {
            int64_t row = rw + m * 8 + fr;
            row = row < h.n ? row : h.n - 1;  // clamped rows are computed and not stored
            up[m] = h.u + row * ldr + fk;
            wp[m] = h.au + row * ldr + fk;
        }
        double fu[kLrAhead][kLrMT], fw[kLrAhead][kLrMT];
#pragma unroll
        for (int s = 0; s < kLrAhead; ++s)
#pragma unroll
            for (int m = 0; m < kLrMT; ++m) {
                const bool ok = s < nsteps;
                fu[s][m] = ok ? __ldcs(up[m] + 4 * s) : 0.0;
                fw[s][m] = ok && !XO ? __ldcs(wp[m] + 4 * s) : 0.0;
            }
        for (int s0 = 0; s0 < nsteps; s0 += kLrAhead) {
#pragma unroll
            for (int u = 0; u < kLrAhead; ++u) {
                const int s = s0 + u;
                double cu[kLrMT], cw[kLrMT];
#pragma unroll
                for (int m = 0; m < kLrMT; ++m) {
                    cu[m] = fu[u][m];
                    cw[m] = fw[u][m];
                    const bool ok = s + kLrAhead < nsteps;
                    fu[u][m] = ok ? __ldcs(up[m] + 4 * (s + kLrAhead)) : 0.0;
                    if constexpr (!XO) fw[u][m] = ok ? __ldcs(wp[m] + 4 * (s + kLrAhead)) : 0.0;
                }
                if (s < nsteps) {
                    double bv[NT];
#pragma unroll
                    for (int n = 0; n < NT; ++n) bv[n] = ys[(4 * s + fk) * YLD + n * 8 + fr];
#pragma unroll
                    for (int m = 0; m < kLrMT; ++m)
#pragma unroll
                        for (int n = 0; n < NT; ++n) {
                            lr_dmma(ua[m][n][0], ua[m][n][1], cu[m], bv[n]);
                            if constexpr (!XO) lr_dmma(wa[m][n][0], wa[m][n][1], cw[m], bv[n]);
                        }
                }
            }
        }
#pragma unroll
        for (int m = 0; m < kLrMT; ++m) {
            const int64_t row = rw + m * 8 + fr;
            if (row >= h.n) continue;
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = j0 + n * 8 + 2 * fk + e;
                    if (j >= jmax) continue;
                    const size_t off = static_cast<size_t>(j / C) * ldv + static_cast<size_t>(row) * C + (j % C);
                    if constexpr (XO) {
                        double x0 = ua[m][n][e];
                        double t2 = 0.0;  // beta^2 (A^2 e_q)_row
                        if (cnt) {
                            const int32_t c = __ldcs(cnt + off);
                            if (c) {
                                t2 = __dmul_rn(__dmul_rn(h.beta, h.beta), static_cast<double>(c));
                                x0 = __dadd_rn(x0, t2);
                            }
                        }
                        x[off] = x0;
                        if (cnt_out) cnt_out[off] = t2;  // three-term start: input of the A^3 e_q SpMM
                        continue;
                    }
                    const double x0 = ua[m][n][e];
                    x[off] = x0;
                    double r0 = __dsub_rn(__dmul_rn(h.beta, wa[m][n][e]), x0);
                    if (cnt) {
                        const int32_t c = __ldcs(cnt + off);
                        if (c) r0 = __dadd_rn(r0, __dmul_rn(__dmul_rn(h.beta, h.beta), static_cast<double>(c)));
                    }
                    r[off] = r0;
                    if (p) p[off] = r0;
                }
        }
    }
}

// r, p (chunked) += beta at the neighbours of q_j: the rhs b = beta A e_q
// (index.py:93-101) added onto r0 = beta (AU) y - x0 (walk start: x += beta
// there instead, p == nullptr); and ||b||^2 = beta^2 deg(q_j) for the stop
// threshold (solver.py:71-72).
template <int C>
__global__ void eigen_add_rhs_kernel(double* __restrict__ r, double* __restrict__ p, int64_t ld,
                                     const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                                     const int64_t* __restrict__ qpos, int b, double beta, double* __restrict__ bnorm2) {
    const int j = blockIdx.x;
    if (j >= b) {
        if (threadIdx.x == 0) bnorm2[j] = 0.0;
        return;
    }
    const int64_t q = qpos[j];
    const int beg = rowptr[q], end = rowptr[q + 1];
    for (int k = beg + threadIdx.x; k < end; k += blockDim.x) {
        const size_t off = static_cast<size_t>(j / C) * ld + static_cast<size_t>(colidx[k]) * C + (j % C);
        r[off] = __dadd_rn(r[off], beta);
        if (p) p[off] = __dadd_rn(p[off], beta);
    }
    if (threadIdx.x == 0) bnorm2[j] = __dmul_rn(__dmul_rn(beta, beta), static_cast<double>(end - beg));
}

// 2-walk counts of the walk start: cnt[i, j] += 1 for every path q_j - t - i
// (t in N(q_j)), i.e. cnt = A^2 e_q per column, in the chunked block layout
// (int32, zeroed by the caller).  blockIdx.y = column; each CTA takes one
// neighbour t of q_j at a time and all its threads push along N(t) with
// order-free integer atomics, 4 index loads in flight per thread (a hub
// neighbour's list of ~10^5 entries is then ~100 rounds, not ~5,000).
template <int C>
__global__ void __launch_bounds__(256) walk2_count_kernel(int32_t* __restrict__ cnt, int64_t ld,
                                                          const int32_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ colidx,
                                                          const int64_t* __restrict__ qpos, int b) {
    constexpr int U = 4;
    const int j = blockIdx.y;
    if (j >= b) return;
    const int64_t q = qpos[j];
    const int beg = rowptr[q], end = rowptr[q + 1];
    int32_t* __restrict__ base = cnt + static_cast<size_t>(j / C) * ld + (j % C);
    for (int k = beg + static_cast<int>(blockIdx.x); k < end; k += gridDim.x) {
        const int t = __ldg(colidx + k);
        const int tb = __ldg(rowptr + t), te = __ldg(rowptr + t + 1);
        int m = tb + threadIdx.x;
        for (; m + (U - 1) * static_cast<int>(blockDim.x) < te; m += U * blockDim.x) {
            int i[U];
#pragma unroll
            for (int u = 0; u < U; ++u) i[u] = __ldcs(colidx + m + u * blockDim.x);
#pragma unroll
            for (int u = 0; u < U; ++u) atomicAdd(base + static_cast<size_t>(i[u]) * C, 1);
        }
        for (; m < te; m += blockDim.x) atomicAdd(base + static_cast<size_t>(__ldcs(colidx + m)) * C, 1);
    }
}

inline size_t lowrank_smem(int64_t ldr, int NC) { return sizeof(double) * static_cast<size_t>(ldr) * (NC + 8); }

}  // namespace kz
