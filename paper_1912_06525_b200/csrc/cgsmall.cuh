// cgsmall.cuh -- the whole CG loop of a small batched solve in ONE
// cooperative kernel (cfg1-sized problems: the vector blocks sit in L2 and
// every separate kernel of the host- or graph-driven loop costs more in
// launch + tail latency than in work).
//
// Per iteration, three phases separated by grid-wide barriers, exactly the
// reference recurrence of cg() (solver.py:78-95) per column:
//   1  q = p - beta*A p (gather), partial p.q per warp -> per CTA
//   2  every CTA reduces the CTA partials of p.q in a fixed order, a = rs/pq
//      (non-positive curvature: the column errs, the solve stops), then
//      r -= a*q over its share with partial r.r
//   3  every CTA reduces r.r, applies the stop test / iteration budget and
//      b = rs'/rs, then x += a*p, p = r + b*p over its share
// Every CTA derives the same per-column scalars from the same partials in the
// same order, so no broadcast step is needed and results are run-to-run
// deterministic.  CTA 0 publishes the per-column state for the reports.
// Rows are cut into cost-balanced contiguous warp segments (cost = entries +
// rows, a binary search of rowptr), fixed for the whole solve.
#pragma once

#include <cooperative_groups.h>

#include "blockops.cuh"

namespace kz {

constexpr int kSmallCgThreads = 256;
constexpr int kSmallCgMaxCols = 256;  // columns (bpad) the fused loop handles
constexpr size_t kSmallCgElems = size_t(1) << 22;  // block size (doubles) up to which the loop is fused

struct SmallCgArgs {
    int32_t rows, nchunks, b, bpad;
    const int32_t* rowptr;
    const int32_t* colidx;
    double beta;
    double *x, *r, *p, *q;  // chunked blocks [nchunks][rows][C]
    double* part;           // [2][gridDim.x][bpad] CTA partials (phase 1 / phase 2 buffers)
    SolveState s;
};

// first row whose cost rowptr[i] + i reaches `target` (rows in [0, n])
__device__ __forceinline__ int32_t cost_row(const int32_t* rowptr, int32_t n, int64_t target) {
    int32_t lo = 0, hi = n;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(rowptr[mid]) + mid < target) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <int C>
__global__ void __launch_bounds__(kSmallCgThreads) cg_small_kernel(SmallCgArgs a) {
    namespace cgr = cooperative_groups;
    cgr::grid_group grid = cgr::this_grid();
    constexpr int NS = 32 / C;  // neighbour streams per warp (lanes of one stream = the C columns)
    constexpr int WPC = kSmallCgThreads / 32;
    __shared__ double s_red[kSmallCgThreads];
    __shared__ double s_a[kSmallCgMaxCols], s_b[kSmallCgMaxCols], s_rs[kSmallCgMaxCols];
    __shared__ int s_on[kSmallCgMaxCols], s_act[kSmallCgMaxCols], s_chunk[kSmallCgMaxCols / 1];
    __shared__ int s_any, s_err;
    const SolveState& s = a.s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * WPC + warp, nw = gridDim.x * WPC;
    const int64_t ld = static_cast<int64_t>(a.rows) * C;
    const int nch = a.nchunks, bpad = a.bpad;
    // cost-balanced row segment of this warp
    const int64_t total = static_cast<int64_t>(a.rowptr[a.rows]) + a.rows;
    const int32_t r0 = cost_row(a.rowptr, a.rows, total * gw / nw);
    const int32_t r1 = cost_row(a.rowptr, a.rows, total * (gw + 1) / nw);
    // element share of this CTA inside each chunk: rows [e0, e1)
    const int32_t e0 = static_cast<int32_t>(static_cast<int64_t>(a.rows) * blockIdx.x / gridDim.x);
    const int32_t e1 = static_cast<int32_t>(static_cast<int64_t>(a.rows) * (blockIdx.x + 1) / gridDim.x);
    for (int c = threadIdx.x; c < bpad; c += kSmallCgThreads) {
        s_act[c] = c < a.b ? s.active[c] : 0;
        s_rs[c] = s.rs[c];
    }
    __syncthreads();
    auto chunk_flags = [&]() {
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
    // CTA partial (threads sharing a column add in fixed order) -> part[cta][col]
    // two partial buffers: a CTA that has finished reducing buffer A may
    // write buffer B while slower CTAs still read A (and vice versa a phase
    // later); a grid barrier separates every reuse of one buffer
    double* partA = a.part;
    double* partB = a.part + static_cast<size_t>(gridDim.x) * bpad;
    auto cta_partial = [&](double v, int chunk) {
        s_red[threadIdx.x] = v;
        __syncthreads();
        if (threadIdx.x < C) {
            double t = 0.0;
            for (int k = threadIdx.x; k < kSmallCgThreads; k += C) t += s_red[k];
            partB[static_cast<size_t>(blockIdx.x) * bpad + chunk * C + threadIdx.x] = t;
        }
        __syncthreads();
    };
    // every CTA: column totals of the CTA partials, fixed order
    auto reduce_cols = [&](const double* part, double* out) {
        for (int c = threadIdx.x; c < bpad; c += kSmallCgThreads) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
            int k = 0;
            for (; k + 3 < static_cast<int>(gridDim.x); k += 4) {
                t0 += __ldcg(part + static_cast<size_t>(k) * bpad + c);
                t1 += __ldcg(part + static_cast<size_t>(k + 1) * bpad + c);
                t2 += __ldcg(part + static_cast<size_t>(k + 2) * bpad + c);
                t3 += __ldcg(part + static_cast<size_t>(k + 3) * bpad + c);
            }
            for (; k < static_cast<int>(gridDim.x); ++k) t0 += __ldcg(part + static_cast<size_t>(k) * bpad + c);
            out[c] = (t0 + t1) + (t2 + t3);
        }
        __syncthreads();
    };
    chunk_flags();
    int64_t it = 0;
    for (;;) {
        if (!s_any || it >= s.max_iter) break;
        ++it;
        // ---- phase 1: q = p - beta*A p, warp partials of p.q -> CTA partials
        for (int ch = 0; ch < nch; ++ch) {
            double dot = 0.0;
            if (s_chunk[ch]) {
                const double* pc = a.p + static_cast<size_t>(ch) * ld;
                double* qc = a.q + static_cast<size_t>(ch) * ld;
                const int col = lane % C, st = lane / C;
                for (int32_t i = r0; i < r1; ++i) {
                    const int32_t beg = a.rowptr[i], end = a.rowptr[i + 1];
                    double acc = 0.0;
                    for (int32_t e = beg + st; e < end; e += NS)
                        acc += pc[static_cast<size_t>(a.colidx[e]) * C + col];
#pragma unroll
                    for (int off = C; off < 32; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                    if (st == 0) {
                        const double pv = pc[static_cast<size_t>(i) * C + col];
                        const double qv = __dadd_rn(pv, __dmul_rn(-a.beta, acc));
                        qc[static_cast<size_t>(i) * C + col] = qv;
                        dot = fma(pv, qv, dot);
                    }
                }
            }
            // warp partial (lanes < C) -> CTA partial, warps in fixed order
            if (lane >= C) dot = 0.0;
            s_red[threadIdx.x] = dot;
            __syncthreads();
            if (threadIdx.x < C) {
                double t = 0.0;
                for (int w = 0; w < WPC; ++w) t += s_red[w * 32 + threadIdx.x];
                partA[static_cast<size_t>(blockIdx.x) * bpad + ch * C + threadIdx.x] = t;
            }
            __syncthreads();
        }
        __threadfence();
        grid.sync();
        // ---- phase 2: a = rs / pq, r -= a*q, CTA partials of r.r
        reduce_cols(partA, s_a);  // s_a := pq
        if (threadIdx.x == 0) s_err = 0;
        __syncthreads();
        for (int c = threadIdx.x; c < bpad; c += kSmallCgThreads) {
            const double pq = s_a[c];
            int on = s_act[c];
            if (on && pq <= 0.0) {
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
            const int col = ch * C + threadIdx.x % C;
            double rr = 0.0;
            if (s_chunk[ch]) {
                double* rc = a.r + static_cast<size_t>(ch) * ld;
                const double* qc = a.q + static_cast<size_t>(ch) * ld;
                const double av = s_a[col];
                const bool on = s_on[col] != 0;
                for (int64_t e = static_cast<int64_t>(e0) * C + threadIdx.x; e < static_cast<int64_t>(e1) * C;
                     e += kSmallCgThreads) {
                    double rv = rc[e];
                    if (on) {
                        rv = __dsub_rn(rv, __dmul_rn(av, qc[e]));
                        rc[e] = rv;
                    }
                    rr = fma(rv, rv, rr);
                }
            }
            cta_partial(rr, ch);
        }
        __threadfence();
        grid.sync();
        // ---- phase 3: stop test, b = rs'/rs, x += a*p, p = r + b*p
        reduce_cols(partB, s_b);  // s_b := r.r
        for (int c = threadIdx.x; c < bpad; c += kSmallCgThreads) {
            double bc = 0.0;
            if (s_on[c]) {
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
            const int col = ch * C + threadIdx.x % C;
            const bool ox = s_on[col] != 0, op = ox && s_act[col];
            if (!ox) continue;
            double* xc = a.x + static_cast<size_t>(ch) * ld;
            double* pc = a.p + static_cast<size_t>(ch) * ld;
            const double* rc = a.r + static_cast<size_t>(ch) * ld;
            const double av = s_a[col], bv = s_b[col];
            for (int64_t e = static_cast<int64_t>(e0) * C + threadIdx.x; e < static_cast<int64_t>(e1) * C;
                 e += kSmallCgThreads) {
                const double pv = pc[e];
                xc[e] = __dadd_rn(xc[e], __dmul_rn(av, pv));
                if (op) pc[e] = __dadd_rn(rc[e], __dmul_rn(bv, pv));
            }
        }
        chunk_flags();
        __threadfence();
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *s.n_active = 0;
}

// Grid of the fused loop: one CTA per SM at most, fewer for tiny problems;
// 0 when the fused loop does not apply (then the caller uses the normal loop).
inline int small_cg_grid(int64_t rows, int C, int bpad, const void* kernel) {
    if (bpad > kSmallCgMaxCols || (kSmallCgThreads % C) != 0) return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSmallCgThreads, 0) != cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        return 0;
    }
    const int64_t want = std::max<int64_t>(1, (rows * bpad) / 4096);
    return static_cast<int>(std::min<int64_t>(static_cast<int64_t>(num_sms()) * std::min(per_sm, 1), want));
}

}  // namespace kz
