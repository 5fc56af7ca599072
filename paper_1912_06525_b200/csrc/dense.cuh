// dense.cuh -- K3/K6: fp64 dense operator times a chunked block, split-K.
//
//   Y[i, :] = alpha * sum_k A[k, i] * X[k, :]  (+ beta * Y[i, :])
//
// A is row-major K x M (lda), so the M outputs of one k are contiguous and a
// CTA of 256 threads (one output row each) reads A with fully coalesced
// 2 KB rows; X rows (all columns of the block, <= 64) are staged in shared
// memory and broadcast.  Used for:
//   t = L^-1 r      A = (L^-1)^T, triangular (k <= i)   (factor.py:331,334)
//   z = L^-T t      A = L^-1,     triangular (k >= i)   (factor.py:331,337)
//   c = U^T t       A = U (n2 x ell)                    (factor.py:335)
//   t += (U D) c    A = (U D)^T (ell x n2)              (factor.py:336-337)
// Tiles entirely outside the triangle are skipped.  The K range is split
// over CTAs (enough to cover 148 SMs when M is small); the last CTA of a row
// tile reduces the split partials in a fixed order (deterministic).
//
// Three kernels share this contract: dense_kernel (CUDA-core FMA, for column
// groups that are not a multiple of 8), dense_dmma_kernel (fp64 tensor cores,
// mma.sync.m8n8k4.f64, fragments straight from global memory: small and
// mid-size operators) and dense_dmma2_kernel (shared-memory staged A/X slabs
// by cp.async: n2 >= 8192).  tcgen05 has no fp64 kind on sm_100a, so DMMA is
// the fp64 tensor path; its measured ceiling here is the cuBLAS DGEMM rate,
// 35.5 TFLOP/s (profiles/r01_fp64_peak.json).
#pragma once

#include "spmm.cuh"

namespace kz {

__host__ __device__ __forceinline__ int64_t mn64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t mx64(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr int kDenseThreads = 256;  // threads per CTA
constexpr int kDenseRows = 512;     // output rows per CTA tile (<= 2 per thread)
constexpr int kDenseK = 16;         // k rows staged per step
constexpr int kDenseMaxCols = 64;
constexpr int kDenseMaxSplit = 16;

struct DenseArgs {
    const double* A;
    int64_t lda, M, K;  // lda even, A[k*lda + i] valid (zero-padded) for i < lda
    int tri;  // 0 full, 1: only k >= i nonzero, 2: only k <= i nonzero
    const double* X;
    int64_t ldx;  // chunk stride of X (K rows)
    double* Y;
    int64_t ldy;  // chunk stride of Y (M rows)
    double alpha, beta;
    int ksplit;
    int64_t kper;
    int64_t rows_tile;  // output rows per CTA tile (256 * TM)
    double* part;  // [mtiles][ksplit][threads][TM*NC]
    int32_t* cnt;  // [mtiles]
    const int32_t* chunk_active;  // optional flags of this launch's chunks (all 0: nothing to do)
    int nchunk;                   // chunks covered by this launch
};

// A launch whose chunks are all inactive (columns frozen by the PCG masks)
// returns at once; the decision is uniform over the grid, so no CTA of a
// split-K launch touches the tile counters.
__device__ __forceinline__ bool dense_skip(const DenseArgs& a) {
    if (!a.chunk_active) return false;
    for (int c = 0; c < a.nchunk; ++c)
        if (a.chunk_active[c]) return false;
    return true;
}

__device__ __forceinline__ bool dense_tile_empty(const DenseArgs& a, int64_t i0, int64_t k0, int64_t k1) {
    if (k0 >= k1) return true;
    const int64_t i1 = mn64(a.M, i0 + a.rows_tile) - 1;
    if (a.tri == 1 && k1 - 1 < i0) return true;  // needs some k >= i
    if (a.tri == 2 && k0 > i1) return true;      // needs some k <= i
    return false;
}

// Each thread owns TM consecutive output rows and all NC columns: per k it
// loads TM entries of A (one 16-byte load for TM = 2) and the X row from
// shared memory in 16-byte pieces, i.e. 2*TM FMAs per shared load.
template <int C, int NCH, int TM>
__global__ void __launch_bounds__(kDenseThreads, (TM * C * NCH <= 16) ? 2 : 1) dense_kernel(DenseArgs a) {
    if (dense_skip(a)) return;
    constexpr int NC = C * NCH;
    constexpr int ROWS = kDenseThreads * TM;
    static_assert(NC % 2 == 0 || NC == 1, "column count");
    const int mt = blockIdx.x / a.ksplit, ks = blockIdx.x - mt * a.ksplit;
    const int64_t i0 = static_cast<int64_t>(mt) * ROWS;
    const int64_t i = i0 + static_cast<int64_t>(threadIdx.x) * TM;
    const int64_t k0 = static_cast<int64_t>(ks) * a.kper;
    const int64_t k1 = mn64(a.K, k0 + a.kper);
    __shared__ __align__(16) double xs[2][kDenseK][NC];
    __shared__ int is_last;
    double acc[TM][NC];
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[t][j] = 0.0;
    const bool empty = dense_tile_empty(a, i0, k0, k1);
    if (!empty) {
        int64_t kb = k0, ke = k1;
        if (a.tri == 1) kb = mx64(kb, i0);
        if (a.tri == 2) ke = mn64(ke, mn64(a.M, i0 + ROWS));
        kb -= (kb - k0) % kDenseK;
        const bool valid = i < a.M;
        constexpr int PT = (kDenseK * NC + kDenseThreads - 1) / kDenseThreads;  // staged values per thread
        double stage[PT];
        auto fetch = [&](int64_t kk) {
#pragma unroll
            for (int u = 0; u < PT; ++u) {
                const int e = threadIdx.x + u * kDenseThreads;
                const int r = e / NC, j = e % NC;
                const int ch = j / C, c = j % C;
                stage[u] = (e < kDenseK * NC && kk + r < ke)
                               ? a.X[static_cast<size_t>(ch) * a.ldx + static_cast<size_t>(kk + r) * C + c]
                               : 0.0;
            }
        };
        auto commit = [&](int buf) {
#pragma unroll
            for (int u = 0; u < PT; ++u) {
                const int e = threadIdx.x + u * kDenseThreads;
                if (e < kDenseK * NC) (&xs[buf][0][0])[e] = stage[u];
            }
        };
        // A entries of a stage are loaded in one batch (kDenseK independent
        // loads per thread) one stage ahead of their use, like X.
        double an[kDenseK][TM];
        auto fetch_a = [&](int64_t kk) {
            const double* Ap = a.A + static_cast<size_t>(kk) * a.lda + i;
            const int nk = static_cast<int>(mn64(kDenseK, ke - kk));
#pragma unroll
            for (int r = 0; r < kDenseK; ++r) {
                if (valid && r < nk) {
                    if constexpr (TM == 2) {
                        const double2 p = __ldg(reinterpret_cast<const double2*>(Ap + static_cast<size_t>(r) * a.lda));
                        an[r][0] = p.x;
                        an[r][1] = p.y;
                    } else {
                        an[r][0] = __ldg(Ap + static_cast<size_t>(r) * a.lda);
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < TM; ++t) an[r][t] = 0.0;
                }
            }
        };
        fetch(kb);
        commit(0);
        fetch_a(kb);
        __syncthreads();
        int buf = 0;
        for (int64_t kk = kb; kk < ke; kk += kDenseK) {
            const int64_t kn = kk + kDenseK;
            double ac[kDenseK][TM];
#pragma unroll
            for (int r = 0; r < kDenseK; ++r)
#pragma unroll
                for (int t = 0; t < TM; ++t) ac[r][t] = an[r][t];
            if (kn < ke) {
                fetch(kn);  // next stage in flight while computing this one
                fetch_a(kn);
            }
#pragma unroll
            for (int r = 0; r < kDenseK; ++r) {
                if constexpr (NC == 1) {
                    const double xv = xs[buf][r][0];
#pragma unroll
                    for (int t = 0; t < TM; ++t) acc[t][0] = fma(ac[r][t], xv, acc[t][0]);
                } else {
#pragma unroll
                    for (int j = 0; j < NC; j += 2) {
                        const double2 xv = *reinterpret_cast<const double2*>(&xs[buf][r][j]);
#pragma unroll
                        for (int t = 0; t < TM; ++t) {
                            acc[t][j] = fma(ac[r][t], xv.x, acc[t][j]);
                            acc[t][j + 1] = fma(ac[r][t], xv.y, acc[t][j + 1]);
                        }
                    }
                }
            }
            if (kn < ke) {
                commit(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }
    auto store = [&](const double (&v)[TM][NC]) {
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            if (i + t >= a.M) continue;
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const int ch = j / C, c = j % C;
                double* yp = a.Y + static_cast<size_t>(ch) * a.ldy + static_cast<size_t>(i + t) * C + c;
                const double s = a.alpha * v[t][j];
                *yp = a.beta != 0.0 ? fma(a.beta, *yp, s) : s;
            }
        }
    };
    if (a.ksplit == 1) {
        store(acc);
        return;
    }
    // split-K: publish partials, the last CTA of the row tile reduces in order
    double* mine = a.part + ((static_cast<size_t>(mt) * a.ksplit + ks) * kDenseThreads + threadIdx.x) * (TM * NC);
    if (!empty) {
#pragma unroll
        for (int t = 0; t < TM; ++t)
#pragma unroll
            for (int j = 0; j < NC; ++j) mine[t * NC + j] = acc[t][j];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(a.cnt + mt, 1) == a.ksplit - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double tot[TM][NC];
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int j = 0; j < NC; ++j) tot[t][j] = 0.0;
    for (int s = 0; s < a.ksplit; ++s) {
        const int64_t s0 = static_cast<int64_t>(s) * a.kper, s1 = mn64(a.K, s0 + a.kper);
        if (dense_tile_empty(a, i0, s0, s1)) continue;
        const double* src = a.part + ((static_cast<size_t>(mt) * a.ksplit + s) * kDenseThreads + threadIdx.x) * (TM * NC);
#pragma unroll
        for (int t = 0; t < TM; ++t)
#pragma unroll
            for (int j = 0; j < NC; ++j) tot[t][j] += __ldcg(src + t * NC + j);
    }
    store(tot);
    if (threadIdx.x == 0) a.cnt[mt] = 0;
}

// ---- fp64 tensor-core (DMMA m8n8k4) variant for NC a multiple of 8 --------
// P = A^T tiles (8 rows x 4 k) and X tiles (4 k x 8 cols) are loaded straight
// into mma fragments from global memory (coalesced 64-byte row pieces of A,
// 64-byte column pieces of X); each warp owns 8 output rows and all NC
// columns, k-steps are software-pipelined kDmmaAhead deep.  No shared memory
// operand traffic, so the kernel is HBM-bound on A.
constexpr int kDmmaWarps = 8;
constexpr int kDmmaRows = 8 * kDmmaWarps;  // rows per CTA tile
constexpr int kDmmaAhead = 8;              // k-steps (of 4) in flight per warp

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int C, int NT>
__global__ void __launch_bounds__(32 * kDmmaWarps) dense_dmma_kernel(DenseArgs a) {
    if (dense_skip(a)) return;
    constexpr int NC = 8 * NT;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int mt = blockIdx.x / a.ksplit, ks = blockIdx.x - mt * a.ksplit;
    const int64_t i0 = static_cast<int64_t>(mt) * kDmmaRows;
    const int64_t iw = i0 + warp * 8;  // this warp's 8 rows
    const int64_t k0 = static_cast<int64_t>(ks) * a.kper;
    const int64_t k1 = mn64(a.K, k0 + a.kper);
    __shared__ int is_last;
    double acc[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
    const int fr = lane >> 2, fk = lane & 3;  // fragment row (A) / col (B), and k
    const bool empty = dense_tile_empty(a, i0, k0, k1);
    if (!empty && iw < a.M) {
        int64_t kb = k0, ke = k1;
        if (a.tri == 1) kb = mx64(kb, iw);
        if (a.tri == 2) ke = mn64(ke, iw + 8);
        kb -= (kb - k0) & 3;
        const int64_t arow = iw + fr;  // P row = A column
        const bool rowok = arow < a.lda;
        // column j = n*8 + fr of the block -> chunk j / C, lane-in-chunk j % C
        size_t xoff[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const int j = n * 8 + fr;
            xoff[n] = static_cast<size_t>(j / C) * a.ldx + (j % C);
        }
        const int64_t nsteps = (ke - kb + 3) >> 2;
        double fa[kDmmaAhead], fb[kDmmaAhead][NT];
        auto load = [&](int64_t st, int slot) {
            const int64_t k = kb + st * 4 + fk;
            const bool ok = st < nsteps && k < ke;
            fa[slot] = (ok && rowok) ? __ldg(a.A + static_cast<size_t>(k) * a.lda + arow) : 0.0;
#pragma unroll
            for (int n = 0; n < NT; ++n)
                fb[slot][n] = ok ? __ldg(a.X + xoff[n] + static_cast<size_t>(k) * C) : 0.0;
        };
#pragma unroll
        for (int u = 0; u < kDmmaAhead; ++u) load(u, u);
        for (int64_t st = 0; st < nsteps; st += kDmmaAhead) {
#pragma unroll
            for (int u = 0; u < kDmmaAhead; ++u) {
                const double av = fa[u];
                double bv[NT];
#pragma unroll
                for (int n = 0; n < NT; ++n) bv[n] = fb[u][n];
                load(st + kDmmaAhead + u, u);  // refill this slot one round ahead
#pragma unroll
                for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[n][0], acc[n][1], av, bv[n]);
            }
        }
    }
    // D fragment: row fr, columns 2*fk, 2*fk+1 of each n-tile
    auto store = [&](const double (&v)[NT][2]) {
        const int64_t row = iw + fr;
        if (row >= a.M) return;
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = n * 8 + 2 * fk + e;
                double* yp = a.Y + static_cast<size_t>(j / C) * a.ldy + static_cast<size_t>(row) * C + (j % C);
                const double s = a.alpha * v[n][e];
                *yp = a.beta != 0.0 ? fma(a.beta, *yp, s) : s;
            }
    };
    if (a.ksplit == 1) {
        store(acc);
        return;
    }
    double* mine = a.part + ((static_cast<size_t>(mt) * a.ksplit + ks) * (32 * kDmmaWarps) + threadIdx.x) * (2 * NT);
    if (!empty) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            mine[2 * n] = acc[n][0];
            mine[2 * n + 1] = acc[n][1];
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(a.cnt + mt, 1) == a.ksplit - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double tot[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) tot[n][0] = tot[n][1] = 0.0;
    for (int sidx = 0; sidx < a.ksplit; ++sidx) {
        const int64_t s0 = static_cast<int64_t>(sidx) * a.kper, s1 = mn64(a.K, s0 + a.kper);
        if (dense_tile_empty(a, i0, s0, s1)) continue;
        const double* src = a.part + ((static_cast<size_t>(mt) * a.ksplit + sidx) * (32 * kDmmaWarps) + threadIdx.x) * (2 * NT);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            tot[n][0] += __ldcg(src + 2 * n);
            tot[n][1] += __ldcg(src + 2 * n + 1);
        }
    }
    store(tot);
    if (threadIdx.x == 0) a.cnt[mt] = 0;
}

// ---- DMMA with shared-memory staged operands, for the big L^-1 products ---
// At R-MAT 18 (n2 ~ 55k, 64 columns) the fragment-from-global kernel above
// re-reads the X block from L2 once per warp (8x the A bytes) and runs at a
// third of the fp64 tensor rate.  Here a CTA owns 128 output rows (8 warps x
// 2 m-fragments) and walks its k range in slabs of 32: A (32 x 128) and X
// (32 x NC) slabs are brought into shared memory by cp.async, double
// buffered, so X is read from L2 once per CTA and every A fragment feeds NT
// DMMAs, every X fragment MT.  Rows are padded to 64 bytes mod 128 so the
// 4 k-rows x 8 doubles of a fragment load hit distinct banks (2 wavefronts).
constexpr int kD2MT = 2;
constexpr int kD2Rows = 8 * kD2MT * kDmmaWarps;  // 128 rows per CTA tile
constexpr int kD2KS = 32;                        // k rows per slab
constexpr int kD2ALd = kD2Rows + 8;              // 136 doubles
constexpr int kD2XLd = 64 + 8;                   // 72 doubles
constexpr size_t kD2Smem = sizeof(double) * 2 * kD2KS * (kD2ALd + kD2XLd);
constexpr int64_t kD2MinDim = 8192;  // smaller operands keep the fragment kernel (faster at cfg1, n2 = 5k)

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

template <int C, int NT>
__global__ void __launch_bounds__(32 * kDmmaWarps, 2) dense_dmma2_kernel(DenseArgs a) {
    if (dense_skip(a)) return;
    constexpr int NC = 8 * NT;
    extern __shared__ __align__(16) double d2s[];
    double* As = d2s;                       // [2][KS][ALd]
    double* Xs = d2s + 2 * kD2KS * kD2ALd;  // [2][KS][XLd]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int mt = blockIdx.x / a.ksplit, ks = blockIdx.x - mt * a.ksplit;
    const int64_t i0 = static_cast<int64_t>(mt) * kD2Rows;
    int64_t k0 = static_cast<int64_t>(ks) * a.kper;
    int64_t k1 = mn64(a.K, k0 + a.kper);
    const bool empty = dense_tile_empty(a, i0, k0, k1);
    if (a.tri == 1) k0 = mx64(k0, i0);            // entries with k < i are stored zeros
    if (a.tri == 2) k1 = mn64(k1, i0 + kD2Rows);  // entries with k > i are stored zeros
    __shared__ int is_last;
    double acc[kD2MT][NT][2];
#pragma unroll
    for (int m = 0; m < kD2MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    const int fr = lane >> 2, fk = lane & 3;
    if (!empty && k0 < k1) {
        const int64_t nslab = (k1 - k0 + kD2KS - 1) / kD2KS;
        auto issue = [&](int64_t s, int buf) {
            const int64_t kk = k0 + s * kD2KS;
            double* as = As + buf * kD2KS * kD2ALd;
            double* xs = Xs + buf * kD2KS * kD2XLd;
            for (int p = threadIdx.x; p < kD2KS * (kD2Rows / 2); p += 32 * kDmmaWarps) {
                const int r = p / (kD2Rows / 2), c2 = (p % (kD2Rows / 2)) * 2;
                const int64_t k = kk + r, i = i0 + c2;
                const bool ok = k < k1 && i < a.lda;
                cp_async16(as + r * kD2ALd + c2, ok ? a.A + static_cast<size_t>(k) * a.lda + i : a.A, ok ? 16 : 0);
            }
            for (int p = threadIdx.x; p < kD2KS * (NC / 2); p += 32 * kDmmaWarps) {
                const int r = p / (NC / 2), j = (p % (NC / 2)) * 2;
                const int64_t k = kk + r;
                const bool ok = k < k1;
                const double* src = a.X + static_cast<size_t>(j / C) * a.ldx + static_cast<size_t>(k) * C + (j % C);
                cp_async16(xs + r * kD2XLd + j, ok ? src : a.X, ok ? 16 : 0);
            }
            cp_async_commit();
        };
        issue(0, 0);
        for (int64_t s = 0; s < nslab; ++s) {
            if (s + 1 < nslab) issue(s + 1, static_cast<int>((s + 1) & 1));
            else cp_async_commit();
            cp_async_wait1();
            __syncthreads();
            const double* as = As + (s & 1) * kD2KS * kD2ALd + warp * (8 * kD2MT) + fr;
            const double* xs = Xs + (s & 1) * kD2KS * kD2XLd + fr;
#pragma unroll
            for (int st = 0; st < kD2KS / 4; ++st) {
                const int kr = st * 4 + fk;
                double av[kD2MT], bv[NT];
#pragma unroll
                for (int m = 0; m < kD2MT; ++m) av[m] = as[kr * kD2ALd + m * 8];
#pragma unroll
                for (int n = 0; n < NT; ++n) bv[n] = xs[kr * kD2XLd + n * 8];
#pragma unroll
                for (int m = 0; m < kD2MT; ++m)
#pragma unroll
                    for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], av[m], bv[n]);
            }
            __syncthreads();
        }
    }
    auto store = [&](const double (&v)[kD2MT][NT][2]) {
#pragma unroll
        for (int m = 0; m < kD2MT; ++m) {
            const int64_t row = i0 + warp * (8 * kD2MT) + m * 8 + fr;
            if (row >= a.M) continue;
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = n * 8 + 2 * fk + e;
                    double* yp = a.Y + static_cast<size_t>(j / C) * a.ldy + static_cast<size_t>(row) * C + (j % C);
                    const double s = a.alpha * v[m][n][e];
                    *yp = a.beta != 0.0 ? fma(a.beta, *yp, s) : s;
                }
        }
    };
    if (a.ksplit == 1) {
        store(acc);
        return;
    }
    constexpr int PER = kD2MT * NT * 2;
    double* mine = a.part + ((static_cast<size_t>(mt) * a.ksplit + ks) * (32 * kDmmaWarps) + threadIdx.x) * PER;
    if (!empty) {
#pragma unroll
        for (int m = 0; m < kD2MT; ++m)
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                mine[(m * NT + n) * 2] = acc[m][n][0];
                mine[(m * NT + n) * 2 + 1] = acc[m][n][1];
            }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(a.cnt + mt, 1) == a.ksplit - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double tot[kD2MT][NT][2];
#pragma unroll
    for (int m = 0; m < kD2MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) tot[m][n][0] = tot[m][n][1] = 0.0;
    for (int sidx = 0; sidx < a.ksplit; ++sidx) {
        const int64_t s0 = static_cast<int64_t>(sidx) * a.kper, s1 = mn64(a.K, s0 + a.kper);
        if (dense_tile_empty(a, i0, s0, s1)) continue;
        const double* src = a.part + ((static_cast<size_t>(mt) * a.ksplit + sidx) * (32 * kDmmaWarps) + threadIdx.x) * PER;
#pragma unroll
        for (int m = 0; m < kD2MT; ++m)
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                tot[m][n][0] += __ldcg(src + (m * NT + n) * 2);
                tot[m][n][1] += __ldcg(src + (m * NT + n) * 2 + 1);
            }
    }
    store(tot);
    if (threadIdx.x == 0) a.cnt[mt] = 0;
}

struct DenseScratch {
    double* part = nullptr;
    int32_t* cnt = nullptr;
    size_t part_cap = 0;  // doubles
    int64_t cnt_cap = 0;
};

inline void dense_plan(int64_t M, int64_t K, int& mtiles, int& ksplit, int64_t& kper,
                       int64_t rows_tile = kDenseRows) {
    mtiles = static_cast<int>((M + rows_tile - 1) / rows_tile);
    const int64_t kblocks = (K + kDenseK - 1) / kDenseK;
    int64_t want = (4 * num_sms() + mtiles - 1) / mtiles;  // ~4 CTAs per SM
    want = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, kblocks), kDenseMaxSplit));
    kper = ((kblocks + want - 1) / want) * kDenseK;
    ksplit = static_cast<int>((K + kper - 1) / kper);
    if (ksplit < 1) ksplit = 1;
}

inline size_t dense_part_doubles(int64_t M, int64_t K, int NC) {
    size_t best = 0;
    for (int64_t rows : {static_cast<int64_t>(kDenseThreads), static_cast<int64_t>(kDenseRows),
                         static_cast<int64_t>(kDmmaRows), static_cast<int64_t>(kD2Rows)}) {
        int mtiles, ksplit;
        int64_t kper;
        dense_plan(M, K, mtiles, ksplit, kper, rows);
        if (ksplit > 1) best = std::max(best, static_cast<size_t>(mtiles) * ksplit * rows * NC);
    }
    return best;
}

// Y(chunks [c0, c0+nch)) = alpha * op(A) X + beta * Y, looping over groups
// of chunks so each launch handles <= 64 columns.  lda must be even with
// A zero-padded up to lda columns (16-byte aligned pair loads).
inline int launch_dense(const double* A, int64_t lda, int64_t M, int64_t K, int tri, const double* X,
                        int64_t ldx, double* Y, int64_t ldy, double alpha, double beta, int C, int nch,
                        const DenseScratch& ds, cudaStream_t st, const int32_t* chunk_active = nullptr) {
    if (M == 0) return KZ_OK;
    if (lda % 2 != 0 || lda < M + (M & 1)) return fail(KZ_EARG, "dense operand needs an even, padded lda");
    auto group = [&](int left) {
        if (C == 1) return left >= 16 ? 16 : left >= 8 ? 8 : left >= 4 ? 4 : left >= 2 ? 2 : 1;
        if (C == 16) return std::min(left, 4);
        if (C == 32) return std::min(left, 2);
        return 1;
    };
    for (int c0 = 0, g = 0; c0 < nch; c0 += g) {
        g = group(nch - c0);
        if (C >= 8 && (C * g) % 8 == 0 && M >= kD2MinDim && K >= kD2MinDim) {
            const int nt = C * g / 8;
            int mtiles, ksplit;
            int64_t kper;
            dense_plan(M, K, mtiles, ksplit, kper, kD2Rows);
            DenseArgs a{};
            a.rows_tile = kD2Rows;
            a.A = A;
            a.lda = lda;
            a.M = M;
            a.K = K;
            a.tri = tri;
            a.X = X + static_cast<size_t>(c0) * ldx;
            a.ldx = ldx;
            a.Y = Y + static_cast<size_t>(c0) * ldy;
            a.ldy = ldy;
            a.alpha = alpha;
            a.beta = beta;
            a.ksplit = ksplit;
            a.kper = kper;
            a.part = ds.part;
            a.cnt = ds.cnt;
            a.chunk_active = chunk_active ? chunk_active + c0 : nullptr;
            a.nchunk = g;
            if (ksplit > 1 && (static_cast<size_t>(mtiles) * ksplit * kD2Rows * g * C > ds.part_cap ||
                               mtiles > ds.cnt_cap))
                return fail(KZ_EARG, "dense scratch too small");
            const unsigned grid = static_cast<unsigned>(mtiles) * ksplit;
#define KZ_DMMA2(CC, NN)                                                                                  \
    do {                                                                                                  \
        static bool attr = false;                                                                         \
        if (!attr) {                                                                                      \
            KZ_CUDA(cudaFuncSetAttribute(dense_dmma2_kernel<CC, NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         static_cast<int>(kD2Smem)));                                     \
            attr = true;                                                                                  \
        }                                                                                                 \
        dense_dmma2_kernel<CC, NN><<<grid, 32 * kDmmaWarps, kD2Smem, st>>>(a);                            \
    } while (0)
            if (C == 8 && nt == 1) KZ_DMMA2(8, 1);
            else if (C == 16 && nt == 2) KZ_DMMA2(16, 2);
            else if (C == 16 && nt == 4) KZ_DMMA2(16, 4);
            else if (C == 16 && nt == 6) KZ_DMMA2(16, 6);
            else if (C == 16 && nt == 8) KZ_DMMA2(16, 8);
            else if (C == 32 && nt == 4) KZ_DMMA2(32, 4);
            else if (C == 32 && nt == 8) KZ_DMMA2(32, 8);
            else return fail(KZ_EARG, "dmma2: unsupported column group");
#undef KZ_DMMA2
            note_launch();
            KZ_LAUNCH_CHECK();
            continue;
        }
        if ((C * g) % 8 == 0) {
            const int nt = C * g / 8;
            int mtiles, ksplit;
            int64_t kper;
            dense_plan(M, K, mtiles, ksplit, kper, kDmmaRows);
            DenseArgs a{};
            a.rows_tile = kDmmaRows;
            a.A = A;
            a.lda = lda;
            a.M = M;
            a.K = K;
            a.tri = tri;
            a.X = X + static_cast<size_t>(c0) * ldx;
            a.ldx = ldx;
            a.Y = Y + static_cast<size_t>(c0) * ldy;
            a.ldy = ldy;
            a.alpha = alpha;
            a.beta = beta;
            a.ksplit = ksplit;
            a.kper = kper;
            a.part = ds.part;
            a.cnt = ds.cnt;
            a.chunk_active = chunk_active ? chunk_active + c0 : nullptr;
            a.nchunk = g;
            if (ksplit > 1 && (static_cast<size_t>(mtiles) * ksplit * kDmmaRows * g * C > ds.part_cap ||
                               mtiles > ds.cnt_cap))
                return fail(KZ_EARG, "dense scratch too small");
            const unsigned grid = static_cast<unsigned>(mtiles) * ksplit;
#define KZ_DMMA(CC, NN) dense_dmma_kernel<CC, NN><<<grid, 32 * kDmmaWarps, 0, st>>>(a)
            if (C == 8 && nt == 1) KZ_DMMA(8, 1);
            else if (C == 16 && nt == 2) KZ_DMMA(16, 2);
            else if (C == 16 && nt == 4) KZ_DMMA(16, 4);
            else if (C == 16 && nt == 6) KZ_DMMA(16, 6);
            else if (C == 16 && nt == 8) KZ_DMMA(16, 8);
            else if (C == 32 && nt == 4) KZ_DMMA(32, 4);
            else if (C == 32 && nt == 8) KZ_DMMA(32, 8);
            else if (C == 1 && nt == 1) KZ_DMMA(1, 1);
            else if (C == 1 && nt == 2) KZ_DMMA(1, 2);
            else return fail(KZ_EARG, "dmma: unsupported column group");
#undef KZ_DMMA
            note_launch();
            KZ_LAUNCH_CHECK();
            continue;
        }
        const int tm = 1;  // TM = 2 spills under the 2-CTA register budget
        int mtiles, ksplit;
        int64_t kper;
        dense_plan(M, K, mtiles, ksplit, kper, static_cast<int64_t>(kDenseThreads) * tm);
        DenseArgs a{};
        a.rows_tile = static_cast<int64_t>(kDenseThreads) * tm;
        a.A = A;
        a.lda = lda;
        a.M = M;
        a.K = K;
        a.tri = tri;
        a.X = X + static_cast<size_t>(c0) * ldx;
        a.ldx = ldx;
        a.Y = Y + static_cast<size_t>(c0) * ldy;
        a.ldy = ldy;
        a.alpha = alpha;
        a.beta = beta;
        a.ksplit = ksplit;
        a.kper = kper;
        a.part = ds.part;
        a.cnt = ds.cnt;
        a.chunk_active = chunk_active ? chunk_active + c0 : nullptr;
        a.nchunk = g;
        if (ksplit > 1 && (static_cast<size_t>(mtiles) * ksplit * a.rows_tile * g * C > ds.part_cap ||
                           mtiles > ds.cnt_cap))
            return fail(KZ_EARG, "dense scratch too small");
        const unsigned grid = static_cast<unsigned>(mtiles) * ksplit;
        const int nc = C * g;
#define KZ_DENSE(CC, NN, TT) dense_kernel<CC, NN, TT><<<grid, kDenseThreads, 0, st>>>(a)
        if (C == 1 && g == 1) KZ_DENSE(1, 1, 1);
        else if (C == 1 && g == 2) KZ_DENSE(1, 2, 1);
        else if (C == 1 && g == 4) KZ_DENSE(1, 4, 1);
        else if (C == 1 && g == 8) KZ_DENSE(1, 8, 1);
        else if (C == 1 && g == 16) KZ_DENSE(1, 16, 1);
        else if (C == 2 && g == 1) KZ_DENSE(2, 1, 1);
        else if (C == 4 && g == 1) KZ_DENSE(4, 1, 1);
        else if (C == 8 && g == 1) KZ_DENSE(8, 1, 1);
        else if (C == 16 && g == 1) KZ_DENSE(16, 1, 1);
        else if (C == 16 && g == 2) KZ_DENSE(16, 2, 1);
        else if (C == 16 && g == 3) KZ_DENSE(16, 3, 1);
        else if (C == 16 && g == 4) KZ_DENSE(16, 4, 1);
        else if (C == 32 && g == 1) KZ_DENSE(32, 1, 1);
        else if (C == 32 && g == 2) KZ_DENSE(32, 2, 1);
        else return fail(KZ_EARG, "dense: unsupported column group " + std::to_string(nc));
#undef KZ_DENSE
        note_launch();
        KZ_LAUNCH_CHECK();
    }
    return KZ_OK;
}

}  // namespace kz
