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
// tile reduces the split partials in a fixed order (deterministic).  fp64
// has no tcgen05 kind on sm_100a and the DMMA rate equals the CUDA-core
// DFMA rate on B200, so this is a bandwidth-first CUDA-core kernel.
#pragma once

#include "spmm.cuh"

namespace kz {

__host__ __device__ __forceinline__ int64_t mn64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t mx64(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr int kDenseRows = 256;  // output rows per CTA (one per thread)
constexpr int kDenseK = 32;      // k rows staged per step
constexpr int kDenseMaxCols = 64;

struct DenseArgs {
    const double* A;
    int64_t lda, M, K;
    int tri;  // 0 full, 1: only k >= i nonzero, 2: only k <= i nonzero
    const double* X;
    int64_t ldx;  // chunk stride of X (K rows)
    double* Y;
    int64_t ldy;  // chunk stride of Y (M rows)
    double alpha, beta;
    int ksplit;
    int64_t kper;
    double* part;  // [mtiles][ksplit][256][NC]
    int32_t* cnt;  // [mtiles]
};

__device__ __forceinline__ bool dense_tile_empty(const DenseArgs& a, int64_t i0, int64_t k0, int64_t k1) {
    if (k0 >= k1) return true;
    const int64_t i1 = mn64(a.M, i0 + kDenseRows) - 1;
    if (a.tri == 1 && k1 - 1 < i0) return true;  // needs some k >= i
    if (a.tri == 2 && k0 > i1) return true;      // needs some k <= i
    return false;
}

template <int C, int NCH>
__global__ void __launch_bounds__(kDenseRows) dense_kernel(DenseArgs a) {
    constexpr int NC = C * NCH;
    const int mt = blockIdx.x / a.ksplit, ks = blockIdx.x - mt * a.ksplit;
    const int64_t i0 = static_cast<int64_t>(mt) * kDenseRows;
    const int64_t i = i0 + threadIdx.x;
    const int64_t k0 = static_cast<int64_t>(ks) * a.kper;
    const int64_t k1 = mn64(a.K, k0 + a.kper);
    __shared__ double xs[kDenseK][NC];
    __shared__ int is_last;
    double acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = 0.0;
    const bool empty = dense_tile_empty(a, i0, k0, k1);
    if (!empty) {
        // triangular bounds for this tile
        int64_t kb = k0, ke = k1;
        if (a.tri == 1) kb = mx64(kb, i0);
        if (a.tri == 2) ke = mn64(ke, mn64(a.M, i0 + kDenseRows));
        kb -= (kb - k0) % kDenseK;  // keep the staging aligned to the split start
        const bool valid = i < a.M;
        for (int64_t kk = kb; kk < ke; kk += kDenseK) {
            const int nk = static_cast<int>(mn64(kDenseK, ke - kk));
            __syncthreads();
            for (int e = threadIdx.x; e < kDenseK * NC; e += kDenseRows) {
                const int r = e / NC, j = e % NC;
                const int ch = j / C, c = j % C;
                xs[r][j] = r < nk ? a.X[static_cast<size_t>(ch) * a.ldx + static_cast<size_t>(kk + r) * C + c] : 0.0;
            }
            __syncthreads();
            if (valid) {
                const double* Ap = a.A + static_cast<size_t>(kk) * a.lda + i;
#pragma unroll 8
                for (int r = 0; r < kDenseK; ++r) {
                    const double av = r < nk ? __ldg(Ap + static_cast<size_t>(r) * a.lda) : 0.0;
#pragma unroll
                    for (int j = 0; j < NC; ++j) acc[j] = fma(av, xs[r][j], acc[j]);
                }
            }
        }
    }
    auto store = [&](const double (&v)[NC]) {
        if (i >= a.M) return;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            const int ch = j / C, c = j % C;
            double* yp = a.Y + static_cast<size_t>(ch) * a.ldy + static_cast<size_t>(i) * C + c;
            const double s = a.alpha * v[j];
            *yp = a.beta != 0.0 ? fma(a.beta, *yp, s) : s;
        }
    };
    if (a.ksplit == 1) {
        store(acc);
        return;
    }
    // split-K: publish partials, the last CTA of the row tile reduces in order
    double* mine = a.part + ((static_cast<size_t>(mt) * a.ksplit + ks) * kDenseRows + threadIdx.x) * NC;
    if (!empty) {
#pragma unroll
        for (int j = 0; j < NC; ++j) mine[j] = acc[j];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(a.cnt + mt, 1) == a.ksplit - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double tot[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) tot[j] = 0.0;
    for (int s = 0; s < a.ksplit; ++s) {
        const int64_t s0 = static_cast<int64_t>(s) * a.kper, s1 = mn64(a.K, s0 + a.kper);
        if (dense_tile_empty(a, i0, s0, s1)) continue;
        const double* src = a.part + ((static_cast<size_t>(mt) * a.ksplit + s) * kDenseRows + threadIdx.x) * NC;
#pragma unroll
        for (int j = 0; j < NC; ++j) tot[j] += __ldcg(src + j);
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

inline void dense_plan(int64_t M, int64_t K, int& mtiles, int& ksplit, int64_t& kper) {
    mtiles = static_cast<int>((M + kDenseRows - 1) / kDenseRows);
    const int64_t kblocks = (K + kDenseK - 1) / kDenseK;
    int64_t want = (2 * kNumSMs + mtiles - 1) / mtiles;  // ~2 CTAs per SM
    want = std::max<int64_t>(1, std::min<int64_t>(want, kblocks));
    kper = ((kblocks + want - 1) / want) * kDenseK;
    ksplit = static_cast<int>((K + kper - 1) / kper);
    if (ksplit < 1) ksplit = 1;
}

inline size_t dense_part_doubles(int64_t M, int64_t K, int NC) {
    int mtiles, ksplit;
    int64_t kper;
    dense_plan(M, K, mtiles, ksplit, kper);
    return ksplit > 1 ? static_cast<size_t>(mtiles) * ksplit * kDenseRows * NC : 0;
}

// Y(chunks [c0, c0+nch)) = alpha * op(A) X + beta * Y, looping over groups
// of chunks so each launch handles <= 64 columns.
inline int launch_dense(const double* A, int64_t lda, int64_t M, int64_t K, int tri, const double* X,
                        int64_t ldx, double* Y, int64_t ldy, double alpha, double beta, int C, int nch,
                        const DenseScratch& ds, cudaStream_t st) {
    if (M == 0) return KZ_OK;
    int mtiles, ksplit;
    int64_t kper;
    dense_plan(M, K, mtiles, ksplit, kper);
    // chunks per launch: the instantiated (C, NCH) combinations below
    auto group = [&](int left) {
        if (C == 1) return left >= 16 ? 16 : left >= 8 ? 8 : left >= 4 ? 4 : left >= 2 ? 2 : 1;
        if (C == 16) return std::min(left, 4);
        if (C == 32) return std::min(left, 2);
        return 1;
    };
    for (int c0 = 0, g = 0; c0 < nch; c0 += g) {
        g = group(nch - c0);
        DenseArgs a{};
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
        if (ksplit > 1 && (static_cast<size_t>(mtiles) * ksplit * kDenseRows * g * C > ds.part_cap ||
                           mtiles > ds.cnt_cap))
            return fail(KZ_EARG, "dense scratch too small");
        const unsigned grid = static_cast<unsigned>(mtiles) * ksplit;
        // NC = C*g must be one of the instantiated widths
        const int nc = C * g;
#define KZ_DENSE(CC, NN) dense_kernel<CC, NN><<<grid, kDenseRows, 0, st>>>(a)
        if (C == 1 && g == 1) KZ_DENSE(1, 1);
        else if (C == 1 && g == 2) KZ_DENSE(1, 2);
        else if (C == 1 && g == 4) KZ_DENSE(1, 4);
        else if (C == 1 && g == 8) KZ_DENSE(1, 8);
        else if (C == 1 && g == 16) KZ_DENSE(1, 16);
        else if (C == 2 && g == 1) KZ_DENSE(2, 1);
        else if (C == 4 && g == 1) KZ_DENSE(4, 1);
        else if (C == 8 && g == 1) KZ_DENSE(8, 1);
        else if (C == 16 && g == 1) KZ_DENSE(16, 1);
        else if (C == 16 && g == 2) KZ_DENSE(16, 2);
        else if (C == 16 && g == 3) KZ_DENSE(16, 3);
        else if (C == 16 && g == 4) KZ_DENSE(16, 4);
        else if (C == 32 && g == 1) KZ_DENSE(32, 1);
        else if (C == 32 && g == 2) KZ_DENSE(32, 2);
        else return fail(KZ_EARG, "dense: unsupported column group " + std::to_string(nc));
#undef KZ_DENSE
        note_launch();
        KZ_LAUNCH_CHECK();
    }
    return KZ_OK;
}

}  // namespace kz
