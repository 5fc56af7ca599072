// blockops.cuh -- streaming kernels over chunked blocks [b/C][rows][C]:
// deterministic column dots with a per-chunk finalize hook, the fused CG
// vector updates, layout transposes in/out.  Shared by the CG (cg.cu) and
// the LRC Schur-PCG (lrc.cu) drivers.
#pragma once

#include "spmm.cuh"

namespace kz {

// Per-column solver state (device arrays of length bpad unless noted).
struct SolveState {
    int32_t b = 0, bpad = 0, C = 0, nchunks = 0;
    int64_t rows = 0;
    int64_t max_iter = 0;
    double tol = 0.0;
    double* rs = nullptr;      // r.r (CG) / r.z (PCG)
    double* alpha = nullptr;   // step length of the current iteration
    double* betac = nullptr;   // direction update coefficient
    double* thresh = nullptr;  // tol * ||b||
    double* rnorm = nullptr;   // ||r|| (recursive)
    double* bnorm2 = nullptr;  // ||b||^2
    double* rr = nullptr;      // scratch: r.r of the current iteration (PCG)
    int64_t* iters = nullptr;
    int32_t* active = nullptr;
    int32_t* xstamp = nullptr;
    int32_t* status = nullptr;
    int32_t* converged = nullptr;
    int32_t* chunk_active = nullptr;  // [nchunks]
    int32_t* chunk_xstamp = nullptr;  // [nchunks]
    int32_t* n_active = nullptr;      // [1]
    int32_t* err = nullptr;           // [1]
    int32_t* iter_dev = nullptr;      // [1] iteration number for graph replay (NULL: host-passed)
    // residual-history CG (cg.cu): the convergence finalize records each
    // column's step length a_k and direction coefficient beta_k of
    // iterations 1..hist_len into [hist_len][bpad] (pre-zeroed)
    double* ahist = nullptr;
    double* bhist = nullptr;
    int32_t hist_len = 0;
};

// The iteration number a kernel of the solve loop works on: passed by the
// host, or read from the device counter when the loop is a replayed graph.
__device__ __forceinline__ int cur_iter(const SolveState& s, int iter) { return s.iter_dev ? *s.iter_dev : iter; }

enum FinalizeMode : int {
    FIN_WRITE = 0,      // out[col] = v
    FIN_INIT_B = 1,     // bnorm2 = v
    FIN_INIT_BR = 2,    // bnorm2 = v and r == b: run init finalize
    FIN_INIT_R = 3,     // v = r.r after a start vector: run init finalize
    FIN_CG_CONV = 4,    // v = r.r after the update: convergence test (cg)
    FIN_PCG_RR = 5,     // v = r.r after the update: store, test convergence (pcg)
    FIN_PCG_RZ = 6,     // v = r.z: direction coefficient (pcg)
    FIN_PCG_INIT_RZ = 7 // v = r.z at start: rs = v (pcg)
};

// init finalize shared by cg() and lrc_pcg(): solver.py:71-77 / 127-133
__device__ __forceinline__ bool init_finalize(const SolveState& s, int col, double rr) {
    const double bn = sqrt(s.bnorm2[col]);
    s.thresh[col] = s.tol * bn;
    const double rn = sqrt(rr);
    s.rnorm[col] = rn;
    s.rs[col] = rr;
    s.iters[col] = 0;
    const bool act = rn > s.thresh[col];
    s.active[col] = act ? 1 : 0;
    s.converged[col] = act ? 0 : 1;
    if (act) atomicAdd(s.n_active, 1);
    return act;
}

// Applies the finalize of `mode` for the C columns of `chunk`; run by the
// last CTA of the chunk with v valid in threads < C.  Returns nothing; keeps
// chunk_active in sync.
template <int C>
__device__ __forceinline__ void finalize_chunk(int mode, const SolveState& s, double* out,
                                               int chunk, int iter, double v) {
    const int col = chunk * C + threadIdx.x;
    bool act = false;
    if (threadIdx.x < C) {
        if (mode == FIN_WRITE) {
            if (out) out[col] = v;
        } else if (col >= s.b) {
            act = false;
        } else if (mode == FIN_INIT_B) {
            s.bnorm2[col] = v;
        } else if (mode == FIN_INIT_BR) {
            s.bnorm2[col] = v;
            act = init_finalize(s, col, v);
        } else if (mode == FIN_INIT_R) {
            act = init_finalize(s, col, v);
        } else if (mode == FIN_CG_CONV) {
            // solver.py:89-95
            if (s.xstamp[col] == iter && s.active[col]) {
                const int64_t it = s.iters[col] + 1;
                s.iters[col] = it;
                const double rn = sqrt(v);
                s.rnorm[col] = rn;
                if (rn <= s.thresh[col]) {
                    s.active[col] = 0;
                    s.converged[col] = 1;
                    atomicSub(s.n_active, 1);
                } else if (it >= s.max_iter) {
                    s.active[col] = 0;
                    atomicSub(s.n_active, 1);
                } else {
                    s.betac[col] = v / s.rs[col];
                    s.rs[col] = v;
                }
                if (s.ahist && iter <= s.hist_len) {
                    const size_t h = static_cast<size_t>(iter - 1) * s.bpad + col;
                    s.ahist[h] = s.alpha[col];
                    s.bhist[h] = s.active[col] ? s.betac[col] : 0.0;
                }
            }
            act = s.active[col] != 0;
        } else if (mode == FIN_PCG_RR) {
            // solver.py:145-148 (norm of r, stop test)
            if (s.xstamp[col] == iter && s.active[col]) {
                const int64_t it = s.iters[col] + 1;
                s.iters[col] = it;
                const double rn = sqrt(v);
                s.rnorm[col] = rn;
                if (rn <= s.thresh[col]) {
                    s.active[col] = 0;
                    s.converged[col] = 1;
                    atomicSub(s.n_active, 1);
                } else if (it >= s.max_iter) {
                    s.active[col] = 0;
                    atomicSub(s.n_active, 1);
                }
            }
            act = s.active[col] != 0;
        } else if (mode == FIN_PCG_RZ) {
            // solver.py:150-152
            if (s.active[col]) {
                s.betac[col] = v / s.rs[col];
                s.rs[col] = v;
            }
            act = s.active[col] != 0;
        } else if (mode == FIN_PCG_INIT_RZ) {
            if (s.active[col]) s.rs[col] = v;
            act = s.active[col] != 0;
        }
    }
    if (mode != FIN_WRITE && mode != FIN_INIT_B && s.chunk_active) {
        const int any = __syncthreads_or(act ? 1 : 0);
        if (threadIdx.x == 0) s.chunk_active[chunk] = any;
    }
}

// Reduce per-thread column values (thread owns columns ((tid*VEC)%C)+q) to
// one value per column in threads < C.  sm: kThreads doubles.
template <int C, int VEC>
__device__ __forceinline__ double block_col_reduce(double (&v)[VEC], double* sm) {
    constexpr int G = C / VEC;  // lanes covering one row segment of C columns
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = G; off < 32; off <<= 1)
#pragma unroll
        for (int q = 0; q < VEC; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
    if (lane < G) {
#pragma unroll
        for (int q = 0; q < VEC; ++q) sm[warp * C + lane * VEC + q] = v[q];
    }
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < C)
        for (int w = 0; w < kWarps; ++w) s += sm[w * C + threadIdx.x];
    __syncthreads();
    return s;
}

struct RedScratch {
    double* part = nullptr;   // [nchunks][nb][C]
    int32_t* cnt = nullptr;   // [nchunks]
    int nb = 1;               // CTAs per chunk
};

// Last-CTA-of-chunk protocol: write this CTA's partial, count, and return
// true (with the fixed-order total in threads < C) in the last CTA.
template <int C>
__device__ __forceinline__ bool chunk_last_reduce(const RedScratch& rs, int chunk, int local,
                                                  double mine, double* sm, double& total) {
    __shared__ int is_last;
    if (threadIdx.x < C) {
        rs.part[(static_cast<size_t>(chunk) * rs.nb + local) * C + threadIdx.x] = mine;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(rs.cnt + chunk, 1) == rs.nb - 1);
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    total = reduce_partials<C>(rs.part + static_cast<size_t>(chunk) * rs.nb * C, rs.nb, sm);
    if (threadIdx.x == 0) rs.cnt[chunk] = 0;
    return true;
}

// out/hook = column dots X.Y over a chunked block.
template <int C>
__global__ void __launch_bounds__(kThreads)
    coldot_kernel(const double* __restrict__ X, const double* __restrict__ Y, int64_t rows,
                  int64_t ldx, int64_t ldy, RedScratch red, int mode, SolveState s, double* out,
                  int iter) {
    constexpr int VEC = Cfg<C>::SVEC;
    const int chunk = blockIdx.x / red.nb, local = blockIdx.x - chunk * red.nb;
    const double* Xb = X + static_cast<size_t>(chunk) * ldx;
    const double* Yb = Y + static_cast<size_t>(chunk) * ldy;
    const size_t npairs = static_cast<size_t>(rows) * C / VEC;
    const size_t stride = static_cast<size_t>(red.nb) * kThreads;
    double acc[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
    for (size_t pi = static_cast<size_t>(local) * kThreads + threadIdx.x; pi < npairs; pi += stride) {
        double x[VEC], y[VEC];
        ld_plain<VEC>(Xb + pi * VEC, x);
        ld_plain<VEC>(Yb + pi * VEC, y);
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = fma(x[q], y[q], acc[q]);
    }
    __shared__ double sm[kThreads];
    const double mine = block_col_reduce<C, VEC>(acc, sm);
    double total;
    if (chunk_last_reduce<C>(red, chunk, local, mine, sm, total))
        finalize_chunk<C>(mode, s, out, chunk, cur_iter(s, iter), total);
}

// CG residual update (solver.py:88-90) fused with r.r:  r -= a*q for the
// columns active in this iteration.  Sparse first iteration (cnt given, see
// cg_sparse_pq_kernel): q = p - beta*A p is formed on the fly from p = r and
// the 2-walk counts, (A p)_i = beta * cnt_i, with K1's epilogue roundings.
template <int C>
__global__ void __launch_bounds__(kThreads)
    cg_update_kernel(double* __restrict__ r, const double* __restrict__ q, int64_t rows,
                     int64_t ldr, int64_t ldq, RedScratch red, int mode, SolveState s, int iter,
                     const int32_t* __restrict__ cnt = nullptr, double beta = 0.0,
                     double* __restrict__ r_out = nullptr, double* __restrict__ q_out = nullptr) {
    constexpr int VEC = Cfg<C>::SVEC;
    const int chunk = blockIdx.x / red.nb, local = blockIdx.x - chunk * red.nb;
    iter = cur_iter(s, iter);
    if (s.chunk_xstamp[chunk] != iter) return;
    r += static_cast<size_t>(chunk) * ldr;
    q += static_cast<size_t>(chunk) * ldq;
    if (cnt) cnt += static_cast<size_t>(chunk) * ldq;
    // history mode: r_{k+1} goes to its own slot, r_k stays for the final x
    double* __restrict__ ro = r_out ? r_out + static_cast<size_t>(chunk) * ldr : r;
    // sparse first iteration of the q-recurrence: q0 (formed from the counts)
    // is kept for the next iteration's q1 = M r1 + beta_0 q0
    double* __restrict__ qo = q_out ? q_out + static_cast<size_t>(chunk) * ldq : nullptr;
    const size_t npairs = static_cast<size_t>(rows) * C / VEC;
    const size_t stride = static_cast<size_t>(red.nb) * kThreads;
    const size_t t0 = static_cast<size_t>(local) * kThreads + threadIdx.x;
    const int c0 = static_cast<int>((t0 * VEC) % C);  // fixed column of this thread
    double a[VEC];
    bool on[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
        const int col = chunk * C + c0 + q;
        on[q] = col < s.b && s.xstamp[col] == iter;
        a[q] = on[q] ? s.alpha[col] : 0.0;
    }
    double acc[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
    for (size_t pi = t0; pi < npairs; pi += stride) {
        double rv[VEC], qv[VEC];
        ld_plain<VEC>(r + pi * VEC, rv);
        if (cnt) {
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                const int32_t c = __ldcs(cnt + pi * VEC + k);
                qv[k] = __dadd_rn(rv[k], __dmul_rn(-beta, __dmul_rn(beta, static_cast<double>(c))));
            }
            if (qo) st_plain<VEC>(qo + pi * VEC, qv);
        } else {
            ld_plain<VEC>(q + pi * VEC, qv);
        }
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            if (on[k]) rv[k] = __dsub_rn(rv[k], __dmul_rn(a[k], qv[k]));
            acc[k] = fma(rv[k], rv[k], acc[k]);
        }
        st_plain<VEC>(ro + pi * VEC, rv);
    }
    __shared__ double sm[kThreads];
    const double mine = block_col_reduce<C, VEC>(acc, sm);
    double total;
    if (chunk_last_reduce<C>(red, chunk, local, mine, sm, total))
        finalize_chunk<C>(mode, s, nullptr, chunk, iter, total);
}

// Sparse first CG iteration of a Katz solve from zero: p0 = r0 = b =
// beta A e_q lives on N(q), so q0 = p0 - beta A p0 needs only
// (A p0)_i = beta * cnt_i with cnt = A^2 e_q the 2-walk counts
// (walk2_count_kernel), and p0.q0 is a sum over N(q).  One CTA per column:
// the fixed-order p0.q0 and the K1 step-length hook (solver.py:83-87:
// a = rs/pq, RuntimeError if pq <= 0); cg_update_kernel then forms q0 from
// the counts.  Replaces the iteration's SpMM (R-MAT 22: 33 G gathered values)
// by sum_{t in N(q)} deg(t) integer increments.
template <int C>
__global__ void __launch_bounds__(kThreads)
    cg_sparse_pq_kernel(const double* __restrict__ r, const int32_t* __restrict__ cnt, int64_t ld,
                        const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                        const int64_t* __restrict__ qpos, double beta, SolveState s, int iter) {
    const int j = blockIdx.x, chunk = j / C;
    if (j % C == 0 && threadIdx.x == 0 && s.chunk_active[chunk]) s.chunk_xstamp[chunk] = iter;
    if (j >= s.b || !s.active[j]) return;
    const int64_t q = qpos[j];
    const int beg = rowptr[q], end = rowptr[q + 1];
    const size_t base = static_cast<size_t>(chunk) * ld + (j % C);
    double acc = 0.0;
    for (int k = beg + threadIdx.x; k < end; k += blockDim.x) {
        const size_t off = base + static_cast<size_t>(colidx[k]) * C;
        const double pv = r[off];
        const double qv = __dadd_rn(pv, __dmul_rn(-beta, __dmul_rn(beta, static_cast<double>(cnt[off]))));
        acc = fma(pv, qv, acc);
    }
    __shared__ double sm[kThreads];
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double v = sm[0];
        if (v <= 0.0) {
            s.status[j] = KZ_ENOTSPD;
            s.active[j] = 0;
            atomicExch(s.err, 1);
            atomicSub(s.n_active, 1);
        } else {
            s.alpha[j] = s.rs[j] / v;
            s.xstamp[j] = iter;
        }
    }
}

// Deferred solution update and new direction (solver.py:87, 95 / 144, 151):
//   x += a*p   for columns active in this iteration
//   p  = d + betac*p  for columns still active   (d = r for CG, z for PCG)
template <int C>
__global__ void __launch_bounds__(kThreads)
    cg_pupdate_kernel(double* __restrict__ x, double* __restrict__ p, const double* __restrict__ d,
                      int64_t rows, int64_t ldx, int64_t ldp, int64_t ldd, int nb, SolveState s,
                      int iter, double* __restrict__ ahist = nullptr, double* __restrict__ bhist = nullptr,
                      const double* __restrict__ p_in = nullptr) {
    constexpr int VEC = Cfg<C>::SVEC;
    const int chunk = blockIdx.x / nb, local = blockIdx.x - chunk * nb;
    iter = cur_iter(s, iter);
    if (s.chunk_xstamp[chunk] != iter) return;
    // history mode (x == nullptr): record this iteration's step length and
    // direction coefficient per column; x is formed at the end from the
    // residual history (cg_hist_coef_kernel / cg_hist_sum)
    if (ahist && local == 0 && threadIdx.x < C) {
        const int col = chunk * C + threadIdx.x;
        if (col < s.b) {
            const bool on = s.xstamp[col] == iter;
            ahist[col] = on ? s.alpha[col] : 0.0;
            bhist[col] = on && s.active[col] ? s.betac[col] : 0.0;
        }
    }
    if (x) x += static_cast<size_t>(chunk) * ldx;
    // p_in: the previous direction when it is not in p (history mode, first
    // iteration: p_0 = r_0 lives in residual slot 0)
    const double* __restrict__ pi_ = (p_in ? p_in : p) + static_cast<size_t>(chunk) * ldp;
    p += static_cast<size_t>(chunk) * ldp;
    d += static_cast<size_t>(chunk) * ldd;
    const size_t npairs = static_cast<size_t>(rows) * C / VEC;
    const size_t stride = static_cast<size_t>(nb) * kThreads;
    const size_t t0 = static_cast<size_t>(local) * kThreads + threadIdx.x;
    const int c0 = static_cast<int>((t0 * VEC) % C);
    double a[VEC], bc[VEC];
    bool ox[VEC], op[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
        const int col = chunk * C + c0 + q;
        ox[q] = col < s.b && s.xstamp[col] == iter;
        op[q] = ox[q] && s.active[col];
        a[q] = ox[q] ? s.alpha[col] : 0.0;
        bc[q] = op[q] ? s.betac[col] : 0.0;
    }
    // every column of the chunk stopped in this iteration's update (the last
    // iteration): p is dead, so only x += a*p runs (3 block passes, not 5)
    if (s.chunk_active && !s.chunk_active[chunk]) {
        if (!x) return;  // history mode: nothing left to do for this chunk
        for (size_t pi = t0; pi < npairs; pi += stride) {
            double xv[VEC], pv[VEC];
            ld_plain<VEC>(x + pi * VEC, xv);
            ld_plain<VEC>(p + pi * VEC, pv);
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                if (ox[k]) xv[k] = __dadd_rn(xv[k], __dmul_rn(a[k], pv[k]));
            st_plain<VEC>(x + pi * VEC, xv);
        }
        return;
    }
    if (!x) {
        // history mode: p = d + betac*p only (3 block passes)
        for (size_t pi = t0; pi < npairs; pi += stride) {
            double pv[VEC], dv[VEC];
            ld_plain<VEC>(pi_ + pi * VEC, pv);
            ld_plain<VEC>(d + pi * VEC, dv);
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                if (op[k]) pv[k] = __dadd_rn(dv[k], __dmul_rn(bc[k], pv[k]));
            st_plain<VEC>(p + pi * VEC, pv);
        }
        return;
    }
    for (size_t pi = t0; pi < npairs; pi += stride) {
        double xv[VEC], pv[VEC], dv[VEC];
        ld_plain<VEC>(x + pi * VEC, xv);
        ld_plain<VEC>(p + pi * VEC, pv);
        ld_plain<VEC>(d + pi * VEC, dv);
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            if (ox[k]) xv[k] = __dadd_rn(xv[k], __dmul_rn(a[k], pv[k]));
            if (op[k]) pv[k] = __dadd_rn(dv[k], __dmul_rn(bc[k], pv[k]));
        }
        st_plain<VEC>(x + pi * VEC, xv);
        st_plain<VEC>(p + pi * VEC, pv);
    }
}

// ---- residual-history form of the solution update ---------------------------
// With p_0 = r_0 and p_{k+1} = r_{k+1} + beta_k p_k, the CG iterate is
//   x_K = x_0 + sum_{k<K} a_k p_k = x_0 + sum_{i<K} c_i r_i,
//   c_{K-1} = a_{K-1},  c_i = a_i + beta_i c_{i+1},
// so while the residuals r_0..r_{H-1} are kept in their own slots the loop
// never touches x (saving its read + write every iteration), and x is formed
// once -- in the output gather, or by a fold when a solve outgrows the slots.
struct CgHistory {
    const double* slots = nullptr;  // [H] blocks of the chunked layout, slot stride `slot`
    size_t slot = 0;                // elements between slots
    const double* coef = nullptr;   // [H][bpad] c_i per column
    const int32_t* kcol = nullptr;  // [bpad] residuals used per column
    const double* x0 = nullptr;     // start block, or nullptr (x_0 = 0)
    int bpad = 0;
};

constexpr int kMaxHist = 16;  // residual-history slots (cg.cu caps H at this)

// element e (chunked offset) of column col (a fully unrolled, predicated
// variant measured 57% slower in the output gather)
__device__ __forceinline__ double hist_value(const CgHistory& h, size_t e, int col) {
    double v = h.x0 ? h.x0[e] : 0.0;
    const int kc = h.kcol[col];
    KZ_DCHECK(kc >= 0 && kc <= kMaxHist);
    for (int i = 0; i < kc; ++i) v = fma(h.coef[static_cast<size_t>(i) * h.bpad + col], h.slots[i * h.slot + e], v);
    return v;
}

// c_i per column from the recorded a_k, beta_k; kcol = min(iterations, limit)
static __global__ void cg_hist_coef_kernel(const double* __restrict__ ahist, const double* __restrict__ bhist,
                                           const int64_t* __restrict__ iters, int limit, int b, int bpad,
                                           double* __restrict__ coef, int32_t* __restrict__ kcol) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= bpad) return;
    const int k = col < b ? static_cast<int>(iters[col] < limit ? iters[col] : limit) : 0;
    kcol[col] = k;
    double c = 0.0;
    for (int i = k - 1; i >= 0; --i) {
        c = fma(bhist[static_cast<size_t>(i) * bpad + col], c, ahist[static_cast<size_t>(i) * bpad + col]);
        coef[static_cast<size_t>(i) * bpad + col] = c;
    }
}

// x = x_0 + sum_i c_i r_i over the whole chunked block (the fold); with
// p_out also the current direction p = sum_i d_i r_i (dcoef [H][bpad],
// cg_hist_dcoef_kernel), which the q-recurrence never materialises
template <int C>
__global__ void cg_hist_fold_kernel(double* __restrict__ x, CgHistory h, int64_t rows, int nchunks,
                                    double* __restrict__ p_out = nullptr, const double* __restrict__ dcoef = nullptr,
                                    int nd = 0) {
    const size_t total = static_cast<size_t>(nchunks) * rows * C;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(e % C);
        const int chunk = static_cast<int>(e / (static_cast<size_t>(rows) * C));
        const int col = chunk * C + c;
        x[e] = hist_value(h, e, col);
        if (p_out) {
            double v = 0.0;
            for (int i = 0; i < nd; ++i) v = fma(dcoef[static_cast<size_t>(i) * h.bpad + col], h.slots[i * h.slot + e], v);
            p_out[e] = v;
        }
    }
}

// d_i of the direction p_{m-1} = r_{m-1} + beta_{m-2} p_{m-2} = sum_{i<m} d_i r_i
// (d_{m-1} = 1, d_i = beta_i d_{i+1}; p_0 = r_0)
static __global__ void cg_hist_dcoef_kernel(const double* __restrict__ bhist, int m, int bpad,
                                            double* __restrict__ dcoef) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= bpad) return;
    double d = 1.0;
    dcoef[static_cast<size_t>(m - 1) * bpad + col] = d;
    for (int i = m - 2; i >= 0; --i) {
        d *= bhist[static_cast<size_t>(i) * bpad + col];
        dcoef[static_cast<size_t>(i) * bpad + col] = d;
    }
}

// rhs of query column j: beta * A[:, qpos[j]] (index.py:93-101), written into
// a zeroed block.  One CTA per column walks CSR row qpos[j] (A symmetric).
template <int C>
__global__ void scatter_rhs_kernel(double* __restrict__ r, int64_t ld,
                                   const int32_t* __restrict__ rowptr,
                                   const int32_t* __restrict__ colidx,
                                   const int64_t* __restrict__ qpos, int b, double beta) {
    const int j = blockIdx.x;
    if (j >= b) return;
    const int64_t q = qpos[j];
    const int beg = rowptr[q], end = rowptr[q + 1];
    for (int k = beg + threadIdx.x; k < end; k += blockDim.x)
        r[static_cast<size_t>(j / C) * ld + static_cast<size_t>(colidx[k]) * C + (j % C)] = beta;
}

// ||b||^2 of the rhs columns scatter_rhs_kernel wrote, in closed form: b has
// deg(q_j) entries equal to beta (binary operator), so ||b||^2 = beta^2 deg(q_j)
// -- the norm solver.py:71-72 takes of the same vector, without a pass over the
// block -- followed by the init finalize for r == b.  One CTA per chunk.
template <int C>
__global__ void rhs_norm_init_kernel(SolveState s, const int32_t* __restrict__ rowptr,
                                     const int64_t* __restrict__ qpos, double beta) {
    const int chunk = blockIdx.x;
    const int col = chunk * C + threadIdx.x;
    double v = 0.0;
    if (threadIdx.x < C && col < s.b) {
        const int64_t q = qpos[col];
        v = __dmul_rn(__dmul_rn(beta, beta), static_cast<double>(rowptr[q + 1] - rowptr[q]));
    }
    finalize_chunk<C>(FIN_INIT_BR, s, nullptr, chunk, 0, v);
}

// column-major [b][rows] -> chunked block (tile transpose through shared memory)
template <int C>
__global__ void load_colmajor_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                     int64_t rows, int64_t ld, int b, int nchunks) {
    constexpr int TR = 64;
    __shared__ double sm[TR * (C + 1)];
    const int64_t ntiles = (rows + TR - 1) / TR;
    for (int64_t t = blockIdx.x; t < ntiles * nchunks; t += gridDim.x) {
        const int chunk = static_cast<int>(t / ntiles);
        const int64_t r0 = (t - static_cast<int64_t>(chunk) * ntiles) * TR;
        for (int e = threadIdx.x; e < TR * C; e += blockDim.x) {
            const int c = e / TR, rr = e % TR;
            const int col = chunk * C + c;
            const int64_t row = r0 + rr;
            sm[rr * (C + 1) + c] = (col < b && row < rows) ? src[static_cast<size_t>(col) * rows + row] : 0.0;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < TR * C; e += blockDim.x) {
            const int rr = e / C, c = e % C;
            const int64_t row = r0 + rr;
            if (row < rows) dst[static_cast<size_t>(chunk) * ld + static_cast<size_t>(row) * C + c] = sm[rr * (C + 1) + c];
        }
        __syncthreads();
    }
}

// chunked block -> column-major scores [b][rows] with scatter through perm and
// the clamp at zero (solver.py:181-184, 223-225).
template <int C>
__global__ void store_colmajor_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                      int64_t rows, int64_t ld, int b, int nchunks,
                                      const int64_t* __restrict__ perm, int clamp, CgHistory hist = CgHistory()) {
    constexpr int TR = 64;
    __shared__ double sm[TR * (C + 1)];
    const int64_t ntiles = (rows + TR - 1) / TR;
    for (int64_t t = blockIdx.x; t < ntiles * nchunks; t += gridDim.x) {
        const int chunk = static_cast<int>(t / ntiles);
        const int64_t r0 = (t - static_cast<int64_t>(chunk) * ntiles) * TR;
        for (int e = threadIdx.x; e < TR * C; e += blockDim.x) {
            const int rr = e / C, c = e % C;
            const int64_t row = r0 + rr;
            const size_t e2 = static_cast<size_t>(chunk) * ld + static_cast<size_t>(row < rows ? row : 0) * C + c;
            sm[rr * (C + 1) + c] = row < rows ? (hist.kcol ? hist_value(hist, e2, chunk * C + c) : src[e2]) : 0.0;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < TR * C; e += blockDim.x) {
            const int c = e / TR, rr = e % TR;
            const int col = chunk * C + c;
            const int64_t row = r0 + rr;
            if (col < b && row < rows) {
                double v = sm[rr * (C + 1) + c];
                if (clamp) v = v > 0.0 ? v : 0.0;
                const int64_t dstrow = perm ? perm[row] : row;
                dst[static_cast<size_t>(col) * rows + dstrow] = v;
            }
        }
        __syncthreads();
    }
}

// Inverse of the output permutation: iperm[perm[i]] = i.
static __global__ void invert_perm_kernel(const int64_t* __restrict__ perm, int64_t* __restrict__ iperm, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        iperm[perm[i]] = i;
}

// chunked block (solve order) -> column-major scores [b][rows] in internal
// order, as a gather: output tile rows k..k+63 read their solve rows
// iperm[k] (one 8*C-byte line each) and write each column coalesced.  Same
// values as store_colmajor_kernel with perm, without the scattered stores.
template <int C>
__global__ void store_gather_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                    int64_t rows, int64_t ld, int b, int nchunks,
                                    const int64_t* __restrict__ iperm, int clamp, CgHistory hist = CgHistory()) {
    constexpr int TR = 64;
    __shared__ double sm[TR * (C + 1)];
    const int64_t ntiles = (rows + TR - 1) / TR;
    for (int64_t t = blockIdx.x; t < ntiles * nchunks; t += gridDim.x) {
        const int chunk = static_cast<int>(t / ntiles);
        const int64_t r0 = (t - static_cast<int64_t>(chunk) * ntiles) * TR;
        for (int e = threadIdx.x; e < TR * C; e += blockDim.x) {
            const int rr = e / C, c = e % C;
            const int64_t row = r0 + rr;
            KZ_DCHECK(row >= rows || (iperm[row] >= 0 && iperm[row] < rows));
            const size_t e2 = static_cast<size_t>(chunk) * ld + static_cast<size_t>(row < rows ? iperm[row] : 0) * C + c;
            sm[rr * (C + 1) + c] = row < rows ? (hist.kcol ? hist_value(hist, e2, chunk * C + c) : src[e2]) : 0.0;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < TR * C; e += blockDim.x) {
            const int c = e / TR, rr = e % TR;
            const int col = chunk * C + c;
            const int64_t row = r0 + rr;
            if (col < b && row < rows) {
                double v = sm[rr * (C + 1) + c];
                if (clamp) v = v > 0.0 ? v : 0.0;
                dst[static_cast<size_t>(col) * rows + row] = v;
            }
        }
        __syncthreads();
    }
}

template <int C>
__global__ void broadcast_kernel(double* __restrict__ dst, const double* __restrict__ v,
                                 int64_t rows, int64_t ld, int b, int nchunks) {
    const size_t total = static_cast<size_t>(nchunks) * rows * C;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(e % C);
        const size_t rowc = e / C;
        const int chunk = static_cast<int>(rowc / rows);
        const int64_t row = static_cast<int64_t>(rowc - static_cast<size_t>(chunk) * rows);
        dst[static_cast<size_t>(chunk) * ld + static_cast<size_t>(row) * C + c] = (chunk * C + c < b) ? v[row] : 0.0;
    }
}

// CTAs per chunk for the streaming kernels
inline int stream_ctas_per_chunk(int64_t rows, int C, int nchunks) {
    const int vec = C >= 2 ? 2 : 1;
    const int64_t pairs = rows * C / vec;
    int64_t nb = (pairs + kThreads * 4 - 1) / (kThreads * 4);
    const int64_t cap = std::max<int64_t>(1, (2 * max_ctas_per_chunk() + nchunks - 1) / nchunks);
    nb = std::max<int64_t>(1, std::min<int64_t>(nb, cap));
    return static_cast<int>(nb);
}

#define KZ_DISPATCH_C(C, ...)                                 \
    switch (C) {                                              \
        case 1: { constexpr int CC = 1; __VA_ARGS__; } break;  \
        case 2: { constexpr int CC = 2; __VA_ARGS__; } break;  \
        case 4: { constexpr int CC = 4; __VA_ARGS__; } break;  \
        case 8: { constexpr int CC = 8; __VA_ARGS__; } break;  \
        case 16: { constexpr int CC = 16; __VA_ARGS__; } break; \
        case 32: { constexpr int CC = 32; __VA_ARGS__; } break; \
        case 64: { constexpr int CC = 64; __VA_ARGS__; } break; \
        default: return fail(KZ_EARG, "unsupported chunk width"); \
    }

}  // namespace kz
