// lrc.cu -- LRC-Katz: batched Schur-complement PCG with the low-rank
// corrected preconditioner (the reference's `query`, solver.py:161-207).
//
// Under the partition order M = I - beta*A = [[M11, M12], [M12', M22]]
// (partition.py:277-297).  For b query columns at once:
//   rhs  = beta * A[:, q]                      (index.py:93-101, exact column)
//   f    = g2 - M12' M11^-1 g1 = g2 + beta*A21 (M11^-1 g1)       (solver.py:104-110)
//   tol_eff = tol*||rhs||/||f||                (solver.py:176)
//   PCG on S x = f, S v = M22 v - M12' M11^-1 M12 v             (solver.py:113-158)
//       = (v - beta*A22 v) + beta*A21 M11^-1 (-beta*A12 v)
//   preconditioner z = L^-T (I + U D U') L^-1 r, D = 1/(1-sigma) - 1
//       (factor.py:322-337: dc.solve(r) + L^-T U D U' L^-1 r, two dense
//        triangular products instead of four solves: L^-1 is formed once)
//   k1 = M11^-1 (g1 - M12 k2) = M11^-1 (g1 + beta*A12 k2)        (solver.py:178)
//   residual ||rhs - M k|| on the whole system, scatter, clamp    (solver.py:180-184)
// Each column keeps its own PCG scalars and stops on its own (masking).
//
// Operators: A12 (n1 x n2), A21 (n2 x n1), A22 (n2 x n2) and the full A are
// binary K1 operators; M11^-1 is the block-diagonal inverse of the interior
// parts as a weighted K1 operator (factor.py:89-106 without the per-part
// Python loop); L^-1, (L^-1)^T, U and (U D)^T are dense row-major K3/K6
// operands.  All device memory of the handle is borrowed from the caller.
#include <algorithm>
#include <cstring>
#include <cmath>
#include <vector>

#include "dense.cuh"
#include "driver.cuh"

using namespace kz;

struct kz_lrc {
    int64_t n = 0, n1 = 0, n2 = 0, ell = 0;
    double beta = 0.0;
    const kz_graph* full = nullptr;
    const kz_graph* a12 = nullptr;
    const kz_graph* a21 = nullptr;
    const kz_graph* a22 = nullptr;
    const kz_graph* minv = nullptr;
    const double* linv = nullptr;   // n2 x ld2 row-major, lower triangular
    const double* linvT = nullptr;  // n2 x ld2 row-major, (L^-1)^T
    const double* u = nullptr;      // n2 x ldl row-major
    const double* udT = nullptr;    // ell x ld2 row-major, (U diag(d))^T
    int64_t ld2 = 0, ldl = 0;       // leading dimensions, rounded up to even (zero padded)
    // every sigma < 1: the preconditioner exists (factor.py:329-330); only
    // the calls that apply it (query, lrc_pcg, PRECOND) raise otherwise
    bool spectrum_ok = true;
    uint64_t uid = 0;  // process-unique id (keys cached solve graphs)
};

namespace {

struct LrcWork {
    int C, nch, bpad, nb;
    double *rhs, *kk;        // [nch][n][C]
    double *t1, *w1;         // [nch][n1][C]
    double *r, *p, *q, *z, *t2, *xs;  // [nch][n2][C]
    double* cl;              // [nch][ell][C]
    SpmmDims dims;
    SpmmScratch sp;
    RedScratch red;
    DenseScratch ds;
    SolveState st;
    double *rhs2, *resid2;
    int64_t* qpos;
    int64_t* iperm;  // inverse output permutation (gather-based store)
};

int64_t rows_or_one(int64_t r) { return r > 0 ? r : 1; }

void carve_lrc(Carver& cv, const kz_lrc* h, int b, int C, LrcWork& w) {
    w.C = C;
    w.nch = (b + C - 1) / C;
    w.bpad = w.nch * C;
    const int64_t n = h->n, n1 = rows_or_one(h->n1), n2 = rows_or_one(h->n2), ell = rows_or_one(h->ell);
    w.nb = stream_ctas_per_chunk(std::max<int64_t>(n, 1), C, w.nch);
    const size_t bp = static_cast<size_t>(w.bpad);
    w.rhs = cv.take<double>(bp * n);
    w.kk = cv.take<double>(bp * n);
    w.t1 = cv.take<double>(bp * n1);
    w.w1 = cv.take<double>(bp * n1);
    w.r = cv.take<double>(bp * n2);
    w.p = cv.take<double>(bp * n2);
    w.q = cv.take<double>(bp * n2);
    w.z = cv.take<double>(bp * n2);
    w.t2 = cv.take<double>(bp * n2);
    w.xs = cv.take<double>(bp * n2);
    w.cl = cv.take<double>(bp * ell);
    w.dims = SpmmDims();
    w.dims.add(h->full);
    w.dims.add(h->a12);
    w.dims.add(h->a21);
    w.dims.add(h->a22);
    w.dims.add(h->minv);
    carve_spmm_scratch(cv, w.dims, w.nch, C, w.sp);
    w.red.nb = w.nb;
    w.red.part = cv.take<double>(static_cast<size_t>(w.nch) * w.nb * C);
    w.red.cnt = cv.take<int32_t>(w.nch);
    const int NC = std::min(kDenseMaxCols, w.bpad);
    size_t dp = 0;
    dp = std::max(dp, dense_part_doubles(n2, n2, NC));
    dp = std::max(dp, dense_part_doubles(ell, n2, NC));
    dp = std::max(dp, dense_part_doubles(n2, ell, NC));
    w.ds.part = cv.take<double>(dp + 1);
    w.ds.part_cap = dp;
    w.ds.cnt_cap = (std::max(n2, ell) + kDmmaRows - 1) / kDmmaRows + 1;
    w.ds.cnt = cv.take<int32_t>(w.ds.cnt_cap);
    SolveState& s = w.st;
    s.rs = cv.take<double>(w.bpad);
    s.alpha = cv.take<double>(w.bpad);
    s.betac = cv.take<double>(w.bpad);
    s.thresh = cv.take<double>(w.bpad);
    s.rnorm = cv.take<double>(w.bpad);
    s.bnorm2 = cv.take<double>(w.bpad);
    s.rr = cv.take<double>(w.bpad);
    w.rhs2 = cv.take<double>(w.bpad);
    w.resid2 = cv.take<double>(w.bpad);
    s.iters = cv.take<int64_t>(w.bpad);
    s.active = cv.take<int32_t>(w.bpad);
    s.xstamp = cv.take<int32_t>(w.bpad);
    s.status = cv.take<int32_t>(w.bpad);
    s.converged = cv.take<int32_t>(w.bpad);
    s.chunk_active = cv.take<int32_t>(w.nch);
    s.chunk_xstamp = cv.take<int32_t>(w.nch);
    s.n_active = cv.take<int32_t>(1);
    s.err = cv.take<int32_t>(1);
    s.iter_dev = cv.take<int32_t>(1);
    w.qpos = cv.take<int64_t>(w.bpad);
    w.iperm = cv.take<int64_t>(n);
}

// LRC init finalize (solver.py:171-177 + 127-133): thresh = tol_eff*||f||
__global__ void lrc_init_finalize_kernel(SolveState s, const double* rhs2, double tol) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= s.bpad) return;
    if (col >= s.b) {
        s.active[col] = 0;
        return;
    }
    const double fn = sqrt(s.bnorm2[col]);
    const double tol_eff = fn > 0.0 ? tol * sqrt(rhs2[col]) / fn : tol;
    s.thresh[col] = tol_eff * fn;
    const double rn = sqrt(s.rr[col]);
    s.rnorm[col] = rn;
    s.iters[col] = 0;
    const bool act = rn > s.thresh[col];
    s.active[col] = act;
    s.converged[col] = !act;
    if (act) atomicAdd(s.n_active, 1);
}

__global__ void chunk_flags_kernel(SolveState s) {
    const int c = threadIdx.x + blockIdx.x * blockDim.x;
    if (c >= s.nchunks) return;
    int any = 0;
    for (int j = 0; j < s.C; ++j) any |= s.active[c * s.C + j];
    s.chunk_active[c] = any;
}

template <int C>
__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, double a,
                            int64_t rows, int64_t ldy, int64_t ldx, int nch) {
    const size_t per = static_cast<size_t>(rows) * C;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < per * nch;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t ch = e / per, off = e - ch * per;
        y[ch * ldy + off] = __dadd_rn(y[ch * ldy + off], __dmul_rn(a, x[ch * ldx + off]));
    }
}

template <int C>
__global__ void copy_blk_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t rows,
                                int64_t ldy, int64_t ldx, int nch) {
    const size_t per = static_cast<size_t>(rows) * C;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < per * nch;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t ch = e / per, off = e - ch * per;
        y[ch * ldy + off] = x[ch * ldx + off];
    }
}

struct LrcCtx {
    const kz_lrc* h;
    LrcWork* w;
    cudaStream_t st;
    int C, nch;
    unsigned egrid(int64_t rows) const {
        return static_cast<unsigned>(std::min<int64_t>(2 * max_ctas_per_chunk(), (rows * C * nch + 255) / 256 + 1));
    }

    int spmm(const kz_graph* g, const double* Xg, int64_t ldxg, const double* Xs, int64_t ldxs,
             const double* Z, int64_t ldz, double* Y, int64_t ldy, double s0, double s1, double s2,
             const double* D, int64_t ldd, bool dot, const DotHook* hook, const int32_t* chunk_active) {
        SpmmArgs a = make_spmm_args(g, w->sp);
        a.Xg = Xg;
        a.ldxg = ldxg;
        a.Xs = Xs;
        a.ldxs = ldxs;
        a.Z = Z;
        a.ldz = ldz;
        a.Y = Y;
        a.ldy = ldy;
        a.D = D;
        a.ldd = ldd;
        a.s0 = s0;
        a.s1 = Xs ? s1 : 0.0;
        a.s2 = s2;
        a.want_dot = dot ? 1 : 0;
        a.chunk_active = chunk_active;
        if (hook) a.hook = *hook;
        return launch_spmm(g, C, nch, a, st);
    }

    // q = S p (+ dots p.q through the hook)
    int schur(const double* p, int64_t ldp, double* q, const DotHook* hook, const int32_t* chunk_active) {
        const int64_t n1 = h->n1, n2 = h->n2;
        const int64_t l1 = n1 * C, l2 = n2 * C;
        const bool dot = hook != nullptr;
        if (n1 > 0) {
            int rc;
            if ((rc = spmm(h->a12, p, ldp, nullptr, 0, nullptr, 0, w->t1, l1, 0.0, 0.0, -h->beta, nullptr, 0,
                           false, nullptr, chunk_active)))
                return rc;
            if ((rc = spmm(h->minv, w->t1, l1, nullptr, 0, nullptr, 0, w->w1, l1, 0.0, 0.0, 1.0, nullptr, 0,
                           false, nullptr, chunk_active)))
                return rc;
            if ((rc = spmm(h->a22, p, ldp, p, ldp, nullptr, 0, q, l2, 0.0, 1.0, -h->beta, nullptr, 0, false,
                           nullptr, chunk_active)))
                return rc;
            return spmm(h->a21, w->w1, l1, nullptr, 0, q, l2, q, l2, 1.0, 0.0, h->beta, p, ldp, dot, hook,
                        chunk_active);
        }
        return spmm(h->a22, p, ldp, p, ldp, nullptr, 0, q, l2, 0.0, 1.0, -h->beta, p, ldp, dot, hook,
                    chunk_active);
    }

    // z = L^-T (I + U D U') L^-1 r
    // chunk_active (optional): skip column groups whose columns have all stopped
    int precond(const double* r, int64_t ldr, double* z, int64_t ldz, const int32_t* chunk_active = nullptr) {
        const int64_t n2 = h->n2, ell = h->ell;
        int rc;
        if ((rc = launch_dense(h->linvT, h->ld2, n2, n2, 2, r, ldr, w->t2, n2 * C, 1.0, 0.0, C, nch, w->ds, st, chunk_active)))
            return rc;
        if (ell > 0) {
            if ((rc = launch_dense(h->u, h->ldl, ell, n2, 0, w->t2, n2 * C, w->cl, ell * C, 1.0, 0.0, C, nch, w->ds,
                                   st, chunk_active)))
                return rc;
            if ((rc = launch_dense(h->udT, h->ld2, n2, ell, 0, w->cl, ell * C, w->t2, n2 * C, 1.0, 1.0, C, nch,
                                   w->ds, st, chunk_active)))
                return rc;
        }
        return launch_dense(h->linv, h->ld2, n2, n2, 1, w->t2, n2 * C, z, ldz, 1.0, 0.0, C, nch, w->ds, st, chunk_active);
    }

    int coldot(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows, int mode,
               double* out, int iter) {
        const unsigned grid = static_cast<unsigned>(nch) * w->nb;
        KZ_DISPATCH_C(C, coldot_kernel<CC><<<grid, kThreads, 0, st>>>(X, Y, rows, ldx, ldy, w->red, mode,
                                                                        w->st, out, iter);
                      note_launch());
        KZ_LAUNCH_CHECK();
        return KZ_OK;
    }
};

}  // namespace

extern "C" int kz_lrc_create(const kz_lrc_desc* d, kz_lrc** out) {
    clear_error();
    if (!d || !out) return fail(KZ_EARG, "NULL argument");
    *out = nullptr;
    if (d->n < 1 || d->n1 < 0 || d->n2 < 0 || d->n1 + d->n2 != d->n || d->ell < 0 || d->ell > d->n2)
        return fail(KZ_EARG, "inconsistent LRC sizes");
    if (!d->full || (d->n1 > 0 && d->n2 > 0 && (!d->a12 || !d->a21)) || (d->n1 > 0 && !d->minv) ||
        (d->n2 > 0 && (!d->a22 || !d->linv || !d->linvT)) || (d->ell > 0 && (!d->u || !d->udT || !d->sigma)))
        return fail(KZ_EARG, "missing LRC operand");
    bool spectrum_ok = true;
    for (int64_t i = 0; i < d->ell; ++i)
        if (!(d->sigma[i] < 1.0)) spectrum_ok = false;
    auto* h = new kz_lrc();
    h->spectrum_ok = spectrum_ok;
    h->uid = next_uid();
    h->n = d->n;
    h->n1 = d->n1;
    h->n2 = d->n2;
    h->ell = d->ell;
    h->beta = d->beta;
    h->full = d->full;
    h->a12 = d->a12;
    h->a21 = d->a21;
    h->a22 = d->a22;
    h->minv = d->minv;
    h->linv = d->linv;
    h->linvT = d->linvT;
    h->u = d->u;
    h->udT = d->udT;
    h->ld2 = d->n2 + (d->n2 & 1);
    h->ldl = d->ell + (d->ell & 1);
    *out = h;
    return KZ_OK;
}

extern "C" int kz_lrc_destroy(kz_lrc* h) {
    delete h;
    return KZ_OK;
}

static int lrc_chunk(const kz_lrc_args* a) { return a && a->chunk > 0 ? a->chunk : default_chunk(a ? a->b : 1); }

extern "C" size_t kz_lrc_workspace_bytes(const kz_lrc* h, int32_t b, int32_t chunk) {
    if (!h || b < 1) return 0;
    const int C = chunk > 0 ? chunk : default_chunk(b);
    if (!chunk_ok(C)) return 0;
    Carver cv(nullptr, 0);
    LrcWork w;
    carve_lrc(cv, h, b, C, w);
    return cv.off + 256;
}

extern "C" int kz_lrc_batch(const kz_lrc* h, const kz_lrc_args* a, void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    if (!h || !a || a->b < 1) return fail(KZ_EARG, "bad LRC arguments");
    const int mode_pcg = a->f != nullptr;  // lrc_pcg on a given Schur rhs
    if (!mode_pcg && !a->qpos) return fail(KZ_EARG, "need qpos or f");
    if (!a->out || !a->reports) return fail(KZ_EARG, "NULL outputs");
    if (mode_pcg && h->n2 == 0) return fail(KZ_EARG, "empty separator");
    if (!h->spectrum_ok) return fail(KZ_ESPECTRUM, "correction eigenvalue at or above 1");
    const int b = a->b;
    const int C = lrc_chunk(a);
    // the PCG dots are fused into K1, whose reduction covers chunks of at most 32 columns
    if (!chunk_ok(C) || C > 32) return fail(KZ_EARG, "bad chunk width");
    if (!ws || ws_bytes < kz_lrc_workspace_bytes(h, b, C)) return fail(KZ_EARG, "workspace too small");
    const int64_t n = h->n, n1 = h->n1, n2 = h->n2;
    if (!mode_pcg)
        for (int j = 0; j < b; ++j)
            if (a->qpos[j] < 0 || a->qpos[j] >= n) return fail(KZ_EARG, "query position out of range");
    StreamScope scope(static_cast<cudaStream_t>(stream));
    cudaStream_t st = scope.st;
    Carver cv(ws, ws_bytes);
    LrcWork w;
    carve_lrc(cv, h, b, C, w);
    SolveState& s = w.st;
    s.b = b;
    s.bpad = w.bpad;
    s.C = C;
    s.nchunks = w.nch;
    s.rows = n2;
    s.tol = a->tol;
    s.max_iter = a->max_iter > 0 ? a->max_iter : 10 * std::max<int64_t>(n2, 1);
    const int nch = w.nch;
    LrcCtx cx{h, &w, st, C, nch};
    const int64_t ln = n * C, l1 = n1 * C, l2 = n2 * C;
    double* xk = mode_pcg ? w.xs : w.kk + l1;  // the Schur unknown (k2)
    const int64_t ldxk = mode_pcg ? l2 : ln;

    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (a->device_ms) {
        KZ_CUDA(cudaEventCreate(&e0));
        KZ_CUDA(cudaEventCreate(&e1));
        KZ_CUDA(cudaEventRecord(e0, st));
    }
    KZ_CUDA(zero_span(s.rs, w.qpos, st));
    KZ_CUDA(cudaMemsetAsync(w.red.cnt, 0, sizeof(int32_t) * nch, st));
    KZ_CUDA(cudaMemsetAsync(w.ds.cnt, 0, sizeof(int32_t) * w.ds.cnt_cap, st));
    if (int rc = zero_spmm_counters(w.dims, nch, w.sp, st)) return rc;
    const unsigned tg = static_cast<unsigned>(std::min<int64_t>(2 * max_ctas_per_chunk(), ((n + 63) / 64) * nch));
    int rc = KZ_OK;
    long long graph_per_iter = 0;  // kernels per iteration of a graph-run loop (launch count)

    if (!mode_pcg) {
        KZ_CUDA(cudaMemsetAsync(w.rhs, 0, sizeof(double) * w.bpad * n, st));
        KZ_CUDA(cudaMemsetAsync(w.kk, 0, sizeof(double) * w.bpad * n, st));
        KZ_CUDA(cudaMemcpyAsync(w.qpos, a->qpos, sizeof(int64_t) * b, cudaMemcpyHostToDevice, st));
        KZ_DISPATCH_C(C, scatter_rhs_kernel<CC><<<b, kThreads, 0, st>>>(w.rhs, ln, h->full->rowptr, h->full->colidx,
                                                                          w.qpos, b, h->beta);
                      note_launch());
        KZ_LAUNCH_CHECK();
        if ((rc = cx.coldot(w.rhs, ln, w.rhs, ln, n, FIN_WRITE, w.rhs2, 0))) return rc;
    } else {
        KZ_CUDA(cudaMemsetAsync(w.xs, 0, sizeof(double) * w.bpad * n2, st));
    }

    if (n2 > 0) {
        // r = f
        if (mode_pcg) {
            KZ_DISPATCH_C(C, load_colmajor_kernel<CC><<<tg, kThreads, 0, st>>>(w.r, a->f, n2, l2, b, nch);
                          note_launch());
            KZ_LAUNCH_CHECK();
        } else if (n1 > 0) {
            if ((rc = cx.spmm(h->minv, w.rhs, ln, nullptr, 0, nullptr, 0, w.w1, l1, 0.0, 0.0, 1.0, nullptr, 0,
                              false, nullptr, nullptr)))
                return rc;
            if ((rc = cx.spmm(h->a21, w.w1, l1, nullptr, 0, w.rhs + l1, ln, w.r, l2, 1.0, 0.0, h->beta, nullptr,
                              0, false, nullptr, nullptr)))
                return rc;
        } else {
            KZ_DISPATCH_C(C, copy_blk_kernel<CC><<<cx.egrid(n2), 256, 0, st>>>(w.r, w.rhs, n2, l2, ln, nch);
                          note_launch());
            KZ_LAUNCH_CHECK();
        }
        // ||f||^2 -> bnorm2
        if ((rc = cx.coldot(w.r, l2, w.r, l2, n2, FIN_WRITE, s.bnorm2, 0))) return rc;
        if (a->x0) {
            KZ_DISPATCH_C(C, broadcast_kernel<CC><<<tg, kThreads, 0, st>>>(xk, a->x0, n2, ldxk, b, nch);
                          note_launch());
            KZ_LAUNCH_CHECK();
            if ((rc = cx.schur(xk, ldxk, w.q, nullptr, nullptr))) return rc;
            KZ_DISPATCH_C(C, axpy_kernel<CC><<<cx.egrid(n2), 256, 0, st>>>(w.r, w.q, -1.0, n2, l2, l2, nch);
                          note_launch());
            KZ_LAUNCH_CHECK();
        }
        if ((rc = cx.coldot(w.r, l2, w.r, l2, n2, FIN_WRITE, s.rr, 0))) return rc;
        if (mode_pcg) {
            // plain lrc_pcg: thresh = tol*||f||; reuse the LRC finalize with rhs2 := f2 and tol_eff = tol
            KZ_CUDA(cudaMemcpyAsync(w.rhs2, s.bnorm2, sizeof(double) * w.bpad, cudaMemcpyDeviceToDevice, st));
        }
        lrc_init_finalize_kernel<<<(w.bpad + 127) / 128, 128, 0, st>>>(s, w.rhs2, a->tol);
        note_launch();
        chunk_flags_kernel<<<(nch + 127) / 128, 128, 0, st>>>(s);
        note_launch();
        KZ_LAUNCH_CHECK();
        // z = P r, rz, p = z
        if ((rc = cx.precond(w.r, l2, w.z, l2))) return rc;
        if ((rc = cx.coldot(w.r, l2, w.z, l2, n2, FIN_PCG_INIT_RZ, nullptr, 0))) return rc;
        KZ_CUDA(cudaMemcpyAsync(w.p, w.z, sizeof(double) * w.bpad * n2, cudaMemcpyDeviceToDevice, st));

        const double work = static_cast<double>(n2) * n2 * 0.5 + static_cast<double>(h->full->nnz);
        const int lag = work * w.bpad > 2e8 ? 1 : 3;
        auto launch_iter = [&](int k) -> int {
            DotHook hk;
            hk.mode = 1;
            hk.b = b;
            hk.rs = s.rs;
            hk.alpha = s.alpha;
            hk.active = s.active;
            hk.xstamp = s.xstamp;
            hk.chunk_xstamp = s.chunk_xstamp;
            hk.status = s.status;
            hk.err = s.err;
            hk.n_active = s.n_active;
            hk.iter = k;
            hk.iter_dev = s.iter_dev;
            int r2;
            if ((r2 = cx.schur(w.p, l2, w.q, &hk, s.chunk_active))) return r2;
            const unsigned sg = static_cast<unsigned>(nch) * w.nb;
            KZ_DISPATCH_C(C, cg_update_kernel<CC><<<sg, kThreads, 0, st>>>(w.r, w.q, n2, l2, l2, w.red,
                                                                            FIN_PCG_RR, s, k);
                          note_launch());
            KZ_LAUNCH_CHECK();
            if ((r2 = cx.precond(w.r, l2, w.z, l2, s.chunk_active))) return r2;
            if ((r2 = cx.coldot(w.r, l2, w.z, l2, n2, FIN_PCG_RZ, nullptr, k))) return r2;
            KZ_DISPATCH_C(C, cg_pupdate_kernel<CC><<<sg, kThreads, 0, st>>>(xk, w.p, w.z, n2, ldxk, l2, l2, w.nb,
                                                                             s, k);
                          note_launch());
            KZ_LAUNCH_CHECK();
            return KZ_OK;
        };
        int64_t ran = 0;
        // launch-bound small solves: the whole PCG loop is one cached graph
        // with a device-side WHILE condition (driver.cuh)
        if (use_graph_loop(work * w.bpad, kGraphWorkLrc)) {
            GraphKey key;
            key.v[0] = h->uid;
            key.v[1] = reinterpret_cast<uint64_t>(ws);
            key.v[2] = ws_bytes;
            key.v[3] = static_cast<uint64_t>(b) | (static_cast<uint64_t>(C) << 32);
            key.v[4] = static_cast<uint64_t>(mode_pcg) | (static_cast<uint64_t>(a->x0 != nullptr) << 1);
            std::memcpy(&key.v[5], &a->tol, sizeof(double));
            key.v[6] = static_cast<uint64_t>(s.max_iter);
            if ((rc = run_iterations_graph(s, st, launch_iter, key, &graph_per_iter))) return rc;
        } else if ((rc = run_iterations(s, s.max_iter, lag, st, launch_iter, &ran))) {
            return rc;
        }
    }

    if (!mode_pcg) {
        // back-substitution k1 = M11^-1 (g1 + beta*A12 k2), then the true residual
        if (n1 > 0) {
            if (n2 > 0) {
                if ((rc = cx.spmm(h->a12, w.kk + l1, ln, nullptr, 0, w.rhs, ln, w.t1, l1, 1.0, 0.0, h->beta,
                                  nullptr, 0, false, nullptr, nullptr)))
                    return rc;
                if ((rc = cx.spmm(h->minv, w.t1, l1, nullptr, 0, nullptr, 0, w.kk, ln, 0.0, 0.0, 1.0, nullptr, 0,
                                  false, nullptr, nullptr)))
                    return rc;
            } else {
                if ((rc = cx.spmm(h->minv, w.rhs, ln, nullptr, 0, nullptr, 0, w.kk, ln, 0.0, 0.0, 1.0, nullptr, 0,
                                  false, nullptr, nullptr)))
                    return rc;
            }
        }
        // rhs - M k = rhs + (-(k - beta*A k))   (solver.py:180)
        if ((rc = cx.spmm(h->full, w.kk, ln, w.kk, ln, w.rhs, ln, w.rhs, ln, 1.0, -1.0, h->beta, nullptr, 0, false,
                          nullptr, nullptr)))
            return rc;
        if ((rc = cx.coldot(w.rhs, ln, w.rhs, ln, n, FIN_WRITE, w.resid2, 0))) return rc;
        if (a->perm) {
            invert_perm_kernel<<<static_cast<unsigned>(std::min<int64_t>(4 * max_ctas_per_chunk(), (n + 255) / 256)), 256, 0, st>>>(a->perm, w.iperm, n);
            note_launch();
            KZ_DISPATCH_C(C, store_gather_kernel<CC><<<tg, kThreads, 0, st>>>(a->out, w.kk, n, ln, b, nch, w.iperm,
                                                                              a->clamp);
                          note_launch());
        } else {
            KZ_DISPATCH_C(C, store_colmajor_kernel<CC><<<tg, kThreads, 0, st>>>(a->out, w.kk, n, ln, b, nch, nullptr,
                                                                                 a->clamp);
                          note_launch());
        }
    } else {
        KZ_DISPATCH_C(C, store_colmajor_kernel<CC><<<tg, kThreads, 0, st>>>(a->out, w.xs, n2, l2, b, nch, nullptr,
                                                                             0);
                      note_launch());
    }
    KZ_LAUNCH_CHECK();
    if (a->device_ms) KZ_CUDA(cudaEventRecord(e1, st));
    std::vector<int64_t> iters(b);
    std::vector<int32_t> conv(b), status(b);
    std::vector<double> rnorm(b), rhs2(b), resid2(b);
    KZ_CUDA(cudaMemcpyAsync(iters.data(), s.iters, sizeof(int64_t) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(conv.data(), s.converged, sizeof(int32_t) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(status.data(), s.status, sizeof(int32_t) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(rnorm.data(), s.rnorm, sizeof(double) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(rhs2.data(), w.rhs2, sizeof(double) * b, cudaMemcpyDeviceToHost, st));
    if (!mode_pcg)
        KZ_CUDA(cudaMemcpyAsync(resid2.data(), w.resid2, sizeof(double) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    if (a->device_ms) {
        KZ_CUDA(cudaEventElapsedTime(a->device_ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    if (graph_per_iter) {
        int64_t mx = 1;
        for (int j = 0; j < b; ++j) mx = std::max<int64_t>(mx, iters[j]);
        add_launches(graph_per_iter * mx);
    }
    bool notspd = false;
    for (int j = 0; j < b; ++j) {
        kz_report& r = a->reports[j];
        r.iterations = n2 > 0 ? iters[j] : 0;
        r.status = status[j];
        notspd = notspd || status[j] == KZ_ENOTSPD;
        if (mode_pcg) {
            r.final_residual_norm = rnorm[j];
            r.converged = conv[j];
            r.rhs_norm = std::sqrt(rhs2[j]);
        } else {
            const double rn = std::sqrt(resid2[j]), bn = std::sqrt(rhs2[j]);
            r.final_residual_norm = rn;
            r.converged = rn <= a->tol * bn ? 1 : 0;
            r.rhs_norm = bn;
        }
    }
    if (notspd) return fail(KZ_ENOTSPD, "Schur operator is not positive definite");
    return KZ_OK;
}

// Single applications for the API mirrors apply_schur / schur_rhs /
// apply_approx_schur_inverse: inputs and outputs column-major [b][rows].
extern "C" int kz_lrc_apply(const kz_lrc* h, int32_t op, int32_t b, const double* in1, const double* in2,
                            double* out, void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    if (!h || b < 1 || !in1 || !out) return fail(KZ_EARG, "bad LRC apply arguments");
    if (!ws || ws_bytes < kz_lrc_workspace_bytes(h, b, 1)) return fail(KZ_EARG, "workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver cv(ws, ws_bytes);
    LrcWork w;
    carve_lrc(cv, h, b, 1, w);
    LrcCtx cx{h, &w, st, 1, b};
    const int64_t n1 = h->n1, n2 = h->n2;
    if (int rc = zero_spmm_counters(w.dims, b, w.sp, st)) return rc;
    KZ_CUDA(cudaMemsetAsync(w.ds.cnt, 0, sizeof(int32_t) * w.ds.cnt_cap, st));
    if (n2 == 0) return fail(KZ_EARG, "empty separator");
    switch (op) {
        case KZ_LRC_SCHUR:
            return cx.schur(in1, n2, out, nullptr, nullptr);
        case KZ_LRC_PRECOND:
            if (!h->spectrum_ok) return fail(KZ_ESPECTRUM, "correction eigenvalue at or above 1");
            return cx.precond(in1, n2, out, n2);
        case KZ_LRC_SCHUR_RHS: {
            if (!in2) return fail(KZ_EARG, "schur_rhs needs g2");
            if (n1 == 0) {
                KZ_CUDA(cudaMemcpyAsync(out, in2, sizeof(double) * n2 * b, cudaMemcpyDeviceToDevice, st));
                return KZ_OK;
            }
            int rc;
            if ((rc = cx.spmm(h->minv, in1, n1, nullptr, 0, nullptr, 0, w.w1, n1, 0.0, 0.0, 1.0, nullptr, 0, false,
                              nullptr, nullptr)))
                return rc;
            return cx.spmm(h->a21, w.w1, n1, nullptr, 0, in2, n2, out, n2, 1.0, 0.0, h->beta, nullptr, 0, false,
                           nullptr, nullptr);
        }
        case KZ_LRC_CORRECTION: {
            // R v = L^-1 M12' M11^-1 M12 L^-T v with M12 = -beta*A12
            // (factor.py:196-202); the Lanczos operator of the index build.
            if (n1 == 0) {
                KZ_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * n2 * b, st));
                return KZ_OK;
            }
            const int64_t l1 = n1, l2 = n2;
            int rc;
            // launch_dense(A) applies A' (column-major view of the row-major
            // operand): the linv buffer gives L^-T, linvT gives L^-1
            if ((rc = launch_dense(h->linv, h->ld2, n2, n2, 1, in1, l2, w.t2, l2, 1.0, 0.0, 1, b, w.ds, st)))
                return rc;
            if ((rc = cx.spmm(h->a12, w.t2, l2, nullptr, 0, nullptr, 0, w.t1, l1, 0.0, 0.0, -h->beta, nullptr, 0,
                              false, nullptr, nullptr)))
                return rc;
            if ((rc = cx.spmm(h->minv, w.t1, l1, nullptr, 0, nullptr, 0, w.w1, l1, 0.0, 0.0, 1.0, nullptr, 0, false,
                              nullptr, nullptr)))
                return rc;
            if ((rc = cx.spmm(h->a21, w.w1, l1, nullptr, 0, nullptr, 0, w.q, l2, 0.0, 0.0, -h->beta, nullptr, 0,
                              false, nullptr, nullptr)))
                return rc;
            return launch_dense(h->linvT, h->ld2, n2, n2, 2, w.q, l2, out, l2, 1.0, 0.0, 1, b, w.ds, st);
        }
        default:
            return fail(KZ_EARG, "unknown LRC op");
    }
}

extern "C" int kz_lrc_info(const kz_lrc* h, int64_t* n, int64_t* n1, int64_t* n2, int64_t* ell) {
    if (!h) return fail(KZ_EARG, "NULL handle");
    if (n) *n = h->n;
    if (n1) *n1 = h->n1;
    if (n2) *n2 = h->n2;
    if (ell) *ell = h->ell;
    return KZ_OK;
}
