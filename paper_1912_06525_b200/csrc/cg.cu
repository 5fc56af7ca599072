// cg.cu -- K2: batched textbook CG for Katz queries (query_cg_baseline / cg).
//
// One call solves b query columns of (I - beta*A) x = beta*A e_q.  Each
// column runs the recurrence of cg() (solver.py:62-101) exactly -- the same
// scalar formulas, the same stop test ||r|| <= tol*||b||, the same
// non-positive-curvature error -- and is frozen (masked) once it stops, so
// its iteration count is its own.
//
// Residual-history form (the default whenever H >= 3 residual blocks fit):
// the direction p is never materialised.  With q_k = M p_k, M = I - beta A,
// p_k = r_k + b_{k-1} p_{k-1} gives the q-recurrence
//   q_k = M r_k + b_{k-1} q_{k-1},      p_k.q_k = r_k.q_k
// (the second by M-conjugacy of p_k and p_{k-1}; in exact arithmetic both are
// the reference's quantities, so a_k = rs_k / (p_k.q_k) and the stop tests
// are the reference's).  Per iteration two kernels run:
//   spmm   q = M r + b*q (in place, per-column b), dots r.q, a = rs / r.q
//   update r_{k+1} = r_k - a*q into its own slot, r.r, stop test, b = rs'/rs
// and x = x_0 + sum_i c_i r_i is formed once at the end from the kept
// residuals (CgHistory) -- 6 block passes per iteration instead of 8.  A
// solve that outgrows the H slots folds x and p from them once and continues
// with the direction form below.
//
// Direction form (small solves replayed as CUDA graphs, or H < 3):
//   spmm   q = p - beta*A p, column dots p.q, step length a = rs/pq
//   update r -= a*q, column dots r.r, stop test, beta_cg = rs_new/rs
//   pupd   x += a*p (deferred from solver.py:87), p = r + beta_cg*p
// Moving `x += a*p` into the p-update pass keeps every rounding identical to
// the reference order while saving one read+write of p and x per iteration.
// The host only polls a device counter of active columns, one iteration
// behind the GPU, so the device queue never drains.
// A solve from zero with query-position rhs (b = beta A e_q) runs its first
// iteration without the SpMM: p0 = b lives on N(q), so A p0 = beta A^2 e_q is
// beta times the integer 2-walk counts (walk2_count_kernel), p0.q0 is a sum
// over N(q) (cg_sparse_pq_kernel) and the update forms q0 from the counts.
// The recurrence and its stop tests are unchanged; only the roundings of
// q0's neighbour sums differ (beta*cnt instead of cnt repeated additions).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "cgsmall.cuh"
#include "driver.cuh"
#include "lowrank.cuh"

using namespace kz;

namespace {

struct CgWork {
    int C, nchunks, bpad, nb;
    int H = 0;             // residual-history slots (0: x updated every iteration)
    double *x, *r, *p, *q; // r = slot 0 of the H residual slots
    double *ahist = nullptr, *bhist = nullptr, *coef = nullptr, *dcoef = nullptr;  // [H][bpad]
    int32_t* kcol = nullptr;                                     // [bpad]
    SpmmScratch sp;
    RedScratch red;
    SolveState st;
    int64_t* qpos;
    int64_t* iperm;  // inverse output permutation (gather-based store)
    double* y;       // eigen start: [nch][ldr][C] Galerkin coefficients
    double* small_part;   // fused small loop (cgsmall.cuh): [2][SMs][bpad] CTA partials
    double* small_carry;  // ... and [SMs * 8 warps][bpad] split-row partials
    int32_t* small_stamp; // ... and [SMs * 8 warps][nchunks] carry stamps
    kz_report* dev_reports;  // fused small solve: the packed reports
};

void carve_cg(Carver& cv, const kz_graph* g, int b, CgWork& w, const kz_eigen* eig = nullptr) {
    w.C = default_chunk(b);
    w.nchunks = (b + w.C - 1) / w.C;
    w.bpad = w.nchunks * w.C;
    w.nb = stream_ctas_per_chunk(g->rows, w.C, w.nchunks);
    const size_t blk = static_cast<size_t>(w.bpad) * g->rows;
    // residual-history slots (see blockops.cuh CgHistory): up to
    // KZ_CG_HISTORY (default 16: cfg5 at tol 1e-10 needs 14) while the vector blocks stay under 64 GB
    {
        const char* e = std::getenv("KZ_CG_HISTORY");
        const int want = e ? std::atoi(e) : 16;
        const double blk_gb = static_cast<double>(blk) * 8.0 / 1e9;
        int h = static_cast<int>(std::min<double>(std::min(want, kMaxHist),
                                                  std::floor(64.0 / std::max(blk_gb, 1e-9)) - 3.0));
        w.H = h >= 3 ? h : 0;
    }
    w.x = cv.take<double>(blk);
    w.r = cv.take<double>(blk * static_cast<size_t>(std::max(1, w.H)));
    w.p = cv.take<double>(blk);
    w.q = cv.take<double>(blk);
    if (w.H) {
        w.ahist = cv.take<double>(static_cast<size_t>(w.H) * w.bpad);
        w.bhist = cv.take<double>(static_cast<size_t>(w.H) * w.bpad);
        w.coef = cv.take<double>(static_cast<size_t>(w.H) * w.bpad);
        w.dcoef = cv.take<double>(static_cast<size_t>(w.H) * w.bpad);
        w.kcol = cv.take<int32_t>(w.bpad);
    }
    carve_spmm_scratch(cv, g, w.nchunks, w.C, w.sp);
    w.red.nb = w.nb;
    w.red.part = cv.take<double>(static_cast<size_t>(w.nchunks) * w.nb * w.C);
    w.red.cnt = cv.take<int32_t>(w.nchunks);
    SolveState& s = w.st;
    // state block: everything zero-initialised by one memset (see kz_cg_batch)
    s.rs = cv.take<double>(w.bpad);
    s.alpha = cv.take<double>(w.bpad);
    s.betac = cv.take<double>(w.bpad);
    s.thresh = cv.take<double>(w.bpad);
    s.rnorm = cv.take<double>(w.bpad);
    s.bnorm2 = cv.take<double>(w.bpad);
    s.rr = cv.take<double>(w.bpad);
    s.iters = cv.take<int64_t>(w.bpad);
    s.active = cv.take<int32_t>(w.bpad);
    s.xstamp = cv.take<int32_t>(w.bpad);
    s.status = cv.take<int32_t>(w.bpad);
    s.converged = cv.take<int32_t>(w.bpad);
    s.chunk_active = cv.take<int32_t>(w.nchunks);
    s.chunk_xstamp = cv.take<int32_t>(w.nchunks);
    s.n_active = cv.take<int32_t>(1);
    s.err = cv.take<int32_t>(1);
    s.iter_dev = cv.take<int32_t>(1);
    w.qpos = cv.take<int64_t>(w.bpad);
    w.iperm = cv.take<int64_t>(g->rows);
    w.y = eig ? cv.take<double>(static_cast<size_t>(w.bpad) * eig->ldr) : nullptr;
    const size_t small_ctas = static_cast<size_t>(num_sms()) * kSmallCgCtasPerSm;
    w.small_part = cv.take<double>(2 * small_ctas * w.bpad);
    w.small_carry = cv.take<double>(small_ctas * kSmallCgWarps * w.bpad);
    w.small_stamp = cv.take<int32_t>(small_ctas * kSmallCgWarps * w.nchunks);
    w.dev_reports = cv.take<kz_report>(w.bpad);
}


}  // namespace

extern "C" size_t kz_cg_workspace_bytes(const kz_graph* g, int32_t b) {
    if (!g || b < 1) return 0;
    Carver cv(nullptr, 0);
    CgWork w;
    carve_cg(cv, g, b, w);
    return cv.off + 256;
}


// The batched CG of kz_cg_batch; with `eig` the columns start from the
// eigen-of-A Galerkin point (lowrank.cuh) instead of zero / x0.
static int cg_batch_impl(const kz_graph* g, const kz_cg_args* a, void* ws, size_t ws_bytes, void* stream,
                         const kz_eigen* eig) {
    if (!g || !a) return fail(KZ_EARG, "NULL argument");
    if (g->rows != g->cols) return fail(KZ_EARG, "CG needs a square operator");
    if (a->b < 1) return fail(KZ_EARG, "empty batch");
    if (!a->scores || !a->reports) return fail(KZ_EARG, "NULL outputs");
    if (!a->rhs && !a->qpos) return fail(KZ_EARG, "need qpos or rhs");
    if (eig && (a->rhs || a->x0 || !a->qpos)) return fail(KZ_EARG, "the eigen start needs query positions only");
    if (!ws || ws_bytes < (eig ? kz_eigen_workspace_bytes(eig, a->b) : kz_cg_workspace_bytes(g, a->b)))
        return fail(KZ_EARG, "workspace too small");
    const int b = a->b;
    const int64_t n = g->rows;
    if (a->qpos && !a->rhs)
        for (int j = 0; j < b; ++j)
            if (a->qpos[j] < 0 || a->qpos[j] >= n) return fail(KZ_EARG, "query position out of range");
    StreamScope scope(static_cast<cudaStream_t>(stream));
    cudaStream_t st = scope.st;

    Carver cv(ws, ws_bytes);
    CgWork w;
    carve_cg(cv, g, b, w, eig);
    SolveState& s = w.st;
    s.b = b;
    s.bpad = w.bpad;
    s.C = w.C;
    s.nchunks = w.nchunks;
    s.rows = n;
    s.tol = a->tol;
    s.max_iter = a->max_iter > 0 ? a->max_iter : 10 * n;
    const int C = w.C, nchunks = w.nchunks, nb = w.nb;

    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (a->device_ms) {
        KZ_CUDA(cudaEventCreate(&e0));
        KZ_CUDA(cudaEventCreate(&e1));
        KZ_CUDA(cudaEventRecord(e0, st));
    }
    const size_t blk_elems = static_cast<size_t>(w.bpad) * n;
    const size_t blk_bytes = sizeof(double) * blk_elems;
    const double work = static_cast<double>(g->nnz + n) * w.bpad;
    // small solves (blocks of at most kSmallCgElems doubles, <= 256 columns):
    // the whole loop is one cooperative kernel (cgsmall.cuh); KZ_CG_FUSED=0
    // turns it off
    int small_grid = 0;
    {
        const char* fe = std::getenv("KZ_CG_FUSED");
        if (!(fe && fe[0] == '0') && blk_elems <= kSmallCgElems && C <= 32) {
            KZ_DISPATCH_C(C, small_grid = small_cg_grid(n, g->nnz, CC, w.bpad,
                                                        reinterpret_cast<const void*>(cg_small_kernel<CC>)));
        }
    }
    if (small_grid > 0 && !eig && !a->rhs && !a->x0 && a->qpos) {
        // the whole query solve -- rhs, start state, iterations, output,
        // reports -- is one cooperative launch (plus the qpos upload and the
        // report download)
        KZ_CUDA(cudaMemcpyAsync(w.qpos, a->qpos, sizeof(int64_t) * b, cudaMemcpyHostToDevice, st));
        KZ_CUDA(cudaMemsetAsync(s.err, 0, sizeof(int32_t), st));
        SmallCgArgs sa{};
        sa.rows = static_cast<int32_t>(n);
        sa.nchunks = nchunks;
        sa.b = b;
        sa.bpad = w.bpad;
        sa.rowptr = g->rowptr;
        sa.colidx = g->colidx;
        sa.beta = a->beta;
        sa.x = w.x;
        sa.r = w.r;
        sa.p = w.p;
        sa.q = w.q;
        sa.part = w.small_part;
        sa.carry = w.small_carry;
        sa.stamp = w.small_stamp;
        sa.s = s;
        sa.init = 1;
        sa.qpos = w.qpos;
        sa.scores = a->scores;
        sa.perm = a->perm;
        sa.clamp = a->clamp;
        sa.reports = w.dev_reports;
        void* kargs[] = {&sa};
        KZ_DISPATCH_C(C, KZ_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(cg_small_kernel<CC>),
                                                            dim3(small_grid), dim3(kSmallCgThreads), kargs, 0, st)));
        note_launch();
        if (a->device_ms) KZ_CUDA(cudaEventRecord(e1, st));
        int32_t err = 0;
        KZ_CUDA(cudaMemcpyAsync(a->reports, w.dev_reports, sizeof(kz_report) * b, cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaMemcpyAsync(&err, s.err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
        if (a->device_ms) {
            KZ_CUDA(cudaEventElapsedTime(a->device_ms, e0, e1));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        for (int j = 0; j < b; ++j)
            if (a->reports[j].status == KZ_ENOTSPD) return fail(KZ_ENOTSPD, "operator is not positive definite");
        return KZ_OK;
    }
    // zero state + counters (contiguous from s.rs to the end of qpos)
    KZ_CUDA(zero_span(s.rs, w.qpos, st));
    KZ_CUDA(cudaMemsetAsync(w.red.cnt, 0, sizeof(int32_t) * nchunks, st));
    if (int rc = zero_spmm_counters(g, nchunks, w.sp, st)) return rc;
    const bool fused = small_grid > 0;
    const bool use_graphs = !fused && use_graph_loop(work, kGraphWorkCg);
    // residual-history mode (blockops.cuh CgHistory): x is formed at the end
    // from the kept residuals instead of being updated every iteration
    const bool hist = w.H >= 3 && !use_graphs && !fused;
    const bool has_x0 = eig != nullptr || a->x0 != nullptr;
    if (hist) {
        KZ_CUDA(cudaMemsetAsync(w.ahist, 0, sizeof(double) * static_cast<size_t>(w.H) * w.bpad, st));
        KZ_CUDA(cudaMemsetAsync(w.bhist, 0, sizeof(double) * static_cast<size_t>(w.H) * w.bpad, st));
        // the convergence finalize records a_k, b_k (iterations 1 .. H-1
        // run in history mode; a fold at H switches to the direction form)
        s.ahist = w.ahist;
        s.bhist = w.bhist;
        s.hist_len = w.H - 1;
    }
    // x0 = 0: the eigen start writes every x, a seeded start broadcasts it,
    // and the history form never reads an x it did not write
    if (!has_x0 && !hist) KZ_CUDA(cudaMemsetAsync(w.x, 0, blk_bytes, st));

    const unsigned sgrid = static_cast<unsigned>(nchunks) * nb;
    const unsigned tgrid = static_cast<unsigned>(std::min<int64_t>(
        static_cast<int64_t>(max_ctas_per_chunk()) * 2, ((n + 63) / 64) * nchunks));

    // right-hand side
    if (a->rhs) {
        KZ_DISPATCH_C(C, load_colmajor_kernel<CC><<<tgrid, kThreads, 0, st>>>(w.r, a->rhs, n, n * CC, b, nchunks); ::kz::note_launch());
    } else {
        KZ_CUDA(cudaMemcpyAsync(w.qpos, a->qpos, sizeof(int64_t) * b, cudaMemcpyHostToDevice, st));
        if (!eig) {  // the eigen start writes r itself and adds the rhs afterwards
            KZ_CUDA(cudaMemsetAsync(w.r, 0, blk_bytes, st));
            KZ_DISPATCH_C(C, scatter_rhs_kernel<CC><<<b, kThreads, 0, st>>>(w.r, n * CC, g->rowptr, g->colidx, w.qpos, b, a->beta); ::kz::note_launch());
        }
    }
    KZ_LAUNCH_CHECK();
    // ||b||, optional start vector (solver.py:51-59), init finalize
    if (!eig) {
        if (!a->rhs && !a->x0 && !g->vals) {
            // rhs = beta A e_q on a binary operator: ||b||^2 = beta^2 deg(q) needs no pass over the block
            KZ_DISPATCH_C(C, rhs_norm_init_kernel<CC><<<nchunks, CC < 32 ? 32 : CC, 0, st>>>(s, g->rowptr, w.qpos, a->beta); ::kz::note_launch());
        } else {
            KZ_DISPATCH_C(C, coldot_kernel<CC><<<sgrid, kThreads, 0, st>>>(w.r, w.r, n, n * CC, n * CC, w.red,
                                                                             a->x0 ? FIN_INIT_B : FIN_INIT_BR,
                                                                             s, nullptr, 0); ::kz::note_launch());
        }
        KZ_LAUNCH_CHECK();
    }
    if (a->x0) {
        KZ_DISPATCH_C(C, broadcast_kernel<CC><<<tgrid, kThreads, 0, st>>>(w.x, a->x0, n, n * CC, b, nchunks); ::kz::note_launch());
        KZ_LAUNCH_CHECK();
        SpmmArgs sa = make_spmm_args(g, w.sp);
        sa.Xg = w.x;
        sa.Xs = w.x;
        sa.Z = w.r;
        sa.Y = w.r;
        sa.s0 = 1.0;
        sa.s1 = -1.0;
        sa.s2 = a->beta;  // r = b - (x - beta*A x)
        sa.want_dot = 0;
        if (int rc = launch_spmm(g, C, nchunks, sa, st)) return rc;
        KZ_DISPATCH_C(C, coldot_kernel<CC><<<sgrid, kThreads, 0, st>>>(w.r, w.r, n, n * CC, n * CC, w.red, FIN_INIT_R, s, nullptr, 0); ::kz::note_launch());
        KZ_LAUNCH_CHECK();
    }
    if (eig) {
        // y = beta W (AU)[q,:]';  x = U y;  r = b - x + beta (AU) y
        if (w.bpad > 65535) return fail(KZ_EARG, "eigen start: at most 65535 columns per call");
        const dim3 cgrid(static_cast<unsigned>((eig->ldr + 127) / 128), static_cast<unsigned>(w.bpad));
        KZ_DISPATCH_C(C, lowrank_coef_kernel<CC><<<cgrid, 128, 0, st>>>(*eig, w.qpos, b, w.y); ::kz::note_launch());
        KZ_LAUNCH_CHECK();
        const int nt = w.bpad >= 64 ? 8 : w.bpad >= 32 ? 4 : w.bpad >= 16 ? 2 : 1;
        const size_t smem = lowrank_smem(eig->ldr, 8 * nt);
        // walk start: 2-walk counts into the (still unused) q block, int32
        int32_t* cnt = nullptr;
        const bool three_term = eig->a4u != nullptr;
        const bool two_term = eig->a3u != nullptr || three_term;
        if (eig->a2u || two_term) {
            cnt = reinterpret_cast<int32_t*>(w.q);
            KZ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * static_cast<size_t>(w.bpad) * n, st));
            const dim3 wgrid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(64, g->max_deg))),
                             static_cast<unsigned>(w.bpad));
            KZ_DISPATCH_C(C, walk2_count_kernel<CC><<<wgrid, kThreads, 0, st>>>(cnt, n * CC, g->rowptr, g->colidx,
                                                                                w.qpos, b);
                          ::kz::note_launch());
            KZ_LAUNCH_CHECK();
        }
        const int64_t ntiles = (n + kLrRows - 1) / kLrRows;
        const unsigned lgrid = static_cast<unsigned>(std::min<int64_t>(KZ_LR_MINBLOCKS * num_sms(), ntiles));
        for (int j0 = 0; j0 < w.bpad; j0 += 8 * nt) {
#define KZ_LR(NN)                                                                                              \
    do {                                                                                                       \
        KZ_DISPATCH_C(C, {                                                                                     \
            if (two_term) {                                                                                    \
                KZ_CUDA(cudaFuncSetAttribute(lowrank_init_kernel<CC, NN, true>,                                \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))); \
                lowrank_init_kernel<CC, NN, true><<<lgrid, 32 * kLrWarps, smem, st>>>(*eig, w.y, w.x, nullptr, \
                                                                                      nullptr, n * CC, j0, w.bpad, cnt, \
                                                                                      three_term ? w.p : nullptr); \
            } else {                                                                                           \
                KZ_CUDA(cudaFuncSetAttribute(lowrank_init_kernel<CC, NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             static_cast<int>(smem)));                                         \
                lowrank_init_kernel<CC, NN><<<lgrid, 32 * kLrWarps, smem, st>>>(*eig, w.y, w.x, w.r, hist ? nullptr : w.p, n * CC, \
                                                                                j0, w.bpad, cnt);              \
            }                                                                                                  \
            ::kz::note_launch();                                                                               \
        });                                                                                                    \
    } while (0)
            if (nt == 8) KZ_LR(8);
            else if (nt == 4) KZ_LR(4);
            else if (nt == 2) KZ_LR(2);
            else KZ_LR(1);
#undef KZ_LR
            KZ_LAUNCH_CHECK();
        }
        // b = beta A e_q onto r0 and p0, or (walk start) onto x0
        KZ_DISPATCH_C(C, eigen_add_rhs_kernel<CC><<<w.bpad, kThreads, 0, st>>>(cnt ? w.x : w.r, cnt || hist ? nullptr : w.p,
                                                                                n * CC, g->rowptr, g->colidx,
                                                                                w.qpos, b, a->beta, s.bnorm2);
                      ::kz::note_launch());
        KZ_LAUNCH_CHECK();
        if (three_term) {
            // third Katz term: x0 += beta * A (beta^2 A^2 e_q), one K1 SpMM on
            // the count block the low-rank kernel left in p
            SpmmArgs sa = make_spmm_args(g, w.sp);
            sa.Xg = w.p;
            sa.Xs = nullptr;
            sa.Z = w.x;
            sa.Y = w.x;
            sa.s0 = 1.0;
            sa.s1 = 0.0;
            sa.s2 = a->beta;
            sa.want_dot = 0;
            sa.chunk_active = nullptr;
            if (int rc = launch_spmm(g, C, nchunks, sa, st)) return rc;
        }
        if (two_term) {
            // r0 = b - (x0 - beta A x0): one K1 SpMM on x0 (exactly consistent
            // with x0), then the rhs scattered on top
            SpmmArgs sa = make_spmm_args(g, w.sp);
            sa.Xg = w.x;
            sa.Xs = w.x;
            sa.Z = nullptr;
            sa.Y = w.r;
            sa.s0 = 0.0;
            sa.s1 = -1.0;
            sa.s2 = a->beta;
            sa.want_dot = 0;
            sa.chunk_active = nullptr;
            if (int rc = launch_spmm(g, C, nchunks, sa, st)) return rc;
            KZ_DISPATCH_C(C, eigen_add_rhs_kernel<CC><<<w.bpad, kThreads, 0, st>>>(w.r, nullptr, n * CC, g->rowptr,
                                                                                    g->colidx, w.qpos, b, a->beta,
                                                                                    s.bnorm2);
                          ::kz::note_launch());
            KZ_LAUNCH_CHECK();
            if (!hist) KZ_CUDA(cudaMemcpyAsync(w.p, w.r, blk_bytes, cudaMemcpyDeviceToDevice, st));
        }
        KZ_DISPATCH_C(C, coldot_kernel<CC><<<sgrid, kThreads, 0, st>>>(w.r, w.r, n, n * CC, n * CC, w.red, FIN_INIT_R, s, nullptr, 0); ::kz::note_launch());
        KZ_LAUNCH_CHECK();
    }
    // p0 = r0; in history mode r0 stays in slot 0, so the first iteration reads
    // its direction from there and p is first written by that pupdate
    if (!eig && !hist) KZ_CUDA(cudaMemcpyAsync(w.p, w.r, blk_bytes, cudaMemcpyDeviceToDevice, st));

    const int lag = work > 2e7 ? 1 : 3;
    auto slot = [&](int i) { return w.r + static_cast<size_t>(i) * blk_elems; };
    auto history = [&]() {
        CgHistory h;
        h.slots = w.r;
        h.slot = blk_elems;
        h.coef = w.coef;
        h.kcol = w.kcol;
        h.x0 = has_x0 ? w.x : nullptr;
        h.bpad = w.bpad;
        return h;
    };
    auto hist_coef = [&](int limit) -> int {
        cg_hist_coef_kernel<<<static_cast<unsigned>((w.bpad + 127) / 128), 128, 0, st>>>(
            w.ahist, w.bhist, s.iters, limit, b, w.bpad, w.coef, w.kcol);
        ::kz::note_launch();
        KZ_LAUNCH_CHECK();
        return KZ_OK;
    };
    bool folded = false;
    // a solve from zero with b = beta A e_q: the first iteration's SpMM is
    // replaced by the 2-walk counts (cg_sparse_pq_kernel); KZ_CG_SPARSE_FIRST=0
    // turns it off
    const char* sf_env = std::getenv("KZ_CG_SPARSE_FIRST");
    const bool sparse_first_on = !(sf_env && sf_env[0] == '0');
    const bool sparse_first = sparse_first_on && !eig && !a->rhs && !a->x0 && a->qpos && !use_graphs && !fused &&
                              w.bpad <= 65535;  // one grid row per column in walk2_count_kernel
    auto k1_args = [&](const double* xin, const double* z, int k) {
        SpmmArgs sa = make_spmm_args(g, w.sp);
        sa.Xg = xin;
        sa.Xs = xin;
        sa.Z = z;
        sa.Y = w.q;
        sa.s0 = 0.0;
        sa.s0v = z ? s.betac : nullptr;  // q-recurrence: q = M r + b_{k-1} q
        sa.s1 = 1.0;
        sa.s2 = -a->beta;
        sa.D = nullptr;  // dots with Xs: p.q (direction form) or r.q (q-recurrence)
        sa.chunk_active = s.chunk_active;
        sa.want_dot = 1;
        sa.hook.mode = 1;
        sa.hook.b = b;
        sa.hook.rs = s.rs;
        sa.hook.alpha = s.alpha;
        sa.hook.active = s.active;
        sa.hook.xstamp = s.xstamp;
        sa.hook.chunk_xstamp = s.chunk_xstamp;
        sa.hook.status = s.status;
        sa.hook.err = s.err;
        sa.hook.n_active = s.n_active;
        sa.hook.iter = k;
        sa.hook.iter_dev = s.iter_dev;
        return sa;
    };
    auto launch_iter = [&](int k) -> int {
        // history mode (q-recurrence) for iterations 1 .. H-1: r_k -> slot k;
        // a solve that needs iteration H folds x and the direction p from the
        // slots once and continues in the direction form, in place
        if (hist && !folded && k >= w.H) {
            if (int rc = hist_coef(w.H - 1)) return rc;
            cg_hist_dcoef_kernel<<<static_cast<unsigned>((w.bpad + 127) / 128), 128, 0, st>>>(w.bhist, w.H, w.bpad,
                                                                                             w.dcoef);
            ::kz::note_launch();
            const unsigned fgrid = static_cast<unsigned>(std::min<int64_t>(8 * max_ctas_per_chunk(), (static_cast<int64_t>(blk_elems) + 255) / 256));
            KZ_DISPATCH_C(C, cg_hist_fold_kernel<CC><<<fgrid, 256, 0, st>>>(w.x, history(), n, nchunks, w.p, w.dcoef,
                                                                            w.H);
                          ::kz::note_launch());
            KZ_LAUNCH_CHECK();
            folded = true;
        }
        if (hist && !folded) {
            double* rin = slot(k - 1);
            double* rout = slot(k);
            if (k == 1 && sparse_first) {
                // q0 = M r0 from the 2-walk counts (kept in p, unused in this
                // form), p0.q0 over N(q); the update stores q0 for q1
                int32_t* cnt = reinterpret_cast<int32_t*>(w.p);
                KZ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * static_cast<size_t>(w.bpad) * n, st));
                const dim3 wgrid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(64, g->max_deg))),
                                 static_cast<unsigned>(w.bpad));
                KZ_DISPATCH_C(C, walk2_count_kernel<CC><<<wgrid, kThreads, 0, st>>>(cnt, n * CC, g->rowptr, g->colidx,
                                                                                    w.qpos, b);
                              ::kz::note_launch());
                KZ_LAUNCH_CHECK();
                KZ_DISPATCH_C(C, cg_sparse_pq_kernel<CC><<<w.bpad, kThreads, 0, st>>>(rin, cnt, n * CC, g->rowptr,
                                                                                      g->colidx, w.qpos, a->beta, s, k);
                              ::kz::note_launch());
                KZ_LAUNCH_CHECK();
                KZ_DISPATCH_C(C, cg_update_kernel<CC><<<sgrid, kThreads, 0, st>>>(rin, nullptr, n, n * CC, n * CC, w.red,
                                                                                  FIN_CG_CONV, s, k, cnt, a->beta, rout,
                                                                                  w.q);
                              ::kz::note_launch());
                KZ_LAUNCH_CHECK();
                return KZ_OK;
            }
            // q_{k-1} = M r_{k-1} + b_{k-2} q_{k-2} (q0 = M r0), a = rs / r.q
            if (int rc = launch_spmm(g, C, nchunks, k1_args(rin, k == 1 ? nullptr : w.q, k), st)) return rc;
            KZ_DISPATCH_C(C, cg_update_kernel<CC><<<sgrid, kThreads, 0, st>>>(rin, w.q, n, n * CC, n * CC, w.red,
                                                                              FIN_CG_CONV, s, k, nullptr, 0.0, rout);
                          ::kz::note_launch());
            KZ_LAUNCH_CHECK();
            return KZ_OK;
        }
        // direction form: after a fold r lives in slot H-1 (updated in place)
        double* rin = hist ? slot(w.H - 1) : w.r;
        if (k == 1 && sparse_first) {
            int32_t* cnt = reinterpret_cast<int32_t*>(w.q);
            KZ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * static_cast<size_t>(w.bpad) * n, st));
            const dim3 wgrid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(64, g->max_deg))),
                             static_cast<unsigned>(w.bpad));
            KZ_DISPATCH_C(C, walk2_count_kernel<CC><<<wgrid, kThreads, 0, st>>>(cnt, n * CC, g->rowptr, g->colidx,
                                                                                w.qpos, b);
                          ::kz::note_launch());
            KZ_LAUNCH_CHECK();
            KZ_DISPATCH_C(C, cg_sparse_pq_kernel<CC><<<w.bpad, kThreads, 0, st>>>(rin, cnt, n * CC, g->rowptr,
                                                                                  g->colidx, w.qpos, a->beta, s, k);
                          ::kz::note_launch());
            KZ_LAUNCH_CHECK();
            KZ_DISPATCH_C(C, cg_update_kernel<CC><<<sgrid, kThreads, 0, st>>>(rin, w.q, n, n * CC, n * CC, w.red,
                                                                              FIN_CG_CONV, s, k, cnt, a->beta);
                          ::kz::note_launch());
            KZ_LAUNCH_CHECK();
            KZ_DISPATCH_C(C, cg_pupdate_kernel<CC><<<sgrid, kThreads, 0, st>>>(w.x, w.p, rin, n, n * CC, n * CC, n * CC, nb, s, k); ::kz::note_launch());
            KZ_LAUNCH_CHECK();
            return KZ_OK;
        }
        if (int rc = launch_spmm(g, C, nchunks, k1_args(w.p, nullptr, k), st)) return rc;
        KZ_DISPATCH_C(C, cg_update_kernel<CC><<<sgrid, kThreads, 0, st>>>(rin, w.q, n, n * CC, n * CC, w.red, FIN_CG_CONV, s, k); ::kz::note_launch());
        KZ_LAUNCH_CHECK();
        KZ_DISPATCH_C(C, cg_pupdate_kernel<CC><<<sgrid, kThreads, 0, st>>>(w.x, w.p, rin, n, n * CC, n * CC, n * CC, nb, s, k); ::kz::note_launch());
        KZ_LAUNCH_CHECK();
        return KZ_OK;
    };
    int64_t ran = 0;
    long long per_iter = 0;
    int rc;
    if (fused) {
        SmallCgArgs sa{};
        sa.rows = static_cast<int32_t>(n);
        sa.nchunks = nchunks;
        sa.b = b;
        sa.bpad = w.bpad;
        sa.rowptr = g->rowptr;
        sa.colidx = g->colidx;
        sa.beta = a->beta;
        sa.x = w.x;
        sa.r = w.r;
        sa.p = w.p;
        sa.q = w.q;
        sa.part = w.small_part;
        sa.carry = w.small_carry;
        sa.stamp = w.small_stamp;
        sa.s = s;
        void* kargs[] = {&sa};
        KZ_DISPATCH_C(C, KZ_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(cg_small_kernel<CC>),
                                                            dim3(small_grid), dim3(kSmallCgThreads), kargs, 0, st)));
        note_launch();
        rc = KZ_OK;
    } else if (use_graphs) {
        // small solves are launch-bound: the whole loop is one cached graph
        // with a device-side WHILE condition (driver.cuh)
        GraphKey key;
        key.v[0] = g->uid;
        key.v[1] = reinterpret_cast<uint64_t>(ws);
        // the workspace layout: history slots and eig change every offset
        key.v[2] = static_cast<uint64_t>(w.H) | (reinterpret_cast<uint64_t>(w.q) << 8);
        key.v[3] = static_cast<uint64_t>(b) | (static_cast<uint64_t>(has_x0) << 32);
        std::memcpy(&key.v[4], &a->beta, sizeof(double));
        std::memcpy(&key.v[5], &a->tol, sizeof(double));
        key.v[6] = static_cast<uint64_t>(s.max_iter);
        key.v[7] = reinterpret_cast<uint64_t>(eig);
        rc = run_iterations_graph(s, st, launch_iter, key, &per_iter);
    } else {
        rc = run_iterations(s, s.max_iter, lag, st, launch_iter, &ran, hist ? w.H : 0);
    }
    if (rc) return rc;

    // the output pass forms x from the residual history unless it was folded
    CgHistory oh;
    if (hist && !folded) {
        if (int rc2 = hist_coef(w.H)) return rc2;
        oh = history();
    }
    if (a->perm) {
        invert_perm_kernel<<<static_cast<unsigned>(std::min<int64_t>(4 * max_ctas_per_chunk(), (n + 255) / 256)), 256, 0, st>>>(a->perm, w.iperm, n);
        ::kz::note_launch();
        KZ_DISPATCH_C(C, store_gather_kernel<CC><<<tgrid, kThreads, 0, st>>>(a->scores, w.x, n, n * CC, b, nchunks, w.iperm, a->clamp, oh); ::kz::note_launch());
    } else {
        KZ_DISPATCH_C(C, store_colmajor_kernel<CC><<<tgrid, kThreads, 0, st>>>(a->scores, w.x, n, n * CC, b, nchunks, nullptr, a->clamp, oh); ::kz::note_launch());
    }
    KZ_LAUNCH_CHECK();
    if (a->device_ms) {
        KZ_CUDA(cudaEventRecord(e1, st));
    }
    // reports
    std::vector<int64_t> iters(b);
    std::vector<int32_t> conv(b), status(b);
    std::vector<double> rnorm(b), bnorm2(b);
    KZ_CUDA(cudaMemcpyAsync(iters.data(), s.iters, sizeof(int64_t) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(conv.data(), s.converged, sizeof(int32_t) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(status.data(), s.status, sizeof(int32_t) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(rnorm.data(), s.rnorm, sizeof(double) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaMemcpyAsync(bnorm2.data(), s.bnorm2, sizeof(double) * b, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    if (a->device_ms) {
        KZ_CUDA(cudaEventElapsedTime(a->device_ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    if (use_graphs) {  // loop iterations the graph ran: at least one, else the longest column
        int64_t mx = 1;
        for (int j = 0; j < b; ++j) mx = std::max<int64_t>(mx, iters[j]);
        add_launches(per_iter * mx);
    }
    bool notspd = false;
    for (int j = 0; j < b; ++j) {
        a->reports[j].iterations = iters[j];
        a->reports[j].converged = conv[j];
        a->reports[j].status = status[j];
        a->reports[j].final_residual_norm = rnorm[j];
        a->reports[j].rhs_norm = std::sqrt(bnorm2[j]);
        notspd = notspd || status[j] == KZ_ENOTSPD;
    }
    if (notspd) return fail(KZ_ENOTSPD, "operator is not positive definite");
    return KZ_OK;
}

extern "C" int kz_cg_batch(const kz_graph* g, const kz_cg_args* a, void* ws, size_t ws_bytes,
                           void* stream) {
    clear_error();
    return cg_batch_impl(g, a, ws, ws_bytes, stream, nullptr);
}

// ---- eigen-of-A low-rank start + CG ----------------------
extern "C" int kz_eigen_create(const kz_eigen_desc* d, kz_eigen** out) {
    clear_error();
    if (!d || !out) return fail(KZ_EARG, "NULL argument");
    *out = nullptr;
    if (!d->op || d->n < 1 || d->r < 1 || d->ldr < d->r || d->ldr % 4 != 0 || !d->u || !d->au || !d->w)
        return fail(KZ_EARG, "bad eigen index description");
    if (d->op->rows != d->n || d->op->cols != d->n) return fail(KZ_EARG, "operator size differs from n");
    if (lowrank_smem(d->ldr, 64) > 227 * 1024) return fail(KZ_EARG, "rank too large (ldr > 384)");
    auto* h = new kz_eigen();
    h->n = d->n;
    h->r = d->r;
    h->ldr = d->ldr;
    h->beta = d->beta;
    h->op = d->op;
    h->u = d->u;
    h->au = d->au;
    h->w = d->w;
    h->a2u = d->a2u;
    h->a3u = d->a3u;
    h->a4u = d->a4u;
    *out = h;
    return KZ_OK;
}

extern "C" int kz_eigen_destroy(kz_eigen* h) {
    delete h;
    return KZ_OK;
}

extern "C" size_t kz_eigen_workspace_bytes(const kz_eigen* h, int32_t b) {
    if (!h || b < 1) return 0;
    Carver cv(nullptr, 0);
    CgWork w;
    carve_cg(cv, h->op, b, w, h);
    return cv.off + 256;
}

extern "C" int kz_eigen_batch(const kz_eigen* h, const kz_cg_args* a, void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    if (!h || !a) return fail(KZ_EARG, "NULL argument");
    if (a->beta != h->beta) return fail(KZ_EARG, "beta differs from the eigen index's");
    return cg_batch_impl(h->op, a, ws, ws_bytes, stream, h);
}

extern "C" size_t kz_coldot_workspace_bytes(int64_t n, int32_t b) {
    if (n < 1 || b < 1) return 256;
    const size_t nb = static_cast<size_t>(stream_ctas_per_chunk(n, 1, b));
    return ((sizeof(double) * static_cast<size_t>(b) * nb + 255) & ~size_t(255)) + sizeof(int32_t) * b + 256;
}

extern "C" int kz_coldot(int64_t n, int32_t b, const double* X, const double* Y, double* out,
                         void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    if (n < 1 || b < 1 || !X || !Y || !out) return fail(KZ_EARG, "bad coldot arguments");
    if (!ws || ws_bytes < kz_coldot_workspace_bytes(n, b)) return fail(KZ_EARG, "workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // column-major == chunk width 1, one chunk per column
    const int nb = stream_ctas_per_chunk(n, 1, b);
    Carver cv(ws, ws_bytes);
    RedScratch red;
    red.nb = nb;
    red.part = cv.take<double>(static_cast<size_t>(b) * nb);
    red.cnt = cv.take<int32_t>(b);
    KZ_CUDA(cudaMemsetAsync(red.cnt, 0, sizeof(int32_t) * b, st));
    SolveState s;
    coldot_kernel<1><<<static_cast<unsigned>(b) * nb, kThreads, 0, st>>>(X, Y, n, n, n, red, FIN_WRITE, s, out, 0); ::kz::note_launch();
    KZ_LAUNCH_CHECK();
    return KZ_OK;
}

// out = a*x + b*y (y may be NULL: out = a*x) with separately rounded products
// and sum -- numpy's `x += a*p`, `r -= a*q`, `p = r + beta*p` bit for bit;
// op 1: out = x / a (numpy's `w / nw`).
__global__ void vec_op_kernel(int op, int64_t n, double a, const double* x, double b, const double* y,
                              double* out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (op == 1) {
            out[i] = __ddiv_rn(x[i], a);
        } else {
            const double ax = __dmul_rn(a, x[i]);
            out[i] = y ? __dadd_rn(ax, __dmul_rn(b, y[i])) : ax;
        }
    }
}

extern "C" int kz_vec_op(int32_t op, int64_t n, double a, const double* x, double b, const double* y,
                         double* out, void* stream) {
    clear_error();
    if (n < 0 || !x || !out || (op != 0 && op != 1)) return fail(KZ_EARG, "bad vec_op arguments");
    if (n == 0) return KZ_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(4 * max_ctas_per_chunk(), (n + 255) / 256));
    vec_op_kernel<<<grid, 256, 0, st>>>(op, n, a, x, b, y, out);
    ::kz::note_launch();
    KZ_LAUNCH_CHECK();
    return KZ_OK;
}
