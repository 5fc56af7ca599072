/*
 * katzb200.h -- C-ABI of the B200-native Katz query hot path (libkatzb200.so).
 *
 * This is the drop-in boundary for the query path of the reference package
 * `lrckatz` (/root/reference/pkg/src/lrckatz).  The reference has no FFI: its
 * boundary is the module-level Python API re-exported in __init__.py:9-72.
 * Each entry point below replaces the numpy/scipy arithmetic behind one of
 * those Python functions; the Python mirror in paper_1912_06525_b200/ binds
 * them through ctypes.
 *
 * Conventions
 *  - Every function returns an int status (KZ_OK == 0).  On failure
 *    kz_last_error() returns a thread-local message.
 *  - Device pointers are plain CUDA device pointers (e.g. torch tensors'
 *    data_ptr()); `stream` is a cudaStream_t passed as void*.
 *  - Dense blocks of b vectors of length n use the "chunked node-major"
 *    layout [b/C][n][C]: element (row i, column j) lives at
 *    ((j / C) * n + i) * C + (j % C).  C == 1 is plain column-major [b][n].
 *  - All arithmetic is IEEE fp64.  Indices are int32 on the device
 *    (nnz < 2^31 is checked at creation).
 *  - Handles are immutable after creation; calls on distinct streams with
 *    distinct workspaces are reentrant (reference SPEC.md:359 threading).
 */
#ifndef KATZB200_H
#define KATZB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python mirror maps them to the reference exceptions */
#define KZ_OK 0
#define KZ_EARG 1      /* ValueError            (solver.py:106-107, linkpred.py:157-181) */
#define KZ_ENOTSPD 2   /* RuntimeError "... not positive definite" (solver.py:84-85,140-141) */
#define KZ_ESPECTRUM 3 /* SpectrumError         (factor.py:27-28,329-330) */
#define KZ_ECUDA 4     /* RuntimeError (CUDA failure) */
#define KZ_EOOM 5      /* MemoryError */

/* Binary-pattern CSR operator A (rows x cols, no stored values) resident on
 * the device, plus its precomputed SpMM schedule (row partition, long-row
 * segments).  Replaces the scipy CSR operands of solver.py:110,115,178 and
 * index.py:89-90. */
typedef struct kz_graph kz_graph;

/* Per-query solve report; mirrors SolveReport (solver.py:29-34). */
typedef struct kz_report {
    int64_t iterations;
    int32_t converged;
    int32_t status; /* per-column KZ_* status (KZ_ENOTSPD for p.q <= 0) */
    double final_residual_norm;
    double rhs_norm;
} kz_report;

const char* kz_last_error(void);
int kz_version(void);
/* total kernels this library has launched in the process (bench evidence) */
long long kz_launch_count(void);
/* SM count of the current device (every persistent grid is sized from it) */
int kz_num_sms(void);
/* K1 launch timing (bench.py's roofline): kz_k1_timing(1) clears and starts
 * recording a pair of CUDA events around every K1 SpMM launch on its own
 * stream (launches inside stream capture are not timed); kz_k1_timing_read
 * synchronises on them and returns the summed launch time and the number
 * of timed launches.  kz_k1_timing(0) stops recording and frees the events. */
int kz_k1_timing(int enable);
/* Checked builds (make EXTRA=-DKZ_CHECKED=1): kz_checked() is 1; every
 * workspace slice gets a 256-byte red zone in front, and
 * kz_checked_redzones(ws, offs, cap) returns how many red zones the calls of
 * this thread carved in workspace `ws` since the last query (their byte
 * offsets in offs[0..cap)), then forgets them.  Release builds: 0 / 0. */
int kz_checked(void);
int64_t kz_checked_redzones(const void* ws, int64_t* offs, int64_t cap);
int kz_k1_timing_read(double* total_ms, long long* launches);

/* ---- operator handles ------------------------------------------------- */

/* Upload a CSR pattern.  rowptr: int64[rows+1], colidx: int32[nnz]; either
 * host or device memory (UVA-detected).  Columns must lie in [0, cols). */
int kz_graph_create(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rowptr,
                    const int32_t* colidx, kz_graph** out);
int kz_graph_destroy(kz_graph* g);
/* rows, cols, nnz, number of long rows, number of long-row segments */
int kz_graph_info(const kz_graph* g, int64_t* rows, int64_t* cols, int64_t* nnz,
                  int64_t* nlong, int64_t* nitems);

/* ---- K1: binary CSR SpMM with fused epilogue ---------------------------
 * Y = s0*Z + s1*Xs + s2*(A Xg)  on b columns in layout [b/C][.][C];
 * Xg has `cols` rows, Xs/Z/Y/D have `rows` rows.  Z or Xs may be NULL.
 * If dots != NULL (device double[b]) it receives dots[j] = sum_i D[i,j]*Y[i,j]
 * (D == NULL means D = Xs; dots need chunk <= 32, chunk 64 computes the
 * product only).  Replaces KatzIndex.apply_m_permuted
 * (index.py:86-91) with s0=0, s1=1, s2=-alpha, and the m12 / m12.T products
 * of solver.py:110,115,178.  Workspace: kz_spmm_workspace_bytes(). */
size_t kz_spmm_workspace_bytes(const kz_graph* g, int32_t b, int32_t chunk);
int kz_spmm(const kz_graph* g, int32_t b, int32_t chunk, const double* Xg, const double* Xs,
            const double* Z, double* Y, double s0, double s1, double s2, const double* D,
            double* dots, void* ws, size_t ws_bytes, void* stream);

/* ---- K2: batched textbook CG on (I - beta*A) x = rhs --------------------
 * One call solves b Katz queries (columns) with per-column convergence
 * masking; each column follows cg() (solver.py:62-101) exactly: x0 = 0 (or
 * the given start vector), stop when ||r|| <= tol*||rhs||, raise (KZ_ENOTSPD)
 * if p.q <= 0, at most max_iter iterations.  The right-hand side of column j
 * is beta * A[:, qpos[j]] (rhs_for_position, index.py:93-101) unless `rhs`
 * is given.  Output: scores[j][perm[i]] = clamp(x_j[i]) (solver.py:223-225). */
typedef struct kz_cg_args {
    int32_t b;            /* number of query columns */
    int32_t clamp;        /* 1: scores = max(x, 0) */
    const int64_t* qpos;  /* host int64[b]: query rows (operator order); ignored if rhs */
    const double* rhs;    /* device double[b][n] column-major, or NULL */
    double beta;          /* damping factor (alpha of the reference) */
    double tol;           /* relative residual tolerance */
    int64_t max_iter;     /* <= 0 means 10*n (solver.py:69-70) */
    const double* x0;     /* device double[n] start vector shared by all columns, or NULL */
    const int64_t* perm;  /* device int64[n] output scatter (perm[i] = internal id), or NULL */
    double* scores;       /* device double[b][n] output */
    kz_report* reports;   /* host kz_report[b] output */
    float* device_ms;     /* optional host float: device time of the solve (CUDA events) */
} kz_cg_args;
size_t kz_cg_workspace_bytes(const kz_graph* g, int32_t b);
int kz_cg_batch(const kz_graph* g, const kz_cg_args* a, void* ws, size_t ws_bytes, void* stream);

/* Weighted operator (fp64 values), e.g. the block-diagonal M11^-1 whose
 * dense per-part blocks replace BlockCholesky.solve (factor.py:89-106). */
int kz_graph_create_weighted(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rowptr,
                             const int32_t* colidx, const double* vals, kz_graph** out);

/* ---- LRC-Katz: batched Schur-complement PCG (query, solver.py:161-207) ----
 * The handle borrows every operand (device memory owned by the caller):
 * K1 operators of A in partition order (full n x n, A12 n1 x n2, A21 n2 x n1,
 * A22 n2 x n2), the weighted block-diagonal M11^-1 (n1 x n1), the dense
 * row-major L^-1 and (L^-1)^T (n2 x n2), U (n2 x ell) and (U diag(d))^T
 * (ell x n2) with d = 1/(1-sigma) - 1 (factor.py:322-337).  Dense operands
 * use a leading dimension rounded up to even (n2 + n2%2, ell + ell%2) with
 * zero padding, so pairs of entries load as one 16-byte access.  sigma is read
 * (host) only to raise KZ_ESPECTRUM when any sigma >= 1 (factor.py:329-330). */
typedef struct kz_lrc kz_lrc;
typedef struct kz_lrc_desc {
    int64_t n, n1, n2, ell;
    double beta;
    const kz_graph* full;
    const kz_graph* a12;
    const kz_graph* a21;
    const kz_graph* a22;
    const kz_graph* minv;
    const double* linv;
    const double* linvT;
    const double* u;
    const double* udT;
    const double* sigma; /* host double[ell] */
} kz_lrc_desc;

/* Query mode (f == NULL): column j solves query position qpos[j] (partition
 * order) end to end -- rhs, Schur reduction, PCG with tol_eff, back
 * substitution, whole-system residual, scatter through perm, clamp -- and
 * writes scores out[j][n]; the report carries the inner PCG iterations and
 * the true residual (solver.py:185-190).  PCG mode (f != NULL, device
 * [b][n2]): lrc_pcg (solver.py:118-158) on the given Schur rhs, x into
 * out[j][n2], recursive residual in the report. */
typedef struct kz_lrc_args {
    int32_t b;
    int32_t chunk; /* 0: default; 1, 2, 4, ..., 32 */
    int32_t clamp;
    int32_t _pad;
    const int64_t* qpos; /* host int64[b] */
    const double* f;
    double tol;
    int64_t max_iter; /* <= 0: 10*n2 */
    const double* x0; /* device double[n2] start vector (start_seed), or NULL */
    const int64_t* perm;
    double* out;
    kz_report* reports;
    float* device_ms;
} kz_lrc_args;

#define KZ_LRC_SCHUR 0     /* out = S in1                      (solver.py:113-115) */
#define KZ_LRC_PRECOND 1   /* out = S~^-1 in1                  (factor.py:322-337) */
#define KZ_LRC_SCHUR_RHS 2 /* out = in2 - M12' M11^-1 in1      (solver.py:104-110) */
#define KZ_LRC_CORRECTION 3 /* out = L^-1 M12' M11^-1 M12 L^-T in1 (factor.py:196-202) */

int kz_lrc_create(const kz_lrc_desc* d, kz_lrc** out);
int kz_lrc_destroy(kz_lrc* h);
int kz_lrc_info(const kz_lrc* h, int64_t* n, int64_t* n1, int64_t* n2, int64_t* ell);
size_t kz_lrc_workspace_bytes(const kz_lrc* h, int32_t b, int32_t chunk);
int kz_lrc_batch(const kz_lrc* h, const kz_lrc_args* a, void* ws, size_t ws_bytes, void* stream);
/* op in KZ_LRC_*; in1/in2/out column-major [b][rows] */
int kz_lrc_apply(const kz_lrc* h, int32_t op, int32_t b, const double* in1, const double* in2,
                 double* out, void* ws, size_t ws_bytes, void* stream);

/* ---- K4: batched masked top-k --------------------------------------------
 * For each column j of scores (device double[b][n], entries >= 0) select the
 * k entries with the largest (score desc, id asc) key among ids that are not
 * masked.  The mask of column j is {self_ids[j]} U neighbors(mask_rows[j]) in
 * mask_graph (either part may be -1 / NULL).  This is _candidate_order
 * (linkpred.py:145-152) and the anchor selection (linkpred.py:186-188).
 * Outputs: ids_out int64[b][k], vals_out double[b][k], count_out int32[b]. */
typedef struct kz_topk_args {
    int32_t b;
    int32_t k;
    int64_t n;
    const double* scores;
    const kz_graph* mask_graph; /* may be NULL */
    const int64_t* mask_rows;   /* host int64[b] or NULL */
    const int64_t* self_ids;    /* host int64[b] or NULL */
    int64_t* ids_out;
    double* vals_out;
    int32_t* count_out;
    /* optional exclusive upper bound per column (device double[b] and
     * int64[b], both or neither): only keys strictly below (bound_vals[j],
     * bound_ids[j]) in (score desc, id asc) order take part; bound_ids[j] < 0
     * means no bound.  One call returns at most 4096 entries per column; a
     * larger k continues from the last key of the previous pass. */
    const double* bound_vals;
    const int64_t* bound_ids;
} kz_topk_args;
size_t kz_topk_workspace_bytes(int32_t b, int64_t n, int32_t k);
int kz_topk_batch(const kz_topk_args* a, void* ws, size_t ws_bytes, void* stream);

/* ---- K7: sparse_katz anchor profiles and Pearson rerank ------------------
 * kz_profile_gather: for each triple t = (src, j, slot) of trip (device
 * int64[ntrip][3]) copy S[src][top_ids[j][c]] into profiles[j][slot][c] for
 * c < counts[j]  (the profile rows of linkpred.py:189-196).
 * kz_pearson_rerank: per query j, corr[c] = Pearson(ref[j], profiles[j][:, c])
 * (0 for zero variance, clipped to [-1, 1]) and the rerank order of
 * lexsort((top, -score, -corr)) (linkpred.py:197-205), sorted in shared
 * memory for s <= 8192; order_out == NULL computes the correlations only
 * (the Python mirror orders s > 8192 candidates with a device sort). */
int kz_profile_gather(const double* S, int64_t n, int32_t ntrip, const int64_t* trip,
                      const int64_t* top_ids, const int32_t* counts, int32_t s, double* profiles,
                      int32_t T1, void* stream);
int kz_pearson_rerank(const double* profiles, const double* ref, const int64_t* top_ids,
                      const double* top_scores, const int32_t* counts, int32_t b, int32_t T1,
                      int32_t s, double* corr_out, int64_t* order_out, void* stream);

/* ---- ingestion: connected components (largest_connected_component) -------
 * labels[i] = smallest node id of i's component (the order in which the
 * reference's BFS numbers components, graph.py:211-229), from device edge
 * endpoints src/dst (int32[nnz], any orientation, duplicates allowed). */
/* from_edges (graph.py:111-148) on the device: drop self-loops, symmetrise,
 * deduplicate, columns sorted within rows (two radix sorts of the 64-bit
 * keys u*n+v and a unique pass) -- the reference's CSR byte for byte.
 * u, v: device int64[m] endpoints in [0, n) (KZ_EARG otherwise).  Outputs:
 * row_offsets device int64[n+1]; col device int32 and src device int32 (the
 * row of each entry; may be NULL), both with capacity 2*m; *nnz_out (host)
 * = stored entries.  Workspace: kz_edges_to_csr_workspace_bytes(n, m). */
size_t kz_edges_to_csr_workspace_bytes(int64_t n, int64_t m);
int kz_edges_to_csr(int64_t n, int64_t m, const int64_t* u, const int64_t* v, int64_t* row_offsets, int32_t* col,
                    int32_t* src, int64_t* nnz_out, void* ws, size_t ws_bytes, void* stream);
int kz_connected_components(int64_t n, int64_t nnz, const int32_t* src, const int32_t* dst,
                            int32_t* labels, void* stream);

/* ---- eigen-of-A low-rank start + CG (north-star LRC) ---
 * Not in the reference (its LRC is the Schur form above); parity is against
 * the exact solution.  Index: U = top-r Ritz vectors of A in the operator's
 * order, AU = A U, W = (I - beta U'AU)^-1.  kz_eigen_batch solves the same
 * systems as kz_cg_batch (query columns by qpos; rhs and x0 must be NULL)
 * but starts each column at the Galerkin point x0 = U W U' b with the exact
 * residual r0 = b - x0 + beta (AU)(W U' b) -- two tall-skinny fp64 DMMA
 * products, no SpMM -- then runs the reference's CG recurrence from there
 * with the stop test ||r|| <= tol ||b|| (solver.py:62-101).
 * With a2u = A^2 U (optional) the start also carries the first Katz-series
 * term exactly: x0 = beta A e_q + U y, y = beta^2 W (A^2 U)[q,:]', whose
 * residual r0 = beta^2 A^2 e_q - U y + beta (AU) y needs only the 2-walk
 * counts from q (an integer sparse push, no SpMM): one CG iteration fewer.
 * With a3u = A^3 U the start carries the first two terms, x0 = beta A e_q +
 * beta^2 A^2 e_q + U y, y = beta^3 W (A^3 U)[q,:]', and r0 comes from one
 * SpMM on x0 (no (AU) y product): one more CG iteration fewer.  With a4u =
 * A^4 U the third term beta^3 A^3 e_q is added by one more SpMM on the
 * beta^2 A^2 e_q block and y = beta^4 W (A^4 U)[q,:]': one more again. */
typedef struct kz_eigen kz_eigen;
typedef struct kz_eigen_desc {
    int64_t n, r;
    int64_t ldr;          /* row stride of u / au: >= r, multiple of 4, zero padded, <= 384 */
    double beta;
    const kz_graph* op;   /* A (n x n) in the solve order */
    const double* u;      /* device n x ldr row-major */
    const double* au;     /* device n x ldr row-major, A U */
    const double* w;      /* device r x r row-major, (I - beta U'AU)^-1 */
    const double* a2u;    /* device n x ldr row-major, A^2 U; NULL: plain Galerkin start */
    const double* a3u;    /* device n x ldr row-major, A^3 U: two-term walk start (takes precedence) */
    const double* a4u;    /* device n x ldr row-major, A^4 U: three-term walk start (x0 += beta^3 A^3 e_q
                             by one more SpMM on the 2-walk counts; takes precedence) */
} kz_eigen_desc;
int kz_eigen_create(const kz_eigen_desc* d, kz_eigen** out);
int kz_eigen_destroy(kz_eigen* h);
size_t kz_eigen_workspace_bytes(const kz_eigen* h, int32_t b);
int kz_eigen_batch(const kz_eigen* h, const kz_cg_args* a, void* ws, size_t ws_bytes, void* stream);

/* ---- index build, host side (no device work) -----------------------------
 * Vertex-separator partition of a connected graph given as a host CSR
 * (int64 rowptr[n+1], colidx[nnz], symmetric, no self loops): the
 * reference's partition_vertex_separator (partition.py:178-248) with its
 * tie rules, so perm / bounds are identical to the reference's.
 * limit = PartitionConfig.resolved_part_size(n) (partition.py:40-45),
 * max_depth = max_recursion_depth.  perm[n] and bounds[n+1] are caller
 * allocated; bounds[0..*num_parts] are written. */
int kz_partition(int64_t n, const int64_t* rowptr, const int64_t* colidx, int64_t limit,
                 int64_t max_depth, int64_t* perm, int64_t* bounds, int64_t* num_parts,
                 int64_t* n1, int64_t* n2);
/* Greedy minimum-degree elimination order of one part (factor.py:31-55),
 * ties to the smallest index; local CSR of the part's internal edges. */
int kz_min_degree_order(int64_t m, const int64_t* rowptr, const int64_t* colidx, int64_t* order);
/* The orders of all parts in one call: part p is rows [bounds[p], bounds[p+1])
 * of the partition-ordered adjacency (global columns; entries leaving the
 * part are ignored); orders[bounds[p] + k] = k-th eliminated local index. */
int kz_min_degree_orders(int64_t nparts, const int64_t* bounds, const int64_t* rowptr,
                         const int64_t* colidx, int64_t* orders);

/* ---- vector helpers used by the generic cg() / lrc_pcg() drivers -------- */
/* out[j] = sum_i X[i,j]*Y[i,j] over b columns of length n (column-major);
 * the numpy `@` dots of solver.py:71-95 / 126-156.  The caller provides the
 * reduction scratch (kz_coldot_workspace_bytes), so calls on distinct
 * streams with distinct workspaces are reentrant. */
size_t kz_coldot_workspace_bytes(int64_t n, int32_t b);
int kz_coldot(int64_t n, int32_t b, const double* X, const double* Y, double* out, void* ws,
              size_t ws_bytes, void* stream);
/* Vector update of the generic cg() driver (solver.py:88-99) with the
 * products and the sum rounded separately, as numpy evaluates them:
 * op 0: out = a*x + b*y (y == NULL: out = a*x); op 1: out = x / a
 * (spectral_norm's v = w / ||w||, graph.py:289).  out may alias x or y. */
int kz_vec_op(int32_t op, int64_t n, double a, const double* x, double b, const double* y, double* out,
              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KATZB200_H */
