// graph.cu -- operator handles (kz_graph) and the K1 SpMM entry point.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>

#include "spmm.cuh"

namespace kz {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
void clear_error() { g_last_error.clear(); }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace kz

using namespace kz;

extern "C" const char* kz_last_error(void) { return g_last_error.c_str(); }
extern "C" long long kz_launch_count(void) { return g_launches.load(); }
extern "C" int kz_version(void) { return 1; }

namespace {

template <class T>
int upload(T** dst, const T* src, size_t count) {
    *dst = nullptr;
    if (count == 0) count = 1;  // keep a valid pointer for empty arrays
    KZ_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), count * sizeof(T)));
    if (src) KZ_CUDA(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyDefault));
    return KZ_OK;
}

void free_graph(kz_graph* g) {
    if (!g) return;
    cudaFree(g->rowptr);
    cudaFree(g->colidx);
    cudaFree(g->long_rows);
    cudaFree(g->long_first);
    cudaFree(g->item_lrow);
    cudaFree(g->cta_rows);
    cudaFree(g->cta_long);
    delete g;
}

}  // namespace

// Builds the SpMM schedule on the host from rowptr (rows+1 ints): long-row
// segments and cost-balanced row ranges per CTA.
extern "C" int kz_graph_create(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rowptr,
                               const int32_t* colidx, kz_graph** out) {
    clear_error();
    if (!out) return fail(KZ_EARG, "out is NULL");
    *out = nullptr;
    if (rows < 1 || cols < 0 || nnz < 0) return fail(KZ_EARG, "bad operator shape");
    if (nnz >= (int64_t(1) << 31) || rows >= (int64_t(1) << 31) - 1 ||
        cols >= (int64_t(1) << 31) - 1)
        return fail(KZ_EARG, "operator too large for int32 indices");
    if (!rowptr || (nnz > 0 && !colidx)) return fail(KZ_EARG, "NULL CSR arrays");

    std::vector<int64_t> rp(rows + 1);
    {
        cudaError_t e = cudaMemcpy(rp.data(), rowptr, sizeof(int64_t) * (rows + 1), cudaMemcpyDefault);
        if (e != cudaSuccess) return fail(KZ_ECUDA, std::string("rowptr copy: ") + cudaGetErrorString(e));
    }
    if (rp[0] != 0 || rp[rows] != nnz) return fail(KZ_EARG, "rowptr does not span [0, nnz]");
    for (int64_t i = 0; i < rows; ++i)
        if (rp[i + 1] < rp[i]) return fail(KZ_EARG, "rowptr not monotone");

    auto* g = new kz_graph();
    g->rows = rows;
    g->cols = cols;
    g->nnz = nnz;
    const int64_t seg = g->seg;

    std::vector<int32_t> rp32(rows + 1), long_rows, long_first, item_lrow;
    std::vector<double> cost_prefix(rows + 1, 0.0);
    int32_t max_deg = 0;
    for (int64_t i = 0; i < rows; ++i) {
        rp32[i] = static_cast<int32_t>(rp[i]);
        const int64_t d = rp[i + 1] - rp[i];
        max_deg = std::max<int32_t>(max_deg, static_cast<int32_t>(d));
        double c;
        if (d > seg) {
            const int64_t ns = (d + seg - 1) / seg;
            long_first.push_back(static_cast<int32_t>(item_lrow.size()));
            for (int64_t s = 0; s < ns; ++s) item_lrow.push_back(static_cast<int32_t>(long_rows.size()));
            long_rows.push_back(static_cast<int32_t>(i));
            c = 8.0 + static_cast<double>(ns);
        } else {
            c = 4.0 + static_cast<double>(d);
        }
        cost_prefix[i + 1] = cost_prefix[i] + c;
    }
    rp32[rows] = static_cast<int32_t>(rp[rows]);
    long_first.push_back(static_cast<int32_t>(item_lrow.size()));
    g->max_deg = max_deg;
    g->nlong = static_cast<int32_t>(long_rows.size());
    g->nitems = static_cast<int32_t>(item_lrow.size());

    // row-range CTAs: about 1 KB-of-index of work each, at most one resident wave per chunk
    const double total = cost_prefix[rows];
    int64_t nshort = static_cast<int64_t>(total / 512.0) + 1;
    nshort = std::max<int64_t>(1, std::min<int64_t>(nshort, kMaxCtasPerChunk));
    nshort = std::min<int64_t>(nshort, rows);
    std::vector<int32_t> cta_rows(nshort + 1), cta_long(nshort + 1);
    cta_rows[0] = 0;
    for (int64_t p = 1; p < nshort; ++p) {
        const double target = total * static_cast<double>(p) / static_cast<double>(nshort);
        int64_t r = std::lower_bound(cost_prefix.begin(), cost_prefix.end(), target) - cost_prefix.begin();
        r = std::max<int64_t>(r, cta_rows[p - 1]);
        r = std::min<int64_t>(r, rows);
        cta_rows[p] = static_cast<int32_t>(r);
    }
    cta_rows[nshort] = static_cast<int32_t>(rows);
    for (int64_t p = 0; p <= nshort; ++p)
        cta_long[p] = static_cast<int32_t>(
            std::lower_bound(long_rows.begin(), long_rows.end(), cta_rows[p]) - long_rows.begin());
    g->nshort = static_cast<int32_t>(nshort);
    g->nlongcta = g->nitems == 0
                      ? 0
                      : static_cast<int32_t>(std::min<int64_t>(
                            kMaxCtasPerChunk, std::max<int64_t>(1, (g->nitems + 4 * kWarps - 1) / (4 * kWarps))));

    int st = KZ_OK;
    if ((st = upload(&g->rowptr, rp32.data(), rows + 1)) ||
        (st = upload(&g->colidx, static_cast<const int32_t*>(nullptr), nnz)) ||
        (st = upload(&g->long_rows, long_rows.data(), long_rows.size())) ||
        (st = upload(&g->long_first, long_first.data(), long_first.size())) ||
        (st = upload(&g->item_lrow, item_lrow.data(), item_lrow.size())) ||
        (st = upload(&g->cta_rows, cta_rows.data(), cta_rows.size())) ||
        (st = upload(&g->cta_long, cta_long.data(), cta_long.size()))) {
        free_graph(g);
        return st;
    }
    if (nnz > 0) {
        cudaError_t e = cudaMemcpy(g->colidx, colidx, sizeof(int32_t) * nnz, cudaMemcpyDefault);
        if (e != cudaSuccess) {
            free_graph(g);
            return fail(KZ_ECUDA, std::string("colidx copy: ") + cudaGetErrorString(e));
        }
    }
    *out = g;
    return KZ_OK;
}

extern "C" int kz_graph_destroy(kz_graph* g) {
    free_graph(g);
    return KZ_OK;
}

extern "C" int kz_graph_info(const kz_graph* g, int64_t* rows, int64_t* cols, int64_t* nnz,
                             int64_t* nlong, int64_t* nitems) {
    if (!g) return fail(KZ_EARG, "NULL graph");
    if (rows) *rows = g->rows;
    if (cols) *cols = g->cols;
    if (nnz) *nnz = g->nnz;
    if (nlong) *nlong = g->nlong;
    if (nitems) *nitems = g->nitems;
    return KZ_OK;
}

extern "C" size_t kz_spmm_workspace_bytes(const kz_graph* g, int32_t b, int32_t chunk) {
    if (!g || b < 1 || !chunk_ok(chunk)) return 0;
    const int nchunks = (b + chunk - 1) / chunk;
    Carver cv(nullptr, 0);
    SpmmScratch s;
    carve_spmm_scratch(cv, g, nchunks, chunk, s);
    return cv.off + 256;
}

extern "C" int kz_spmm(const kz_graph* g, int32_t b, int32_t chunk, const double* Xg,
                       const double* Xs, const double* Z, double* Y, double s0, double s1,
                       double s2, const double* D, double* dots, void* ws, size_t ws_bytes,
                       void* stream) {
    clear_error();
    if (!g) return fail(KZ_EARG, "NULL graph");
    if (b < 1 || !chunk_ok(chunk) || b % chunk != 0)
        return fail(KZ_EARG, "b must be a positive multiple of the chunk width (1,2,4,...,32)");
    if (!Xg || !Y) return fail(KZ_EARG, "NULL X or Y");
    if (dots && !D && !Xs) return fail(KZ_EARG, "dots need D or Xs");
    if (Xs && g->rows != g->cols) {
        // allowed: Xs simply has `rows` rows
    }
    const int nchunks = b / chunk;
    if (!ws || ws_bytes < kz_spmm_workspace_bytes(g, b, chunk))
        return fail(KZ_EARG, "workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver cv(ws, ws_bytes);
    SpmmScratch s;
    carve_spmm_scratch(cv, g, nchunks, chunk, s);
    int rc = zero_spmm_counters(g, nchunks, s, st);
    if (rc) return rc;
    SpmmArgs a = make_spmm_args(g, s);
    a.Xg = Xg;
    a.Xs = Xs;
    a.Z = Z;
    a.Y = Y;
    a.D = D;
    a.s0 = s0;
    a.s1 = Xs ? s1 : 0.0;
    a.s2 = s2;
    a.chunk_active = nullptr;
    a.want_dot = dots ? 1 : 0;
    a.hook.mode = 0;
    a.hook.b = b;
    a.hook.dots_out = dots;
    return launch_spmm(g, chunk, nchunks, a, st);
}
