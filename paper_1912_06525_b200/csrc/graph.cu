// graph.cu -- operator handles (kz_graph) and the K1 SpMM entry point.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "spmm.cuh"
#ifndef KZ_EXPERIMENTS
#define KZ_EXPERIMENTS 0  // 1: build the experiment entry points (tools/k1_coldpass_proto.py)
#endif
#if KZ_EXPERIMENTS
#include "spmmcold.cuh"
#endif

namespace kz {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
void clear_error() { g_last_error.clear(); }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
static std::atomic<uint64_t> g_uid{0};
uint64_t next_uid() { return ++g_uid; }

// red zones of the workspaces carved by this thread since the last query
static thread_local std::vector<std::pair<const void*, size_t>> g_redzones;
void note_redzone(const void* base, size_t off) {
    if (g_redzones.size() < (1u << 20)) g_redzones.emplace_back(base, off);
}
void forget_redzones(const void* p0, const void* p1) {
    const char* a = static_cast<const char*>(p0);
    const char* b = static_cast<const char*>(p1);
    g_redzones.erase(std::remove_if(g_redzones.begin(), g_redzones.end(),
                                    [&](const std::pair<const void*, size_t>& z) {
                                        const char* q = static_cast<const char*>(z.first) + z.second;
                                        return q >= a && q < b;
                                    }),
                     g_redzones.end());
}

int num_sms() {
    static std::mutex mu;
    static std::vector<int> cache;  // per device ordinal
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 148;  // B200; only reached without a usable device
    }
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1, 0);
    if (cache[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 148;
        }
        cache[dev] = v;
    }
    return cache[dev];
}

// ---- K1 launch timing (kz_k1_timing / kz_k1_timing_read) ----
static std::atomic<bool> g_k1_timing{false};
static std::mutex g_k1_mu;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_k1_events;

bool k1_timing_on() { return g_k1_timing.load(std::memory_order_relaxed); }
void k1_timing_begin(cudaStream_t st, cudaEvent_t* e0) {
    *e0 = nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    if (cudaEventCreate(e0) != cudaSuccess) {
        cudaGetLastError();
        *e0 = nullptr;
        return;
    }
    cudaEventRecord(*e0, st);
}
void k1_timing_end(cudaStream_t st, cudaEvent_t e0) {
    if (!e0) return;
    cudaEvent_t e1 = nullptr;
    if (cudaEventCreate(&e1) != cudaSuccess) {
        cudaGetLastError();
        cudaEventDestroy(e0);
        return;
    }
    cudaEventRecord(e1, st);
    std::lock_guard<std::mutex> lock(g_k1_mu);
    g_k1_events.emplace_back(e0, e1);
}

}  // namespace kz

using namespace kz;

extern "C" const char* kz_last_error(void) { return g_last_error.c_str(); }
extern "C" long long kz_launch_count(void) { return g_launches.load(); }
extern "C" int kz_version(void) { return 1; }

extern "C" int kz_k1_timing(int enable) {
    std::lock_guard<std::mutex> lock(g_k1_mu);
    for (auto& p : g_k1_events) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    g_k1_events.clear();
    g_k1_timing.store(enable != 0);
    return KZ_OK;
}

extern "C" int kz_k1_timing_read(double* total_ms, long long* launches) {
    std::lock_guard<std::mutex> lock(g_k1_mu);
    double tot = 0.0;
    for (auto& p : g_k1_events) {
        KZ_CUDA(cudaEventSynchronize(p.second));
        float ms = 0.f;
        KZ_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = static_cast<long long>(g_k1_events.size());
    return KZ_OK;
}

extern "C" int kz_num_sms(void) { return num_sms(); }

extern "C" int kz_checked(void) { return KZ_CHECKED; }

extern "C" int64_t kz_checked_redzones(const void* ws, int64_t* offs, int64_t cap) {
    int64_t k = 0;
    for (const auto& z : g_redzones)
        if (z.first == ws) {
            if (offs && k < cap) offs[k] = static_cast<int64_t>(z.second);
            ++k;
        }
    g_redzones.clear();
    return k;
}

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
    cudaFree(g->vals);
    cudaFree(g->tasks);
    cudaFree(g->group_first);
    cudaFree(g->long_seg0);
    cudaFree(g->seg_range);
    delete g;
}

__global__ void check_cols_kernel(const int32_t* __restrict__ col, int64_t nnz, int32_t cols, int32_t* bad) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t c = col[i];
        if (c < 0 || c >= cols) atomicExch(bad, 1);
    }
}

// Column blocking of the long rows (see spmm.cuh).  For an operator whose
// gathered chunk (cols * 32 doubles) is far larger than L2, rows of degree >
// min_deg are cut by column block as well as by length, and those segments
// run block-major: while block k's segments run, the gathered slice of X is
// about slice_mb and stays L2-resident, so each of its rows is fetched from
// HBM about once per chunk instead of about once per gather.
struct SchedOpts {
    int nblocks = 1;             // 1: no column blocking (long rows = deg > kSegLen)
    int64_t min_deg = kSegLen;   // blocked: rows with deg > min_deg are long rows
    int interleave = 1;          // blocked: short-row tasks spread over the block phases
};

// Host schedule for K1 (see spmm.cuh): warp tasks in row order, then (column
// blocking) the long rows' segments block by block.  col is the host copy of
// the column indices; with nblocks > 1 each long row's entries are stably
// grouped by column block in place (this changes summation order only).
void build_schedule(const std::vector<int64_t>& rp, int64_t rows, int64_t cols, int32_t* col,
                    const SchedOpts& o, std::vector<int4>& tasks, std::vector<int32_t>& long_seg0,
                    std::vector<int2>& seg_range, std::vector<int32_t>& group_first, int32_t& max_deg) {
    std::vector<double> cost;
    int64_t s_open = -1, s_rows = 0;
    double s_cost = 0.0;
    auto close_s = [&](int64_t end) {
        if (s_open >= 0) {
            tasks.push_back(make_int4(static_cast<int>(s_open), static_cast<int>(end), TASK_S, 0));
            cost.push_back(s_cost);
            s_open = -1;
        }
    };
    const bool blocked = o.nblocks > 1 && col != nullptr && cols > 0;
    int32_t nlong = 0, nseg = 0;
    max_deg = 0;
    // granularity: aim for >= ~2 work units per resident warp of one chunk pass
    const double est_total = static_cast<double>(rp[rows]) + 4.0 * static_cast<double>(rows);
    const double unit = std::max(64.0, std::min(kGroupCost, est_total / (2.0 * num_sms() * kSpmmMinBlocks * kWarps)));
    // hub segments no longer than a work unit (at least 1,024): large
    // operators get kSegLen, small ones keep short segments so one hub row
    // does not become a serial tail
    const int64_t seglen = std::max<int64_t>(1024, std::min<int64_t>(kSegLen, static_cast<int64_t>(unit)));
    const int64_t min_deg = blocked ? std::min<int64_t>(std::max<int64_t>(o.min_deg, kMedDeg), seglen) : seglen;
    const int s_rows_max = unit >= 512.0 ? 32 : (unit >= 128.0 ? 8 : 4);
#ifndef KZ_K1_SCOST
#define KZ_K1_SCOST 256.0
#endif
    const double s_cost_max = std::min(KZ_K1_SCOST, unit);
    std::vector<int64_t> long_rows;  // blocked: rows deferred to the block phases
    for (int64_t i = 0; i < rows; ++i) {
        const int64_t d = rp[i + 1] - rp[i];
        max_deg = std::max<int32_t>(max_deg, static_cast<int32_t>(d));
        if (d <= kMedDeg) {
            if (s_open >= 0 && (s_rows >= s_rows_max || s_cost + d + 4 > s_cost_max)) close_s(i);
            if (s_open < 0) {
                s_open = i;
                s_rows = 0;
                s_cost = 0.0;
            }
            s_rows += 1;
            s_cost += d + 4.0;
        } else if (d <= min_deg) {
            close_s(i);
            tasks.push_back(make_int4(static_cast<int>(i), 0, TASK_M, 0));
            cost.push_back(d + 8.0);
        } else if (blocked) {
            close_s(i);
            long_rows.push_back(i);
        } else {
            close_s(i);
            long_seg0.push_back(nseg);
            int k = 0;
            for (int64_t p = rp[i]; p < rp[i + 1]; p += seglen, ++k) {
                const int64_t e = std::min<int64_t>(p + seglen, rp[i + 1]);
                tasks.push_back(make_int4(static_cast<int>(i), nlong, TASK_L, k));
                cost.push_back(static_cast<double>(e - p) + 8.0);
                seg_range.push_back(make_int2(static_cast<int>(p), static_cast<int>(e)));
            }
            nseg += k;
            ++nlong;
        }
    }
    close_s(rows);
    if (blocked) {
        // group each long row's entries by column block (stable counting
        // sort), then emit the segments block-major; a row's segments are
        // numbered in queue order, so its last segment (the combiner) is
        // dequeued last
        const int K = o.nblocks;
        const size_t nl = long_rows.size();
        std::vector<int64_t> bstart(nl * (K + 1));
        std::vector<int32_t> tmp;
        std::vector<int64_t> cnt(K + 1);
        auto block_of = [&](int32_t c) { return static_cast<int>((static_cast<int64_t>(c) * K) / cols); };
        for (size_t l = 0; l < nl; ++l) {
            const int64_t i = long_rows[l], b0 = rp[i], d = rp[i + 1] - b0;
            std::fill(cnt.begin(), cnt.end(), 0);
            for (int64_t p = 0; p < d; ++p) cnt[1 + block_of(col[b0 + p])] += 1;
            for (int k = 0; k < K; ++k) cnt[k + 1] += cnt[k];
            for (int k = 0; k <= K; ++k) bstart[l * (K + 1) + k] = b0 + cnt[k];
            tmp.resize(d);
            for (int64_t p = 0; p < d; ++p) {
                const int32_t c = col[b0 + p];
                tmp[cnt[block_of(c)]++] = c;
            }
            std::copy(tmp.begin(), tmp.end(), col + b0);
        }
        std::vector<int32_t> seg0(nl + 1, 0), next(nl, 0);
        for (size_t l = 0; l < nl; ++l) {
            int64_t ns = 0;
            for (int k = 0; k < K; ++k)
                ns += (bstart[l * (K + 1) + k + 1] - bstart[l * (K + 1) + k] + seglen - 1) / seglen;
            seg0[l + 1] = seg0[l] + static_cast<int32_t>(ns);
        }
        long_seg0.assign(seg0.begin(), seg0.end());
        seg_range.assign(seg0[nl], make_int2(0, 0));
        // short-row tasks: spread over the block phases (their HBM misses
        // overlap the L2-resident block phases) or all first
        std::vector<int4> stasks;
        std::vector<double> scost;
        stasks.swap(tasks);
        scost.swap(cost);
        const size_t nst = stasks.size();
        for (int k = 0; k < K; ++k) {
            const size_t a0 = o.interleave ? nst * k / K : (k == 0 ? 0 : nst);
            const size_t a1 = o.interleave ? nst * (k + 1) / K : nst;
            for (size_t t = a0; t < a1; ++t) {
                tasks.push_back(stasks[t]);
                cost.push_back(scost[t]);
            }
            for (size_t l = 0; l < nl; ++l) {
                const int64_t i = long_rows[l], e = bstart[l * (K + 1) + k + 1];
                for (int64_t p = bstart[l * (K + 1) + k]; p < e; p += seglen) {
                    const int kk = next[l]++;
                    const int64_t pe = std::min<int64_t>(p + seglen, e);
                    tasks.push_back(make_int4(static_cast<int>(i), static_cast<int>(l), TASK_L, kk));
                    cost.push_back(static_cast<double>(pe - p) + 8.0);
                    seg_range[seg0[l] + kk] = make_int2(static_cast<int>(p), static_cast<int>(pe));
                }
            }
        }
    } else {
        long_seg0.push_back(nseg);
    }
    // warp work units: consecutive tasks up to ~kGroupCost neighbour-equivalents
    // (at most kGroupTasks tasks); a hub segment is a unit of its own
    group_first.push_back(0);
    double acc = 0.0;
    int cnt = 0;
    for (size_t t = 0; t < tasks.size(); ++t) {
        if (cnt > 0 && (acc + cost[t] > unit || cnt >= kGroupTasks)) {
            group_first.push_back(static_cast<int32_t>(t));
            acc = 0.0;
            cnt = 0;
        }
        acc += cost[t];
        ++cnt;
    }
    if (group_first.back() != static_cast<int32_t>(tasks.size()))
        group_first.push_back(static_cast<int32_t>(tasks.size()));
}

}  // namespace

namespace kz {

// Creates an operator handle; vals (host or device, nnz doubles) makes it a
// weighted operator (used for the block-diagonal M11^-1 of the LRC path).
int create_graph(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rowptr,
                 const int32_t* colidx, const double* vals, kz_graph** out) {
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
    g->uid = next_uid();
    g->rows = rows;
    g->cols = cols;
    g->nnz = nnz;
    std::vector<int32_t> rp32(rows + 1);
    for (int64_t i = 0; i <= rows; ++i) rp32[i] = static_cast<int32_t>(rp[i]);
    // column blocking (spmm.cuh): binary operators whose C = 32 chunk of X
    // exceeds ~4 slices; KZ_K1_SLICE_MB = 0 turns it off
    SchedOpts so;
    std::vector<int32_t> hcol;
    {
        const char* e = std::getenv("KZ_K1_SLICE_MB");
        const double slice_mb = e ? std::atof(e) : kColBlockSliceMB;
        const double chunk_mb = static_cast<double>(cols) * 32.0 * 8.0 / 1e6;
        if (!vals && slice_mb > 0.0 && chunk_mb > 4.0 * slice_mb && nnz > 0) {
            so.nblocks = static_cast<int>(std::ceil(chunk_mb / slice_mb));
            if (const char* m = std::getenv("KZ_K1_MINDEG")) so.min_deg = std::atoll(m);
            else so.min_deg = kColBlockMinDeg;
            if (const char* m = std::getenv("KZ_K1_INTERLEAVE")) so.interleave = std::atoi(m);
            hcol.resize(nnz);
            cudaError_t ce = cudaMemcpy(hcol.data(), colidx, sizeof(int32_t) * nnz, cudaMemcpyDefault);
            if (ce != cudaSuccess) return fail(KZ_ECUDA, std::string("colidx copy: ") + cudaGetErrorString(ce));
            for (int64_t p = 0; p < nnz; ++p)
                if (hcol[p] < 0 || hcol[p] >= cols) return fail(KZ_EARG, "column index out of range [0, cols)");
        }
    }
    std::vector<int4> tasks;
    std::vector<int32_t> long_seg0, group_first;
    std::vector<int2> seg_range;
    build_schedule(rp, rows, cols, hcol.empty() ? nullptr : hcol.data(), so, tasks, long_seg0, seg_range,
                   group_first, g->max_deg);
    g->nblocks = hcol.empty() ? 1 : so.nblocks;
    if (!hcol.empty()) colidx = hcol.data();  // long rows regrouped by column block
    g->ngroups = static_cast<int32_t>(group_first.size()) - 1;
    g->ntasks = static_cast<int32_t>(tasks.size());
    g->nlong = static_cast<int32_t>(long_seg0.size()) - 1;
    g->nseg = long_seg0.back();

    int st = KZ_OK;
    if ((st = upload(&g->rowptr, rp32.data(), rows + 1)) ||
        (st = upload(&g->colidx, static_cast<const int32_t*>(nullptr), nnz)) ||
        (st = upload(&g->tasks, tasks.data(), tasks.size())) ||
        (st = upload(&g->group_first, group_first.data(), group_first.size())) ||
        (st = upload(&g->long_seg0, long_seg0.data(), long_seg0.size())) ||
        (st = upload(&g->seg_range, seg_range.data(), seg_range.size())) ||
        (vals && (st = upload(&g->vals, static_cast<const double*>(nullptr), nnz)))) {
        free_graph(g);
        return st;
    }
    if (nnz > 0) {
        cudaError_t e = cudaMemcpy(g->colidx, colidx, sizeof(int32_t) * nnz, cudaMemcpyDefault);
        if (e == cudaSuccess && vals) e = cudaMemcpy(g->vals, vals, sizeof(double) * nnz, cudaMemcpyDefault);
        if (e != cudaSuccess) {
            free_graph(g);
            return fail(KZ_ECUDA, std::string("CSR copy: ") + cudaGetErrorString(e));
        }
        // every column index must address a row of Xg: checked once on the
        // device so a bad operator fails here, not as an illegal access later
        int32_t* bad = nullptr;
        if (cudaMalloc(&bad, sizeof(int32_t)) != cudaSuccess) {
            free_graph(g);
            return fail(KZ_EOOM, "validation flag");
        }
        cudaMemset(bad, 0, sizeof(int32_t));
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(4 * max_ctas_per_chunk(), (nnz + 255) / 256));
        check_cols_kernel<<<grid, 256>>>(g->colidx, nnz, static_cast<int32_t>(cols), bad);
        note_launch();
        int32_t h = 0;
        e = cudaMemcpy(&h, bad, sizeof(int32_t), cudaMemcpyDeviceToHost);
        cudaFree(bad);
        if (e != cudaSuccess || h) {
            free_graph(g);
            return fail(e != cudaSuccess ? KZ_ECUDA : KZ_EARG, "column index out of range [0, cols)");
        }
    }
    *out = g;
    return KZ_OK;
}

}  // namespace kz

extern "C" int kz_graph_create(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rowptr,
                               const int32_t* colidx, kz_graph** out) {
    return create_graph(rows, cols, nnz, rowptr, colidx, nullptr, out);
}

extern "C" int kz_graph_create_weighted(int64_t rows, int64_t cols, int64_t nnz, const int64_t* rowptr,
                                        const int32_t* colidx, const double* vals, kz_graph** out) {
    if (!vals && nnz > 0) return fail(KZ_EARG, "NULL values");
    return create_graph(rows, cols, nnz, rowptr, colidx, vals, out);
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
    if (nitems) *nitems = g->nseg;
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
    // the column-dot reduction maps one lane to one column of the chunk
    if (dots && chunk > 32) return fail(KZ_EARG, "dots need a chunk width of at most 32");
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

#if KZ_EXPERIMENTS
// Experiment entry (tools/k1_coldpass_proto.py): one launch of the cold pass
// on caller-built streams (all device pointers); P[chunk][ng*slots][32].
extern "C" int kz_spmm_cold_debug(const uint32_t* ent, const int32_t* segoff, const uint8_t* nslot,
                                  int32_t ng, int32_t nslabs, int64_t cols, int32_t b, const double* X,
                                  double* P, int32_t* done, void* stream) {
    clear_error();
    if (!ent || !segoff || !nslot || !X || !P || !done || ng < 1 || ng % (kThreads / 8) != 0 || b % 32 != 0)
        return fail(KZ_EARG, "bad cold-pass arguments");
    const int grid = ng / (kThreads / 8);
    if (grid > num_sms() * cold_ctas_per_sm()) return fail(KZ_EARG, "cold-pass grid is not co-resident");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    KZ_CUDA(cudaMemsetAsync(done, 0, sizeof(int32_t) * (b / 32) * nslabs, st));
    ColdArgs a{};
    a.ent = ent;
    a.segoff = segoff;
    a.nslot = nslot;
    a.ng = ng;
    a.nslabs = nslabs;
    a.nchunks = b / 32;
    a.cols = static_cast<int32_t>(cols);
    a.Xg = X;
    a.ldxg = cols * 32;
    a.P = P;
    a.done = done;
    {
        const char* e = std::getenv("KZ_COLD_THROTTLE");
        a.throttle = e ? std::atoi(e) : 1;
    }
    return launch_spmm_cold(a, grid, st);
}

extern "C" int kz_cold_slots(void) { return kColdSlots; }
#endif  // KZ_EXPERIMENTS
