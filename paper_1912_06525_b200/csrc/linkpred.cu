// linkpred.cu -- K7: anchor-profile gather and the Pearson rerank of
// sparse_katz (linkpred.py:165-207), batched over queries.
//
// profiles[j][t][c]: proximity of candidate c of query j to profile node t
// (t = 0 is the query, t = 1..T its anchors).  The rerank is computed per
// query by one CTA: centred Pearson correlation of each candidate's profile
// with the query's reference profile (0 when either has zero variance,
// clipped to [-1, 1]; linkpred.py:197-204), then a bitonic sort by
// (corr desc, Katz score desc, id asc) -- lexsort((top, -score, -corr)).
#include <algorithm>

#include "spmm.cuh"

using namespace kz;

namespace {

// candidates one CTA sorts in shared memory (20 bytes each, dynamic smem)
constexpr int kMaxCand = 8192;

// out[j][slot][c] = S[src][top[j][c]] for each triple (src, j, slot)
__global__ void profile_gather_kernel(const double* __restrict__ S, int64_t n,
                                      const int64_t* __restrict__ trip, int ntrip,
                                      const int64_t* __restrict__ top, const int32_t* __restrict__ count,
                                      int s, double* __restrict__ prof, int T1) {
    for (int t = blockIdx.x; t < ntrip; t += gridDim.x) {
        const int64_t src = trip[3 * t], j = trip[3 * t + 1], slot = trip[3 * t + 2];
        const int m = count[j];
        KZ_DCHECK(m >= 0 && m <= s && slot >= 0 && slot < T1);
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
            const int64_t id = top[j * s + c];
            KZ_DCHECK(id >= 0 && id < n);
            prof[(j * T1 + slot) * s + c] = S[src * n + id];
        }
    }
}

__global__ void __launch_bounds__(kThreads)
    pearson_rerank_kernel(const double* __restrict__ prof, const double* __restrict__ ref,
                          const int64_t* __restrict__ top, const double* __restrict__ top_score,
                          const int32_t* __restrict__ count, int T1, int s,
                          double* __restrict__ corr_out, int64_t* __restrict__ order_out) {
    const int j = blockIdx.x;
    const int m = count[j];
    int P = 1;
    while (P < m) P <<= 1;
    extern __shared__ double dsm[];
    double* sc = dsm;        // [P]
    double* ss = dsm + P;    // [P]
    int* si = reinterpret_cast<int*>(dsm + 2 * P);  // [P]
    __shared__ double s_rm, s_sr;
    const double* r = ref + static_cast<size_t>(j) * T1;
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int t = 0; t < T1; ++t) sum += r[t];
        const double rm = sum / T1;
        double ss2 = 0.0;
        for (int t = 0; t < T1; ++t) ss2 += (r[t] - rm) * (r[t] - rm);
        s_rm = rm;
        s_sr = sqrt(ss2);
    }
    __syncthreads();
    const double rm = s_rm, sr = s_sr;
    const double* pj = prof + static_cast<size_t>(j) * T1 * s;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
        double sum = 0.0;
        for (int t = 0; t < T1; ++t) sum += pj[t * s + c];
        const double pm = sum / T1;
        double sp2 = 0.0, dot = 0.0;
        for (int t = 0; t < T1; ++t) {
            const double d = pj[t * s + c] - pm;
            sp2 += d * d;
            dot += (r[t] - rm) * d;
        }
        const double sp = sqrt(sp2);
        double cr = 0.0;
        if (sp > 0.0 && sr > 0.0) cr = fmin(1.0, fmax(-1.0, dot / (sr * sp)));
        corr_out[static_cast<size_t>(j) * s + c] = cr;
        if (order_out) {  // the shared-memory sort keys exist only when ordering
            sc[c] = cr;
            ss[c] = top_score[static_cast<size_t>(j) * s + c];
            si[c] = c;
        }
    }
    if (!order_out) return;  // correlations only (the caller orders them)
    for (int c = m + threadIdx.x; c < P; c += blockDim.x) {
        sc[c] = -INFINITY;
        ss[c] = -INFINITY;
        si[c] = 0x7fffffff;
    }
    __syncthreads();
    const int64_t* tj = top + static_cast<size_t>(j) * s;
    auto before = [&](int a, int b2) {  // a ranks before b2
        if (sc[a] != sc[b2]) return sc[a] > sc[b2];
        if (ss[a] != ss[b2]) return ss[a] > ss[b2];
        const int64_t ia = si[a] < m ? tj[si[a]] : INT64_MAX;
        const int64_t ib = si[b2] < m ? tj[si[b2]] : INT64_MAX;
        return ia < ib;
    };
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int partner = i ^ stride;
                if (partner > i) {
                    const bool desc = (i & size) == 0;
                    const bool swap = desc ? before(partner, i) : before(i, partner);
                    if (swap) {
                        double t = sc[i]; sc[i] = sc[partner]; sc[partner] = t;
                        t = ss[i]; ss[i] = ss[partner]; ss[partner] = t;
                        const int u = si[i]; si[i] = si[partner]; si[partner] = u;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int c = threadIdx.x; c < m; c += blockDim.x) order_out[static_cast<size_t>(j) * s + c] = si[c];
}

}  // namespace

extern "C" int kz_profile_gather(const double* S, int64_t n, int32_t ntrip, const int64_t* trip,
                                 const int64_t* top_ids, const int32_t* counts, int32_t s,
                                 double* profiles, int32_t T1, void* stream) {
    clear_error();
    if (ntrip < 0 || !S || (ntrip > 0 && !trip) || !top_ids || !counts || !profiles || s < 1 || T1 < 1)
        return fail(KZ_EARG, "bad profile gather arguments");
    if (ntrip == 0) return KZ_OK;
    const int grid = std::min(ntrip, max_ctas_per_chunk() * 2);
    profile_gather_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(S, n, trip, ntrip, top_ids, counts, s, profiles, T1); ::kz::note_launch();
    KZ_LAUNCH_CHECK();
    return KZ_OK;
}

extern "C" int kz_pearson_rerank(const double* profiles, const double* ref, const int64_t* top_ids,
                                 const double* top_scores, const int32_t* counts, int32_t b,
                                 int32_t T1, int32_t s, double* corr_out, int64_t* order_out,
                                 void* stream) {
    clear_error();
    if (b < 1 || T1 < 2 || s < 1 || !profiles || !ref || !top_ids || !top_scores || !counts || !corr_out)
        return fail(KZ_EARG, "bad rerank arguments");
    if (order_out && s > kMaxCand)
        return fail(KZ_EARG, "rerank sorts at most 8192 candidates per query (pass order_out = NULL for correlations only)");
    int P = 1;
    while (P < std::min(s, kMaxCand)) P <<= 1;
    const size_t smem = order_out ? static_cast<size_t>(P) * 20 : 0;
    KZ_CUDA(cudaFuncSetAttribute(pearson_rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(8192 * 20)));
    pearson_rerank_kernel<<<b, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(
        profiles, ref, top_ids, top_scores, counts, T1, s, corr_out, order_out); ::kz::note_launch();
    KZ_LAUNCH_CHECK();
    return KZ_OK;
}
