// topk.cu -- K4: batched masked top-k by (score desc, id asc).
//
// Mirrors _candidate_order (linkpred.py:145-152): the query and its
// neighbours are removed, the rest ordered by lexsort((id, -score)), and the
// first k kept; and the anchor choice (linkpred.py:186-188), which only
// removes the query.
//
// Each element is a unique 96-bit composite key K = (score bits << 32) |
// (~id): scores are >= 0 after the clamp, so their IEEE bits order like the
// values, and ~id makes smaller ids rank higher among equal scores.  A
// radix select over 12-bit digits of K (most significant first) narrows the
// pivot range until everything at or above it fits a CAP-sized candidate
// buffer; masked ids are subtracted from the digit histograms by walking the
// (short) mask list instead of testing every element.  One final pass
// collects the candidates and one CTA per column bitonic-sorts them.  Every
// round is a fixed launch sequence (no host synchronisation); columns that
// finished early make the later rounds no-ops.
#include <algorithm>

#include "spmm.cuh"

using namespace kz;

namespace {

constexpr int kDigit = 12;
constexpr int kBins = 1 << kDigit;
constexpr int kCap = 4096;
constexpr int kRounds = 8;  // 96 bits / 12

struct ColState {
    unsigned long long phi;  // prefix: score bits
    unsigned int plo;        // prefix: ~id bits
    int shift;               // unresolved low bits of K
    int need;                // still to take from the pivot range
    int above;               // certain members above the pivot range
    int done;
    int ncand;
    int pad;
};

__device__ __forceinline__ unsigned long long score_key(double v) {
    return v > 0.0 ? static_cast<unsigned long long>(__double_as_longlong(v)) : 0ull;
}

// (K >> s) compared with (P >> s): returns -1, 0, +1
__device__ __forceinline__ int cmp_prefix(unsigned long long hi, unsigned int lo,
                                          const ColState& c, int s) {
    if (s >= 96) return 0;
    if (s >= 32) {
        const int t = s - 32;
        const unsigned long long a = hi >> t, b = c.phi >> t;
        return a == b ? 0 : (a > b ? 1 : -1);
    }
    if (hi != c.phi) return hi > c.phi ? 1 : -1;
    const unsigned int a = lo >> s, b = c.plo >> s;
    return a == b ? 0 : (a > b ? 1 : -1);
}

__device__ __forceinline__ int digit_of(unsigned long long hi, unsigned int lo, int ns) {
    if (ns >= 32) return static_cast<int>((hi >> (ns - 32)) & (kBins - 1));
    const unsigned long long v = (static_cast<unsigned long long>(lo) >> ns) | (hi << (32 - ns));
    return static_cast<int>(v & (kBins - 1));
}

struct MaskRef {
    const int32_t* rowptr;  // mask graph CSR (may be null)
    const int32_t* colidx;
    const int64_t* rows;    // device [b], -1 = none
    const int64_t* self;    // device [b], -1 = none
    // exclusive upper bound on the key (score, id) per column: elements at or
    // above (bval[j], bid[j]) are left out -- the continuation pass of a
    // top-k larger than one candidate buffer (bid[j] < 0 = no bound)
    const double* bval;     // device [b] or null
    const int64_t* bid;     // device [b] or null
};

__device__ __forceinline__ bool above_bound(const MaskRef& m, int j, unsigned long long hi, unsigned int lo) {
    if (!m.bid) return false;
    const int64_t id = m.bid[j];
    if (id < 0) return false;
    const unsigned long long bhi = score_key(m.bval[j]);
    const unsigned int blo = ~static_cast<unsigned int>(id);
    return hi > bhi || (hi == bhi && lo >= blo);
}

__device__ __forceinline__ bool is_masked(const MaskRef& m, int j, int64_t id) {
    if (m.self && m.self[j] == id) return true;
    if (!m.rowptr || !m.rows) return false;
    const int64_t r = m.rows[j];
    if (r < 0) return false;
    int lo = m.rowptr[r], hi = m.rowptr[r + 1];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int v = m.colidx[mid];
        if (v == id) return true;
        if (v < id) lo = mid + 1;
        else hi = mid;
    }
    return false;
}

__global__ void topk_init_kernel(ColState* cs, int b, int64_t n, int k) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= b) return;
    ColState c{};
    c.shift = 96;
    c.need = static_cast<int>((k < n ? (int64_t)k : n));
    c.done = 0;
    cs[j] = c;
}

// per-column histogram of the next digit among elements matching the prefix
__global__ void __launch_bounds__(kThreads)
    topk_hist_kernel(const double* __restrict__ scores, int64_t n, int slices,
                     const ColState* __restrict__ cs, unsigned int* __restrict__ hist, MaskRef m) {
    const int j = blockIdx.x / slices, sl = blockIdx.x % slices;
    const ColState c = cs[j];
    if (c.done) return;
    __shared__ unsigned int h[kBins];
    for (int i = threadIdx.x; i < kBins; i += kThreads) h[i] = 0;
    __syncthreads();
    const int ns = max(c.shift - kDigit, 0);
    const double* col = scores + static_cast<size_t>(j) * n;
    const int64_t per = (n + slices - 1) / slices;
    const int64_t i0 = sl * per, i1 = (n < i0 + per ? n : i0 + per);
    // 4 loads in flight per thread: the scan streams the whole score block
    for (int64_t ib = i0 + threadIdx.x; ib < i1; ib += 4 * kThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = ib + static_cast<int64_t>(u) * kThreads;
            v[u] = i < i1 ? col[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = ib + static_cast<int64_t>(u) * kThreads;
            if (i >= i1) break;
            const unsigned long long hi = score_key(v[u]);
            const unsigned int lo = ~static_cast<unsigned int>(i);
            if (cmp_prefix(hi, lo, c, c.shift) == 0 && !above_bound(m, j, hi, lo)) atomicAdd(&h[digit_of(hi, lo, ns)], 1u);
        }
    }
    __syncthreads();
    unsigned int* gh = hist + static_cast<size_t>(j) * kBins;
    for (int i = threadIdx.x; i < kBins; i += kThreads)
        if (h[i]) atomicAdd(gh + i, h[i]);
}

// remove masked ids from the histogram (one CTA per column)
__global__ void topk_mask_kernel(const double* __restrict__ scores, int64_t n,
                                 const ColState* __restrict__ cs, unsigned int* __restrict__ hist,
                                 MaskRef m) {
    const int j = blockIdx.x;
    const ColState c = cs[j];
    if (c.done) return;
    const int ns = max(c.shift - kDigit, 0);
    const double* col = scores + static_cast<size_t>(j) * n;
    unsigned int* gh = hist + static_cast<size_t>(j) * kBins;
    auto visit = [&](int64_t id) {
        const unsigned long long hi = score_key(col[id]);
        const unsigned int lo = ~static_cast<unsigned int>(id);
        if (cmp_prefix(hi, lo, c, c.shift) == 0 && !above_bound(m, j, hi, lo)) atomicSub(gh + digit_of(hi, lo, ns), 1u);
    };
    const int64_t self = m.self ? m.self[j] : -1;
    if (threadIdx.x == 0 && self >= 0) visit(self);
    if (m.rowptr && m.rows && m.rows[j] >= 0) {
        const int64_t r = m.rows[j];
        for (int e = m.rowptr[r] + threadIdx.x; e < m.rowptr[r + 1]; e += blockDim.x) {
            const int64_t id = m.colidx[e];
            if (id != self) visit(id);
        }
    }
}

// pick the pivot digit, update the column state, clear the histogram
__global__ void __launch_bounds__(kThreads) topk_select_kernel(ColState* cs, unsigned int* hist) {
    const int j = blockIdx.x;
    __shared__ unsigned int part[kThreads];
    __shared__ int s_bin, s_cum;
    ColState c = cs[j];
    if (c.done) return;
    unsigned int* gh = hist + static_cast<size_t>(j) * kBins;
    constexpr int PB = kBins / kThreads;  // bins per thread
    // thread t owns bins [t*PB, t*PB+PB); suffix sums from the top bin down
    unsigned int loc = 0;
    for (int i = 0; i < PB; ++i) loc += gh[threadIdx.x * PB + i];
    part[threadIdx.x] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int cum = 0;
        int bin = -1;
        for (int t = kThreads - 1; t >= 0 && bin < 0; --t) {
            if (cum + part[t] >= static_cast<unsigned int>(c.need)) {
                for (int i = PB - 1; i >= 0; --i) {
                    const unsigned int hv = gh[t * PB + i];
                    if (cum + hv >= static_cast<unsigned int>(c.need)) {
                        bin = t * PB + i;
                        break;
                    }
                    cum += hv;
                }
            } else {
                cum += part[t];
            }
        }
        s_bin = bin;
        s_cum = static_cast<int>(cum);
    }
    __syncthreads();
    const int bin = s_bin;
    if (threadIdx.x == 0) {
        if (bin < 0) {
            // fewer unmasked elements than needed in range: take them all
            c.done = 1;
        } else {
            const int ns = max(c.shift - kDigit, 0);
            const unsigned int pivot = gh[bin];
            c.above += s_cum;
            c.need -= s_cum;
            if (ns >= 32) {
                c.phi |= static_cast<unsigned long long>(bin) << (ns - 32);
            } else {
                // digit straddles or lies in the id word
                const unsigned long long v = static_cast<unsigned long long>(bin) << ns;  // bits of K
                c.plo |= static_cast<unsigned int>(v & 0xffffffffull);
                c.phi |= v >> 32;
            }
            c.shift = ns;
            if (c.above + static_cast<int>(pivot) <= kCap || ns == 0) c.done = 1;
        }
        cs[j] = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kBins; i += kThreads) gh[i] = 0;
}

// gather every unmasked element at or above the pivot range
__global__ void __launch_bounds__(kThreads)
    topk_collect_kernel(const double* __restrict__ scores, int64_t n, int slices, ColState* cs,
                        unsigned long long* __restrict__ ckey, int* __restrict__ cid, MaskRef m) {
    const int j = blockIdx.x / slices, sl = blockIdx.x % slices;
    const ColState c = cs[j];
    const double* col = scores + static_cast<size_t>(j) * n;
    const int64_t per = (n + slices - 1) / slices;
    const int64_t i0 = sl * per, i1 = (n < i0 + per ? n : i0 + per);
    for (int64_t ib = i0 + threadIdx.x; ib < i1; ib += 4 * kThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = ib + static_cast<int64_t>(u) * kThreads;
            v[u] = i < i1 ? col[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = ib + static_cast<int64_t>(u) * kThreads;
            if (i >= i1) break;
            const unsigned long long hi = score_key(v[u]);
            const unsigned int lo = ~static_cast<unsigned int>(i);
            if (cmp_prefix(hi, lo, c, c.shift) >= 0 && !above_bound(m, j, hi, lo) && !is_masked(m, j, i)) {
                const int pos = atomicAdd(&cs[j].ncand, 1);
                if (pos < kCap) {
                    ckey[static_cast<size_t>(j) * kCap + pos] = hi;
                    cid[static_cast<size_t>(j) * kCap + pos] = static_cast<int>(i);
                }
            }
        }
    }
}

// bitonic sort of the candidates, descending by (score, -id); emit top k
__global__ void __launch_bounds__(kThreads)
    topk_sort_kernel(const ColState* __restrict__ cs, const unsigned long long* __restrict__ ckey,
                     const int* __restrict__ cid, int k, int64_t* __restrict__ ids_out,
                     double* __restrict__ vals_out, int32_t* __restrict__ count_out) {
    const int j = blockIdx.x;
    __shared__ unsigned long long sk[kCap];
    __shared__ int si[kCap];
    const int m = min(cs[j].ncand, kCap);
    int P = 1;
    while (P < m) P <<= 1;
    for (int i = threadIdx.x; i < P; i += kThreads) {
        if (i < m) {
            sk[i] = ckey[static_cast<size_t>(j) * kCap + i];
            si[i] = cid[static_cast<size_t>(j) * kCap + i];
        } else {
            sk[i] = 0ull;
            si[i] = 0x7fffffff;  // sorts last
        }
    }
    __syncthreads();
    // "greater" = earlier in the output
    auto before = [&](int a, int b2) {
        return sk[a] > sk[b2] || (sk[a] == sk[b2] && si[a] < si[b2]);
    };
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += kThreads) {
                const int partner = i ^ stride;
                if (partner > i) {
                    const bool desc = (i & size) == 0;  // first half of each block: best first
                    const bool swap = desc ? before(partner, i) : before(i, partner);
                    if (swap) {
                        const unsigned long long tk = sk[i];
                        sk[i] = sk[partner];
                        sk[partner] = tk;
                        const int ti = si[i];
                        si[i] = si[partner];
                        si[partner] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    const int take = min(k, m);
    for (int i = threadIdx.x; i < take; i += kThreads) {
        ids_out[static_cast<size_t>(j) * k + i] = si[i];
        vals_out[static_cast<size_t>(j) * k + i] = __longlong_as_double(static_cast<long long>(sk[i]));
    }
    for (int i = take + threadIdx.x; i < k; i += kThreads) {
        ids_out[static_cast<size_t>(j) * k + i] = -1;
        vals_out[static_cast<size_t>(j) * k + i] = 0.0;
    }
    if (threadIdx.x == 0) count_out[j] = take;
}

// ---- small columns: the whole select in one CTA per column -------------------
// For n <= kSmallN the 8 radix rounds, the mask subtraction, the collect and
// the sort run inside one CTA per column (histogram and candidates in shared
// memory): 1 launch instead of ~27 (latency-bound configs such as cfg1).
// Same keys, same digits, same tie order as the multi-CTA path.
constexpr int64_t kSmallN = 65536;
constexpr int kSmallThreads = 512;

__global__ void __launch_bounds__(kSmallThreads)
    topk_small_kernel(const double* __restrict__ scores, int64_t n, int k, MaskRef m,
                      int64_t* __restrict__ ids_out, double* __restrict__ vals_out, int32_t* __restrict__ count_out) {
    extern __shared__ unsigned char tsm[];
    unsigned int* h = reinterpret_cast<unsigned int*>(tsm);                        // [kBins]
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(h + kBins);     // [kCap]
    int* si = reinterpret_cast<int*>(sk + kCap);                                   // [kCap]
    __shared__ ColState c;
    __shared__ unsigned int part[kSmallThreads];
    __shared__ int s_bin, s_cum;
    const int j = blockIdx.x;
    const double* col = scores + static_cast<size_t>(j) * n;
    int scap = 64;
    while (scap < 2 * k && scap < kCap) scap <<= 1;
    if (threadIdx.x == 0) {
        c = ColState{};
        c.shift = 96;
        c.need = static_cast<int>(k < n ? static_cast<int64_t>(k) : n);
    }
    __syncthreads();
    for (int round = 0; round < kRounds && !c.done; ++round) {
        for (int i = threadIdx.x; i < kBins; i += kSmallThreads) h[i] = 0;
        __syncthreads();
        const ColState cc = c;
        const int ns = max(cc.shift - kDigit, 0);
        // 4 loads in flight per thread (the scan is latency-bound at these sizes)
        for (int64_t i0 = threadIdx.x; i0 < n; i0 += 4 * kSmallThreads) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t i = i0 + u * kSmallThreads;
                v[u] = i < n ? col[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t i = i0 + u * kSmallThreads;
                if (i >= n) break;
                const unsigned long long hi = score_key(v[u]);
                const unsigned int lo = ~static_cast<unsigned int>(i);
                if (cmp_prefix(hi, lo, cc, cc.shift) == 0 && !above_bound(m, j, hi, lo))
                    atomicAdd(&h[digit_of(hi, lo, ns)], 1u);
            }
        }
        __syncthreads();
        // masked ids leave the histogram (topk_mask_kernel)
        auto visit = [&](int64_t id) {
            const unsigned long long hi = score_key(col[id]);
            const unsigned int lo = ~static_cast<unsigned int>(id);
            if (cmp_prefix(hi, lo, cc, cc.shift) == 0 && !above_bound(m, j, hi, lo)) atomicSub(&h[digit_of(hi, lo, ns)], 1u);
        };
        const int64_t self = m.self ? m.self[j] : -1;
        if (threadIdx.x == 0 && self >= 0) visit(self);
        if (m.rowptr && m.rows && m.rows[j] >= 0) {
            const int64_t r = m.rows[j];
            for (int e = m.rowptr[r] + threadIdx.x; e < m.rowptr[r + 1]; e += kSmallThreads) {
                const int64_t id = m.colidx[e];
                if (id != self) visit(id);
            }
        }
        __syncthreads();
        // pivot digit (topk_select_kernel)
        constexpr int PB = kBins / kSmallThreads;
        unsigned int loc = 0;
        for (int i = 0; i < PB; ++i) loc += h[threadIdx.x * PB + i];
        part[threadIdx.x] = loc;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int cum = 0;
            int bin = -1;
            for (int t = kSmallThreads - 1; t >= 0 && bin < 0; --t) {
                if (cum + part[t] >= static_cast<unsigned int>(c.need)) {
                    for (int i = PB - 1; i >= 0; --i) {
                        const unsigned int hv = h[t * PB + i];
                        if (cum + hv >= static_cast<unsigned int>(c.need)) {
                            bin = t * PB + i;
                            break;
                        }
                        cum += hv;
                    }
                } else {
                    cum += part[t];
                }
            }
            s_bin = bin;
            s_cum = static_cast<int>(cum);
            if (bin < 0) {
                c.done = 1;
            } else {
                const unsigned int pivot = h[bin];
                c.above += s_cum;
                c.need -= s_cum;
                if (ns >= 32) {
                    c.phi |= static_cast<unsigned long long>(bin) << (ns - 32);
                } else {
                    const unsigned long long v = static_cast<unsigned long long>(bin) << ns;
                    c.plo |= static_cast<unsigned int>(v & 0xffffffffull);
                    c.phi |= v >> 32;
                }
                c.shift = ns;
                // refine until few candidates remain: the final sort is the
                // costly step here (bitonic over the next power of two)
                if (c.above + static_cast<int>(pivot) <= scap || ns == 0) c.done = 1;
            }
        }
        __syncthreads();
    }
    // collect every unmasked element at or above the pivot range
    if (threadIdx.x == 0) c.ncand = 0;
    __syncthreads();
    const ColState cc = c;
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += 4 * kSmallThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * kSmallThreads;
            v[u] = i < n ? col[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * kSmallThreads;
            if (i >= n) break;
            const unsigned long long hi = score_key(v[u]);
            const unsigned int lo = ~static_cast<unsigned int>(i);
            if (cmp_prefix(hi, lo, cc, cc.shift) >= 0 && !above_bound(m, j, hi, lo) && !is_masked(m, j, i)) {
                const int pos = atomicAdd(&c.ncand, 1);
                if (pos < kCap) {
                    sk[pos] = hi;
                    si[pos] = static_cast<int>(i);
                }
            }
        }
    }
    __syncthreads();
    const int mm = min(c.ncand, kCap);
    int P = 1;
    while (P < mm) P <<= 1;
    for (int i = mm + threadIdx.x; i < P; i += kSmallThreads) {
        sk[i] = 0ull;
        si[i] = 0x7fffffff;
    }
    __syncthreads();
    auto before = [&](int a, int b2) { return sk[a] > sk[b2] || (sk[a] == sk[b2] && si[a] < si[b2]); };
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += kSmallThreads) {
                const int partner = i ^ stride;
                if (partner > i) {
                    const bool desc = (i & size) == 0;
                    const bool swap = desc ? before(partner, i) : before(i, partner);
                    if (swap) {
                        const unsigned long long tk = sk[i];
                        sk[i] = sk[partner];
                        sk[partner] = tk;
                        const int ti = si[i];
                        si[i] = si[partner];
                        si[partner] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    const int take = min(k, mm);
    for (int i = threadIdx.x; i < take; i += kSmallThreads) {
        ids_out[static_cast<size_t>(j) * k + i] = si[i];
        vals_out[static_cast<size_t>(j) * k + i] = __longlong_as_double(static_cast<long long>(sk[i]));
    }
    for (int i = take + threadIdx.x; i < k; i += kSmallThreads) {
        ids_out[static_cast<size_t>(j) * k + i] = -1;
        vals_out[static_cast<size_t>(j) * k + i] = 0.0;
    }
    if (threadIdx.x == 0) count_out[j] = take;
}

struct TopkWork {
    ColState* cs;
    unsigned int* hist;
    unsigned long long* ckey;
    int* cid;
    int64_t* mrows;
    int64_t* mself;
};

void carve_topk(Carver& cv, int b, TopkWork& w) {
    w.cs = cv.take<ColState>(b);
    w.hist = cv.take<unsigned int>(static_cast<size_t>(b) * kBins);
    w.ckey = cv.take<unsigned long long>(static_cast<size_t>(b) * kCap);
    w.cid = cv.take<int>(static_cast<size_t>(b) * kCap);
    w.mrows = cv.take<int64_t>(b);
    w.mself = cv.take<int64_t>(b);
}

}  // namespace

extern "C" size_t kz_topk_workspace_bytes(int32_t b, int64_t n, int32_t k) {
    (void)n;
    (void)k;
    if (b < 1) return 0;
    Carver cv(nullptr, 0);
    TopkWork w;
    carve_topk(cv, b, w);
    return cv.off + 256;
}

extern "C" int kz_topk_batch(const kz_topk_args* a, void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    if (!a || a->b < 1 || a->n < 1 || a->k < 1 || !a->scores || !a->ids_out || !a->vals_out ||
        !a->count_out)
        return fail(KZ_EARG, "bad top-k arguments");
    if (a->n >= (int64_t(1) << 31) - 1) return fail(KZ_EARG, "n too large");
    if (std::min<int64_t>(a->k, a->n) > kCap)
        return fail(KZ_EARG, "k above 4096 per pass (continue with bound_vals/bound_ids)");
    if ((a->bound_vals == nullptr) != (a->bound_ids == nullptr)) return fail(KZ_EARG, "bound needs values and ids");
    if (!ws || ws_bytes < kz_topk_workspace_bytes(a->b, a->n, a->k)) return fail(KZ_EARG, "workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver cv(ws, ws_bytes);
    TopkWork w;
    carve_topk(cv, a->b, w);
    const int b = a->b;
    MaskRef m{};
    if (a->mask_graph && a->mask_rows) {
        m.rowptr = a->mask_graph->rowptr;
        m.colidx = a->mask_graph->colidx;
        KZ_CUDA(cudaMemcpyAsync(w.mrows, a->mask_rows, sizeof(int64_t) * b, cudaMemcpyHostToDevice, st));
        m.rows = w.mrows;
    }
    if (a->self_ids) {
        KZ_CUDA(cudaMemcpyAsync(w.mself, a->self_ids, sizeof(int64_t) * b, cudaMemcpyHostToDevice, st));
        m.self = w.mself;
    }
    m.bval = a->bound_vals;
    m.bid = a->bound_ids;
    if (a->n <= kSmallN) {
        constexpr size_t smem = sizeof(unsigned int) * kBins + (sizeof(unsigned long long) + sizeof(int)) * kCap;
        static bool attr = false;
        if (!attr) {
            KZ_CUDA(cudaFuncSetAttribute(topk_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            attr = true;
        }
        topk_small_kernel<<<b, kSmallThreads, smem, st>>>(a->scores, a->n, a->k, m, a->ids_out, a->vals_out,
                                                         a->count_out);
        ::kz::note_launch();
        KZ_LAUNCH_CHECK();
        return KZ_OK;
    }
    KZ_CUDA(cudaMemsetAsync(w.hist, 0, sizeof(unsigned int) * b * kBins, st));
    topk_init_kernel<<<(b + 127) / 128, 128, 0, st>>>(w.cs, b, a->n, a->k); ::kz::note_launch();
    KZ_LAUNCH_CHECK();
    // slices per column: ~64k elements each, enough CTAs to fill the chip
    int slices = static_cast<int>((a->n + 65535) / 65536);
    slices = std::max(slices, static_cast<int>(std::min<int64_t>((2 * max_ctas_per_chunk() + b - 1) / b,
                                                                  (a->n + 4095) / 4096)));
    slices = std::max(slices, 1);
    for (int r = 0; r < kRounds; ++r) {
        topk_hist_kernel<<<static_cast<unsigned>(b) * slices, kThreads, 0, st>>>(a->scores, a->n, slices, w.cs, w.hist, m); ::kz::note_launch();
        topk_mask_kernel<<<b, kThreads, 0, st>>>(a->scores, a->n, w.cs, w.hist, m); ::kz::note_launch();
        topk_select_kernel<<<b, kThreads, 0, st>>>(w.cs, w.hist); ::kz::note_launch();
        KZ_LAUNCH_CHECK();
    }
    topk_collect_kernel<<<static_cast<unsigned>(b) * slices, kThreads, 0, st>>>(a->scores, a->n, slices, w.cs, w.ckey, w.cid, m); ::kz::note_launch();
    topk_sort_kernel<<<b, kThreads, 0, st>>>(w.cs, w.ckey, w.cid, a->k, a->ids_out, a->vals_out, a->count_out); ::kz::note_launch();
    KZ_LAUNCH_CHECK();
    return KZ_OK;
}
