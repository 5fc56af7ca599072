// common.cuh -- shared helpers for libkatzb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "katzb200.h"

namespace kz {

int fail(int code, const std::string& msg);  // records msg, returns code
void clear_error();
void note_launch();  // counts every kernel launch of the library (kz_launch_count)
void add_launches(long long n);
uint64_t next_uid();  // process-unique handle ids
// K1 launch timing for bench.py (kz_k1_timing): when enabled, every K1
// launch outside stream capture is bracketed by two CUDA events on its
// own stream; kz_k1_timing_read sums their elapsed times.
bool k1_timing_on();
void k1_timing_begin(cudaStream_t st, cudaEvent_t* e0);
void k1_timing_end(cudaStream_t st, cudaEvent_t e0);

#define KZ_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return ::kz::fail(e_ == cudaErrorMemoryAllocation ? KZ_EOOM : KZ_ECUDA,     \
                              std::string(#call) + ": " + cudaGetErrorString(e_));     \
    } while (0)

#define KZ_LAUNCH_CHECK()                                                               \
    do {                                                                                \
        cudaError_t e_ = cudaGetLastError();                                            \
        if (e_ != cudaSuccess)                                                          \
            return ::kz::fail(KZ_ECUDA, std::string("kernel launch: ") +                \
                                            cudaGetErrorString(e_));                    \
    } while (0)

constexpr int kThreads = 256;        // threads per CTA for the streaming kernels
constexpr int kWarps = kThreads / 32;
// SM count of the current device (148 on B200), queried once per device;
// every persistent grid is sized from it.
int num_sms();
inline int max_ctas_per_chunk() { return num_sms() * 8; }

// ---- checked builds (make EXTRA=-DKZ_CHECKED=1; tools/checked_tier.sh) ----
// compute-sanitizer is not available on the GPU pool, so a checked build
// stands in for it: device bounds checks that trap (KZ_DCHECK), a bounded
// spin-wait in K1's segment fix-up, and 256-byte red zones between every
// workspace slice.  The Python layer fills each workspace with 0xFF before
// the call (NaN doubles / -1 ints: reads of unwritten scratch poison the
// result) and verifies after it that no red zone was written
// (kz_checked_redzones, _lib.Workspace).
#ifndef KZ_CHECKED
#define KZ_CHECKED 0
#endif
#if KZ_CHECKED
#define KZ_DCHECK(c)                                                                        \
    do {                                                                                    \
        if (!(c)) {                                                                         \
            printf("KZ_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);                \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define KZ_DCHECK(c) \
    do {             \
    } while (0)
#endif
constexpr size_t kRedzone = KZ_CHECKED ? 256 : 0;
void note_redzone(const void* base, size_t off);  // checked builds: remembers a red zone of a carve
void forget_redzones(const void* p0, const void* p1);  // ... and drops those inside [p0, p1)

// zero the contiguous span [p0, p1) of a workspace that covers several
// carved slices (counter / state blocks zeroed by one memset); in checked
// builds the red zones inside the span are zeroed too, so they are dropped
inline cudaError_t zero_span(void* p0, void* p1, cudaStream_t st) {
    if (kRedzone) forget_redzones(p0, p1);
    return cudaMemsetAsync(p0, 0, static_cast<size_t>(static_cast<char*>(p1) - static_cast<char*>(p0)), st);
}

// Bump allocator over a caller-provided workspace (256-byte aligned slices;
// checked builds put a 256-byte red zone in front of every slice).
struct Carver {
    char* base;
    size_t off = 0;
    size_t cap;
    Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        if (kRedzone) {
            if (base) note_redzone(base, off);
            off += kRedzone;
        }
        T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
        off += count * sizeof(T);
        return p;
    }
    bool ok() const { return off <= cap; }
};

// Layout helper: the chunked node-major block [b/C][rows][C].
__host__ __device__ inline size_t blk_index(int64_t rows, int C, int64_t i, int j) {
    return (static_cast<size_t>(j / C) * rows + i) * C + (j % C);
}

// Supported chunk widths (columns per chunk) and the default choice for b.
inline bool chunk_ok(int C) { return C == 1 || C == 2 || C == 4 || C == 8 || C == 16 || C == 32 || C == 64; }
inline int default_chunk(int b) {
    // experiments: KZ_CHUNK = chunk width cap (8 / 16 / 32 / 64) for wide batches
    static const int cap = [] {
        const char* e = std::getenv("KZ_CHUNK");
        const int v = e ? std::atoi(e) : 0;
        return v >= 8 && chunk_ok(v) ? v : 0;
    }();
    if (cap && b >= cap) return cap;
    if (b >= 32) return 32;  // 256-byte gathered segments, half the index passes of C=16
    if (b >= 16) return 16;
    int c = 1;
    while (c < b) c <<= 1;
    return c;
}

}  // namespace kz
