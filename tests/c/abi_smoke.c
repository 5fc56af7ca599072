/* abi_smoke.c -- the C-ABI of libkatzb200.so driven from plain C, no Python:
 * what a non-Python host binding does.
 *
 *   cpu mode: version, the host-side build entry points (kz_partition,
 *             kz_min_degree_order) and their argument errors;
 *   gpu mode: kz_graph_create + kz_cg_batch on a 6-node graph with device
 *             buffers from cudaMalloc, checked against a dense Gaussian
 *             elimination of (I - beta A) x = beta A e_q done here. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "katzb200.h"

/* cuda runtime (only the few calls the gpu mode needs) */
typedef int cudaError_t;
extern cudaError_t cudaMalloc(void** p, size_t n);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* d, const void* s, size_t n, int kind);
extern cudaError_t cudaDeviceSynchronize(void);

#define CHECK(c)                                                                 \
    do {                                                                         \
        if (!(c)) {                                                              \
            fprintf(stderr, "FAIL %s:%d %s (%s)\n", __FILE__, __LINE__, #c,      \
                    kz_last_error() ? kz_last_error() : "");                     \
            return 1;                                                            \
        }                                                                        \
    } while (0)

/* 0-1-2-3-4 path plus the chord 1-4 and a pendant 5 on 3 */
static const int64_t N = 6;
static const int64_t RP[7] = {0, 1, 4, 6, 9, 11, 12};
static const int64_t CI64[12] = {1, 0, 2, 4, 1, 3, 2, 4, 5, 1, 3, 3};

static int cpu_mode(void) {
    CHECK(kz_version() > 0);
    int64_t perm[6], bounds[7], nparts = 0, n1 = 0, n2 = 0;
    CHECK(kz_partition(N, RP, CI64, 2, 64, perm, bounds, &nparts, &n1, &n2) == KZ_OK);
    int seen[6] = {0};
    for (int i = 0; i < N; ++i) {
        CHECK(perm[i] >= 0 && perm[i] < N && !seen[perm[i]]);
        seen[perm[i]] = 1;
    }
    CHECK(n1 + n2 == N && bounds[0] == 0 && bounds[nparts] == n1);
    CHECK(kz_partition(0, RP, CI64, 2, 64, perm, bounds, &nparts, &n1, &n2) == KZ_EARG);
    CHECK(kz_partition(N, RP, CI64, 0, 64, perm, bounds, &nparts, &n1, &n2) == KZ_EARG);
    int64_t order[6];
    CHECK(kz_min_degree_order(N, RP, CI64, order) == KZ_OK);
    for (int i = 0; i < N; ++i) seen[i] = 0;
    for (int i = 0; i < N; ++i) {
        CHECK(order[i] >= 0 && order[i] < N && !seen[order[i]]);
        seen[order[i]] = 1;
    }
    CHECK(order[0] == 0); /* degree-1 nodes 0 and 5: ties go to the smaller index */
    printf("cpu ok: version %d, %lld parts, n2 %lld\n", kz_version(), (long long)nparts, (long long)n2);
    return 0;
}

/* dense reference: solve (I - beta A) x = beta A e_q by Gaussian elimination */
static void dense_katz(double beta, int q, double* x) {
    double m[6][7];
    memset(m, 0, sizeof m);
    for (int i = 0; i < N; ++i) m[i][i] = 1.0;
    for (int i = 0; i < N; ++i)
        for (int64_t e = RP[i]; e < RP[i + 1]; ++e) {
            m[i][CI64[e]] -= beta;
            if (CI64[e] == q) m[i][6] += beta;
        }
    for (int c = 0; c < N; ++c)
        for (int r = c + 1; r < N; ++r) {
            const double f = m[r][c] / m[c][c];
            for (int k = c; k < 7; ++k) m[r][k] -= f * m[c][k];
        }
    for (int r = (int)N - 1; r >= 0; --r) {
        double s = m[r][6];
        for (int k = r + 1; k < N; ++k) s -= m[r][k] * x[k];
        x[r] = s / m[r][r];
    }
}

static int gpu_mode(void) {
    int32_t ci32[12];
    for (int i = 0; i < 12; ++i) ci32[i] = (int32_t)CI64[i];
    kz_graph* g = NULL;
    CHECK(kz_graph_create(N, N, 12, RP, ci32, &g) == KZ_OK && g);
    const int b = 2;
    int64_t qpos[2] = {0, 4};
    const double beta = 0.3;
    double* scores = NULL;
    void* ws = NULL;
    const size_t wsb = kz_cg_workspace_bytes(g, b);
    CHECK(wsb > 0);
    CHECK(cudaMalloc((void**)&scores, sizeof(double) * b * N) == 0);
    CHECK(cudaMalloc(&ws, wsb) == 0);
    kz_report reps[2];
    kz_cg_args a;
    memset(&a, 0, sizeof a);
    a.b = b;
    a.clamp = 1;
    a.qpos = qpos;
    a.beta = beta;
    a.tol = 1e-13;
    a.scores = scores;
    a.reports = reps;
    CHECK(kz_cg_batch(g, &a, ws, wsb, NULL) == KZ_OK);
    double host[12];
    CHECK(cudaMemcpy(host, scores, sizeof host, 2 /* device to host */) == 0);
    for (int j = 0; j < b; ++j) {
        double want[6], err = 0.0, nrm = 0.0;
        dense_katz(beta, (int)qpos[j], want);
        for (int i = 0; i < N; ++i) {
            err += (host[j * N + i] - want[i]) * (host[j * N + i] - want[i]);
            nrm += want[i] * want[i];
        }
        CHECK(reps[j].converged == 1);
        CHECK(sqrt(err / nrm) <= 1e-12);
    }
    /* argument errors come back as statuses with a message */
    a.b = 0;
    CHECK(kz_cg_batch(g, &a, ws, wsb, NULL) == KZ_EARG && kz_last_error()[0] != 0);
    cudaFree(scores);
    cudaFree(ws);
    CHECK(kz_graph_destroy(g) == KZ_OK);
    printf("gpu ok: %lld kernel launches\n", kz_launch_count());
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_mode();
    return cpu_mode();
}
