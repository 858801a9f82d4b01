/*
 * c_abi_smoke.c -- the C ABI (include/gdraa.h) used from plain C11: no Python, no torch.
 * Built by tests/test_c_abi.py (compile + link on CPU; run under -m gpu).
 *
 * Four virtual ranks on one GPU (gdraa_vr_sgd_step, the same kernels as the
 * multi-process path) step integer-valued inputs whose every intermediate is exactly
 * representable (SURVEY §8(c) integer family): g in [-128, 128], w in [-48, 48],
 * v in [-15, 15], lr = 1/8, mom = 1/2.  Then m = (g0+g1+g2+g3)/4, v' = v/2 + m and
 * w' = w - v'/8 are exact in any order and rounding, so the program checks the closed
 * form directly: w' on every rank, v' on each rank's owner shard (gdraa_shard), v
 * untouched elsewhere, g unchanged (AMB-18, AMB-19).
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "gdraa.h"

#define N 4
#define L 1000003u

static int ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
        return 1;
    }
    return 0;
}

static float g_of(int p, size_t i) { return (float)((int)((i * 7u + (size_t)p * 13u) % 257u) - 128); }
static float w_of(size_t i) { return (float)((int)(i % 97u) - 48); }
static float v_of(size_t i) { return (float)((int)(i % 31u) - 15); }

int main(void) {
    const float lr = 0.125f, mom = 0.5f;
    float *h = malloc(sizeof(float) * L), *hv = malloc(sizeof(float) * L);
    float *g[N], *w[N], *v[N];
    if (h == NULL || hv == NULL) return 1;
    for (int p = 0; p < N; ++p) {
        if (ck(cudaMalloc((void **)&g[p], sizeof(float) * L), "cudaMalloc g") ||
            ck(cudaMalloc((void **)&w[p], sizeof(float) * L), "cudaMalloc w") ||
            ck(cudaMalloc((void **)&v[p], sizeof(float) * L), "cudaMalloc v"))
            return 1;
        for (size_t i = 0; i < L; ++i) h[i] = g_of(p, i);
        if (ck(cudaMemcpy(g[p], h, sizeof(float) * L, cudaMemcpyHostToDevice), "H2D g")) return 1;
        for (size_t i = 0; i < L; ++i) h[i] = w_of(i);
        if (ck(cudaMemcpy(w[p], h, sizeof(float) * L, cudaMemcpyHostToDevice), "H2D w")) return 1;
        for (size_t i = 0; i < L; ++i) h[i] = v_of(i);
        if (ck(cudaMemcpy(v[p], h, sizeof(float) * L, cudaMemcpyHostToDevice), "H2D v")) return 1;
    }
    int rc = gdraa_vr_sgd_step(N, w, (const void *const *)g, v, L, GDRAA_F32, lr, mom, NULL);
    if (rc != GDRAA_OK) {
        fprintf(stderr, "gdraa_vr_sgd_step: %d %s\n", rc, gdraa_last_error());
        return 1;
    }
    if (ck(cudaDeviceSynchronize(), "sync")) return 1;
    size_t bad = 0;
    for (int r = 0; r < N; ++r) {
        size_t off = 0, len = 0;
        if (gdraa_shard(N, r, L, &off, &len) != GDRAA_OK) return 1;
        if (ck(cudaMemcpy(h, w[r], sizeof(float) * L, cudaMemcpyDeviceToHost), "D2H w") ||
            ck(cudaMemcpy(hv, v[r], sizeof(float) * L, cudaMemcpyDeviceToHost), "D2H v"))
            return 1;
        for (size_t i = 0; i < L; ++i) {
            const float m = (g_of(0, i) + g_of(1, i) + g_of(2, i) + g_of(3, i)) / 4.0f;
            const float v1 = mom * v_of(i) + m;
            const float w1 = w_of(i) - lr * v1;
            const int own = i >= off && i < off + len;
            bad += h[i] != w1;
            bad += own ? hv[i] != v1 : hv[i] != v_of(i);
        }
        if (ck(cudaMemcpy(h, g[r], sizeof(float) * L, cudaMemcpyDeviceToHost), "D2H g")) return 1;
        for (size_t i = 0; i < L; ++i) bad += h[i] != g_of(r, i);
    }
    for (int p = 0; p < N; ++p) {
        cudaFree(g[p]);
        cudaFree(w[p]);
        cudaFree(v[p]);
    }
    free(h);
    free(hv);
    printf("%s %s: %zu mismatches over %d ranks x %u elements\n", bad ? "FAIL" : "OK",
           gdraa_version(), bad, N, L);
    return bad != 0;
}
