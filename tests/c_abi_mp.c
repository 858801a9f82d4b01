/*
 * c_abi_mp.c -- the whole multi-process path driven from plain C11 (no Python, no torch):
 * the parent starts the job server (lib/gdraa_jobserver) and forks `world`
 * rank processes; each rank joins with gdraa_init, registers its device buffers
 * (P:123), and runs gdraa_sgd_step on a small call (the latency kernel) and a large one
 * (the two-shot kernel) and gdraa_allreduce_mean, on integer-valued inputs whose
 * results are exact in any order (SURVEY §8(c) integer family), checked against the
 * closed form; then gdraa_finalize.  Ranks share the GPUs round-robin (time-sliced when
 * there are fewer GPUs than ranks).  Built and run by tests/test_c_abi.py.
 *
 *   c_abi_mp <path to gdraa_jobserver> <world>
 */
#define _POSIX_C_SOURCE 200809L
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/types.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cuda_runtime_api.h>

#include "gdraa.h"

static float g_of(int p, size_t i) { return (float)((int)((i * 7u + (size_t)p * 13u) % 257u) - 128); }
static float w_of(size_t i) { return (float)((int)(i % 97u) - 48); }
static float v_of(size_t i) { return (float)((int)(i % 31u) - 15); }

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            fprintf(stderr, "rank %d: %s: %s\n", rank, #x, cudaGetErrorString(e_));       \
            return 1;                                                                    \
        }                                                                                \
    } while (0)
#define GK(x)                                                                            \
    do {                                                                                 \
        int r_ = (x);                                                                    \
        if (r_ != GDRAA_OK) {                                                            \
            fprintf(stderr, "rank %d: %s: %d %s\n", rank, #x, r_, gdraa_last_error());    \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

/* One gdraa_sgd_step of n elements (world must be a power of two: exact closed form). */
static int step(int rank, int world, size_t n, size_t *bad) {
    const float lr = 0.125f, mom = 0.5f;
    float *h = malloc(sizeof(float) * n), *g, *w, *v;
    if (h == NULL) return 1;
    CK(cudaMalloc((void **)&g, sizeof(float) * n));
    CK(cudaMalloc((void **)&w, sizeof(float) * n));
    CK(cudaMalloc((void **)&v, sizeof(float) * n));
    for (size_t i = 0; i < n; ++i) h[i] = g_of(rank, i);
    CK(cudaMemcpy(g, h, sizeof(float) * n, cudaMemcpyHostToDevice));
    for (size_t i = 0; i < n; ++i) h[i] = w_of(i);
    CK(cudaMemcpy(w, h, sizeof(float) * n, cudaMemcpyHostToDevice));
    for (size_t i = 0; i < n; ++i) h[i] = v_of(i);
    CK(cudaMemcpy(v, h, sizeof(float) * n, cudaMemcpyHostToDevice));
    GK(gdraa_register(w, n, GDRAA_F32));
    GK(gdraa_register(g, n, GDRAA_F32));
    GK(gdraa_sgd_step(w, g, v, lr, mom, NULL));
    CK(cudaDeviceSynchronize());
    size_t off = 0, len = 0;
    GK(gdraa_shard(world, rank, n, &off, &len));
    float *hv = malloc(sizeof(float) * n);
    if (hv == NULL) return 1;
    CK(cudaMemcpy(h, w, sizeof(float) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hv, v, sizeof(float) * n, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) {
        float s = g_of(0, i);
        for (int p = 1; p < world; ++p) s += g_of(p, i);
        const float m = s / (float)world;
        const float v1 = mom * v_of(i) + m;
        *bad += h[i] != w_of(i) - lr * v1;
        *bad += (i >= off && i < off + len) ? hv[i] != v1 : hv[i] != v_of(i);
    }
    /* allreduce_mean in place on the gradient buffer */
    GK(gdraa_allreduce_mean(g, NULL));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, g, sizeof(float) * n, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) {
        float s = g_of(0, i);
        for (int p = 1; p < world; ++p) s += g_of(p, i);
        *bad += h[i] != s / (float)world;
    }
    GK(gdraa_deregister(w));
    GK(gdraa_deregister(g));
    free(h);
    free(hv);
    return 0;
}

static int run_rank(int rank, int world) {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    CK(cudaSetDevice(rank % ndev));
    GK(gdraa_init(world, rank));
    size_t bad = 0;
    if (step(rank, world, 1000, &bad) || step(rank, world, 3000017, &bad)) return 1;
    gdraa_stats_t st;
    GK(gdraa_get_stats(&st));
    GK(gdraa_finalize());
    printf("rank %d: %zu mismatches, calls %llu, ll_calls %llu, sync_waits %llu\n", rank, bad,
           (unsigned long long)st.calls, (unsigned long long)st.ll_calls,
           (unsigned long long)st.sync_waits);
    /* 4 calls: the small pair on the latency kernels, the large pair two-shot */
    return bad != 0 || st.calls != 4 || st.ll_calls != 2 || st.sync_waits != 4;
}

int main(int argc, char **argv) {
    if (argc != 3) {
        fprintf(stderr, "usage: %s <gdraa_jobserver> <world>\n", argv[0]);
        return 2;
    }
    const int world = atoi(argv[2]);
    char sock[128];
    snprintf(sock, sizeof sock, "/tmp/gdraa_c_abi_mp_%d.sock", (int)getpid());
    char wstr[16];
    snprintf(wstr, sizeof wstr, "%d", world);
    const pid_t js = fork();
    if (js == 0) {
        execl(argv[1], argv[1], "--socket", sock, "--world", wstr, "--timeout-ms", "120000",
              (char *)NULL);
        _exit(127);
    }
    setenv("GDRAA_JOBSERVER", sock, 1);
    pid_t kids[GDRAA_MAX_WORLD];
    for (int r = 0; r < world; ++r) {
        kids[r] = fork();
        if (kids[r] == 0) _exit(run_rank(r, world));   /* CUDA only ever in the children */
    }
    int failed = 0;
    for (int r = 0; r < world; ++r) {
        int status = 0;
        waitpid(kids[r], &status, 0);
        failed |= !WIFEXITED(status) || WEXITSTATUS(status) != 0;
    }
    int status = 0;
    waitpid(js, &status, 0);
    failed |= !WIFEXITED(status) || WEXITSTATUS(status) != 0;
    printf("%s\n", failed ? "FAIL" : "OK");
    return failed;
}
