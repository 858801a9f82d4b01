/*
 * gdraa_oracle.c -- plain CPU oracle for the GDRAA hot path.  TEST INFRASTRUCTURE:
 * see gdraa_oracle.h for who may use it, the paper passages each function follows,
 * and the precision contract.  Shares no code with the CUDA path.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared
 * (oracle/build.py).  Plain loops, one element at a time, in the paper's order.
 */
#include "gdraa_oracle.h"

#include <math.h>
#include <string.h>

/* P:185 "MiMatrix is designed for maximum 32 workers". */
#define ORACLE_MAX_N 32

int oracle_partition(uint64_t L, int N, uint64_t Q, int r, uint64_t *off, uint64_t *len)
{
    if (L == 0 || N < 1 || N > ORACLE_MAX_N || Q == 0 || r < 0 || r >= N) return -1;
    /* "Divide D(i) by N, and get D(i,m), m in [1,N]" -- ceil(L/N) per block. */
    uint64_t c = (L + (uint64_t)N - 1) / (uint64_t)N;
    /* AMB-8: round the block length up to a multiple of Q elements. */
    uint64_t blk = ((c + Q - 1) / Q) * Q;
    uint64_t o = (uint64_t)r * blk;
    if (o > L) o = L;
    uint64_t l = blk;
    if (l > L - o) l = L - o;
    *off = o;
    *len = l;
    return 0;
}

float oracle_bf16_to_f32(uint16_t b)
{
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

uint16_t oracle_f32_to_bf16_rne(float f)
{
    uint32_t u;
    memcpy(&u, &f, sizeof u);
    /* round to nearest, ties to even, on the 16 discarded bits (finite inputs). */
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

static float load_elem(int dtype, const void *buf, uint64_t i)
{
    if (dtype == ORACLE_F32) return ((const float *)buf)[i];
    return oracle_bf16_to_f32(((const uint16_t *)buf)[i]);
}

/* Aggregation "Average D(k,i), k in [1,N]": left fold in ascending rank
 * starting from rank 0's value (AMB-2, AMB-3), then one division by N (Eq. 3's
 * L/N "multiply" term is read as one correctly rounded division, AMB-2). */
static float average_elem(int N, int dtype, const void *const *in, uint64_t i)
{
    float s = load_elem(dtype, in[0], i);
    for (int p = 1; p < N; p++) {
        float x = load_elem(dtype, in[p], i);
        s = s + x;
    }
    float m = s / (float)N;
    return m;
}

int oracle_allreduce_mean(int N, uint64_t L, int dtype, const void *const *in, void *out)
{
    if (N < 1 || N > ORACLE_MAX_N || (dtype != ORACLE_F32 && dtype != ORACLE_BF16)) return -1;
    if (L == 0) return -1;
    for (uint64_t i = 0; i < L; i++) {
        float m = average_elem(N, dtype, in, i);
        /* "send D(i) to all workers": every rank receives this same value. */
        if (dtype == ORACLE_F32)
            ((float *)out)[i] = m;
        else
            ((uint16_t *)out)[i] = oracle_f32_to_bf16_rne(m);
    }
    return 0;
}

int oracle_sgd_step(int N, uint64_t L, int dtype, const void *const *g, float *w, float *v,
                    float lr, float mom)
{
    if (N < 1 || N > ORACLE_MAX_N || (dtype != ORACLE_F32 && dtype != ORACLE_BF16)) return -1;
    if (L == 0) return -1;
    for (uint64_t i = 0; i < L; i++) {
        float m = average_elem(N, dtype, g, i);
        /* "Update model with gradient of differential D", momentum SGD
         * v <- mom*v + D; w <- w - lr*v (lambda = 0; AMB-4: four roundings). */
        float t = mom * v[i];
        float vn = t + m;
        float u = lr * vn;
        float wn = w[i] - u;
        v[i] = vn;
        w[i] = wn;
    }
    return 0;
}

int oracle_sgd_step_wd(int N, uint64_t L, int dtype, const void *const *g, float *w, float *v,
                       float lr, float mom, float wd, void *model, int model_dtype)
{
    if (N < 1 || N > ORACLE_MAX_N || (dtype != ORACLE_F32 && dtype != ORACLE_BF16)) return -1;
    if (L == 0) return -1;
    if (model != 0 && model_dtype != ORACLE_F32 && model_dtype != ORACLE_BF16) return -1;
    for (uint64_t i = 0; i < L; i++) {
        float m = average_elem(N, dtype, g, i);
        /* v <- mu*v + (g + lambda*w); w <- w - lr*v, one rounding per operation */
        float ge = m;
        if (wd != 0.0f) {
            float d = wd * w[i];
            ge = m + d;
        }
        float t = mom * v[i];
        float vn = t + ge;
        float u = lr * vn;
        float wn = w[i] - u;
        v[i] = vn;
        w[i] = wn;
        if (model != 0) {
            if (model_dtype == ORACLE_F32)
                ((float *)model)[i] = wn;
            else
                ((uint16_t *)model)[i] = oracle_f32_to_bf16_rne(wn);
        }
    }
    return 0;
}

float oracle_poly_lr(float lr0, uint64_t iter, uint64_t max_iter, float power)
{
    if (max_iter == 0) return -1.0f;
    if (iter >= max_iter) return 0.0f;
    double frac = 1.0 - (double)iter / (double)max_iter;
    return (float)((double)lr0 * pow(frac, (double)power));
}

int oracle_counters(uint64_t L, int N, uint64_t Q, int r, int s_g, int s_w,
                    oracle_counters_t *out)
{
    uint64_t off, len;
    if (oracle_partition(L, N, Q, r, &off, &len) != 0) return -1;
    if (s_g <= 0 || s_w <= 0) return -1;
    (void)off;
    uint64_t n1 = (uint64_t)(N - 1);
    /* Eq. 1: worker r sends its N-1 foreign blocks, L - len_r elements. */
    out->rs_sent = (uint64_t)s_g * (L - len);
    /* Eq. 2: worker r receives its own block from each of the N-1 others. */
    out->rs_recv = (uint64_t)s_g * n1 * len;
    /* "For the step 2, the proof [is] similar": broadcast mirrors step 1. */
    out->ag_sent = (uint64_t)s_w * n1 * len;
    out->ag_recv = (uint64_t)s_w * (L - len);
    /* Eq. 3: (N-1) adds and one multiply (here: divide) per owned element. */
    out->adds = n1 * len;
    out->divides = len;
    out->sync_waits = N >= 2 ? 2 : 0;
    return 0;
}
