/*
 * gdraa_oracle.h -- plain, slow, obviously-correct CPU oracle for the GDRAA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (include/gdraa.h, paper_1802_02326_b200/) never includes, links or calls it, and
 * this oracle includes nothing from the product path.
 *
 * What it computes (arxiv 1802.02326, PAPER.md = P:<line>):
 *   - Algorithm 1 "Divide D(i) ... by N, and get D(i,m)"            P:162, §3
 *   - Algorithm 1 "Average D(k,i), k in [1,N]"                       P:168, Eq. 3
 *   - Algorithm 1 "Update model with gradient of differential D"     P:157, hyper-params P:246
 *   - Lemma 1 (Eq. 1-2) traffic and Lemma 2 (Eq. 3-4) op counts
 * Readings of the paper where it is silent are listed in DESIGN.md ("Readings") and
 * named below as AMB-k (SURVEY.md §8(c) ambiguity register).
 *
 * Precision: IEEE-754 binary32 with round-to-nearest-even, one rounding per operation,
 * no contraction (compiled -O2 -ffp-contract=off -fno-fast-math).  The paper fixes
 * single precision and the north star pins fp32 accumulation, so the
 * oracle computes in fp32 with a pinned order instead of fp64.
 */
#ifndef GDRAA_ORACLE_H
#define GDRAA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_F32 = 0, ORACLE_BF16 = 1 };

/* Block partition, Algorithm 1 line 8 "Divide D(i) by N", AMB-8:
 *   c = ceil(L/N); len = ceil(c/Q)*Q; off_r = min(r*len, L); len_r = min(len, L-off_r).
 * With Q = 1 this is SPEC's ceil rule.  Returns 0, or -1 on
 * invalid arguments (L = 0, N outside [1,32], Q = 0, r outside [0,N)). */
int oracle_partition(uint64_t L, int N, uint64_t Q, int r, uint64_t *off, uint64_t *len);

/* bf16 -> fp32 widening (exact: bits << 16). */
float oracle_bf16_to_f32(uint16_t b);
/* fp32 -> bf16 round-to-nearest-even (finite inputs; AMB-13). */
uint16_t oracle_f32_to_bf16_rne(float f);

/* Aggregation (Eq. 3): for every element i,
 *   s = x_0[i]; for p = 1..N-1: s = fl(s + x_p[i]);  m = fl(s / N)
 * Left fold in ascending rank starting from rank 0's value (AMB-2, AMB-3), one
 * IEEE division by N.  in[p] is rank p's buffer (dtype), out receives the mean in the
 * same dtype (bf16: RNE of the fp32 mean).  This is the value every rank holds after
 * the broadcast.  Returns 0 or -1. */
int oracle_allreduce_mean(int N, uint64_t L, int dtype, const void *const *in, void *out);

/* Update with the averaged gradient (lr/mom of P:246; SGD form S:412 with
 * lambda = 0, AMB-4): for every element i, with m the aggregation above,
 *   t = fl(mom * v[i]); v[i] = fl(t + m); u = fl(lr * v[i]); w[i] = fl(w[i] - u)
 * w is the single replicated weight vector (identical on every rank before and after).
 * v is the momentum state; element i is owned by the rank whose partition block holds
 * it (AMB-19), so a full-length array models the union of all owners' shards.
 * g[p] is rank p's gradient (dtype), unchanged (AMB-18).  Returns 0 or -1. */
int oracle_sgd_step(int N, uint64_t L, int dtype, const void *const *g, float *w, float *v,
                    float lr, float mom);

/* The update with weight decay ("weight decay is 0.001"; SGD form S:412
 * v <- mu*v + (g + lambda*w)), AMB-5: for every element i, with m the aggregation,
 *   d = fl(wd * w[i]); ge = fl(m + d); t = fl(mom * v[i]); v[i] = fl(t + ge);
 *   u = fl(lr * v[i]); w[i] = fl(w[i] - u)
 * and, when wd == 0, exactly oracle_sgd_step (no decay term is formed).
 * model (optional, may be NULL): the broadcast model copy in model_dtype, i.e. w[i]
 * itself (f32) or bf16 RNE(w[i]) -- NEXT-1's mixed-precision all-gather, where the fp32
 * master w is sharded like v and only the model copy travels.  Returns 0 or -1. */
int oracle_sgd_step_wd(int N, uint64_t L, int dtype, const void *const *g, float *w, float *v,
                       float lr, float mom, float wd, void *model, int model_dtype);

/* "poly" learning-rate policy with "gamma" read as the power:
 *   lr = lr0 * (1 - iter/max_iter)^power, evaluated in double, rounded once to float.
 * Returns lr0 * 0 = 0 for iter >= max_iter; -1.0f on max_iter == 0. */
float oracle_poly_lr(float lr0, uint64_t iter, uint64_t max_iter, float power);

/* Lemma 1 / Lemma 2 accounting for rank r (Eq. 1-2, Eq. 3-4). */
typedef struct {
    uint64_t rs_sent;     /* reduce: blocks j != r of D(r) leave r: s_g * (L - len_r)   (Eq. 1) */
    uint64_t rs_recv;     /* reduce: block r arrives from N-1 peers: s_g * (N-1) * len_r (Eq. 2) */
    uint64_t ag_sent;     /* broadcast: AG(r) to N-1 peers: s_w * (N-1) * len_r                 */
    uint64_t ag_recv;     /* broadcast: AG(j), j != r, arrive: s_w * (L - len_r)                */
    uint64_t adds;        /* (N-1) * len_r  (Eq. 3, first term)                                 */
    uint64_t divides;     /* len_r          (Eq. 3, second term)                                */
    uint64_t sync_waits;  /* 2 for N >= 2, 0 for N = 1 (Alg. 1 lines 153/166)            */
} oracle_counters_t;
int oracle_counters(uint64_t L, int N, uint64_t Q, int r, int s_g, int s_w,
                    oracle_counters_t *out);

#ifdef __cplusplus
}
#endif
#endif
