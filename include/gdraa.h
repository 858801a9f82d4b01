/*
 * gdraa.h -- C ABI of the B200-native GDRAA hot path (arxiv 1802.02326).
 *
 * GDRAA = "GPUDirect RDMA-Aware AllReduce" (PAPER.md = P:<line>; Algorithm 1
 * P:142-174, §3).  Per training iteration every rank's gradient D(i) is
 * divided into N blocks, block m of every rank is reduced and averaged by
 * rank m ("Reduce" + "Aggregation"), the averaged block is applied to the
 * weights and sent to every rank ("Broadcast"), with exactly two
 * synchronisations per iteration (Alg. 1 lines 153/166).
 *
 * On one NVSwitch node the "registered memory region" of P:123 (ibv_reg_mr) becomes a
 * CUDA IPC mapping of the caller's buffer in every peer process, and one sm_100a
 * kernel per call pulls the owner shard from every peer over NVLink, sums it in rank
 * order, divides by N, applies the momentum-SGD update, and pushes the updated shard
 * into every peer's buffer.  A host job server only
 * exchanges the 64-byte IPC handles and per-iteration go/done flags; it never touches
 * weight data.
 *
 * Conventions for every entry point:
 *  - Returns GDRAA_OK (0) or a negative gdraa_err_t.  On error a thread-local message
 *    is available from gdraa_last_error().  Nothing is enqueued on an error return.
 *  - Pointers named "device" are CUDA device pointers on the current device (the
 *    device current at gdraa_init); "host" pointers are ordinary host memory.
 *  - Calls that take a stream enqueue asynchronously and return immediately; results
 *    are visible to later work on that stream.  Device-side failures (a peer that
 *    never arrives within GDRAA_TIMEOUT_MS, default 30000) are STICKY: the next call and
 *    gdraa_finalize return GDRAA_ETIMEOUT and gdraa_last_error() names the missing ranks.
 *  - Collective calls (init, register, allreduce_mean, sgd_step, finalize) must be
 *    issued in the same order with the same sizes on every rank ("same iteration
 *    number and same L").  Calls on one stream run back to back; a call issued on a
 *    different stream than the previous call is ordered after all work issued so far
 *    on that previous stream (an event the library records there and waits on), so
 *    collectives never overlap on the device.  The previous call's stream must still
 *    exist when such a call is made.  Inside a CUDA-graph capture this ordering is the
 *    graph's (the library adds no cross-stream edge to a capturing stream).
 *  - The caller owns every data buffer and keeps it allocated until gdraa_finalize.
 *    The library owns its signal pads, peer mappings and host-mapped flag pages.
 */
#ifndef GDRAA_H
#define GDRAA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A cudaStream_t (layout-compatible; NULL = the legacy default stream). */
typedef struct CUstream_st *gdraa_stream_t;

typedef enum { GDRAA_F32 = 0, GDRAA_BF16 = 1 } gdraa_dtype_t;

typedef enum {
    GDRAA_OK = 0,
    GDRAA_EINVAL = -1,      /* bad argument (range, alignment, non-finite lr/mom, ...)   */
    GDRAA_ENOTREG = -2,     /* buffer not registered with gdraa_register                   */
    GDRAA_ESHAPE = -3,      /* n / dtype differ across ranks ("shape-mismatch")     */
    GDRAA_ECUDA = -4,       /* a CUDA runtime/driver call failed                           */
    GDRAA_ETIMEOUT = -5,    /* a peer missed a synchronisation ("peer-timeout")      */
    GDRAA_ESTATE = -6,      /* not initialised / already initialised / after a fatal error */
    GDRAA_EJOBSERVER = -7   /* job server unreachable or protocol error                    */
} gdraa_err_t;

/* Largest world on one NVSwitch node (the paper's design bound is 32 workers). */
#define GDRAA_MAX_WORLD 8
/* Shard alignment quantum in elements (AMB-8): shard starts are 64-element aligned. */
#define GDRAA_SHARD_QUANTUM 64

/*
 * gdraa_init -- join the communicator (collective over all `world` ranks).
 *   world: 1..GDRAA_MAX_WORLD ranks, one process per GPU of one node.
 *   rank:  0..world-1 (SPEC 0-based ranks).
 * Uses the CUDA device current on the calling thread.  For world > 1 the job server
 * socket path is read from the environment variable GDRAA_JOBSERVER (started by
 * paper_1802_02326_b200.jobserver); the call blocks until all ranks have joined and the
 * signal pads are mapped (GDRAA_CONNECT_TIMEOUT_MS, default 120000).  The small-message
 * thresholds (GDRAA_LL_MAX_BYTES, GDRAA_LL_SGD_MAX_BYTES) are read here, fixed for the
 * communicator's lifetime and checked to agree on every rank, since they decide which
 * kernel -- with which synchronisation protocol -- serves a call.
 * Errors: EINVAL (range), ESTATE (already initialised), ESHAPE (ranks disagree on the
 * thresholds), EJOBSERVER, ECUDA.  A failed call releases whatever it had acquired
 * (pads, mappings, socket), so it may be retried.
 */
int gdraa_init(int world, int rank);

/*
 * gdraa_register -- register a device buffer for peer access (collective, P:123's
 * "whole and continuous GPU memory registered by ibv_reg_mr").
 *   buf:   device pointer, 16-byte aligned, n elements of dtype.  May point into a
 *          larger cudaMalloc allocation (e.g. a PyTorch caching-allocator block); the
 *          whole enclosing allocation is exported with cudaIpcGetMemHandle.
 *   n:     element count >= 1, identical on every rank.
 *   dtype: GDRAA_F32 or GDRAA_BF16, identical on every rank.
 * Every rank must register its buffers in the same order.  Both the gradient g and
 * the weights w of gdraa_sgd_step, and the buffer of gdraa_allreduce_mean, must be
 * registered; the momentum buffer v is rank-local and need not be.
 * Errors: EINVAL, ESTATE, ESHAPE (n/dtype mismatch across ranks, reported on every
 * rank), EJOBSERVER, ECUDA.
 */
int gdraa_register(void *buf, size_t n, int dtype);

/*
 * gdraa_deregister -- forget a registration (local, not collective).  Peer mappings
 * of the enclosing allocation stay open until gdraa_finalize, so the same memory can be
 * registered again (e.g. after a caching allocator hands the address out anew).
 *   buf: a pointer previously passed to gdraa_register.
 * Errors: ENOTREG, ESTATE.
 */
int gdraa_deregister(void *buf);

/*
 * gdraa_allreduce_mean -- in place, buf <- (1/N) * sum_p buf_p on every rank
 * (Algorithm 1 without the update).
 *   buf: a registered device buffer (f32 or bf16).
 *   s:   stream; the call is ordered after prior work on s on this rank.
 * Per element: s = x_0; s = fl(s + x_p) for p = 1..N-1 (ascending rank); m = fl(s / N);
 * bf16 buffers accumulate in fp32 and store bf16 RNE(m).  Bitwise deterministic and
 * identical on every rank.  One kernel launch; two device-side synchronisations.
 * Errors: ENOTREG, ESTATE, ETIMEOUT (sticky, from an earlier call), ECUDA.
 */
int gdraa_allreduce_mean(void *buf, gdraa_stream_t s);

/*
 * gdraa_sgd_step -- fused reduce -> average -> momentum-SGD update -> broadcast
 * (Algorithm 1, hyper-parameters P:246).
 *   w:   registered f32 device buffer, n elements, identical on all ranks before the
 *        call; identical (updated) on all ranks after it.
 *   g:   registered gradient buffer (f32 or bf16), n elements.  Read only.
 *   v:   f32 device buffer, n elements, rank-local momentum state.  Only the owner
 *        shard [off_r, off_r + len_r) of gdraa_shard() is read and written.
 *   lr, mom: finite learning rate and momentum.
 * Per element: m as in gdraa_allreduce_mean; v = fl(fl(mom*v) + m); w = fl(w - fl(lr*v))
 * (four roundings, no FMA contraction).  Weight decay is not applied here.
 * Errors: EINVAL, ENOTREG, ESTATE, ETIMEOUT (sticky), ECUDA.
 */
int gdraa_sgd_step(float *w, const void *g, float *v, float lr, float mom, gdraa_stream_t s);

/*
 * gdraa_sgd_step_ex -- gdraa_sgd_step with weight decay wd ("weight decay is
 * 0.001"; SGD form S:412 v <- mu*v + (g + lambda*w)).  Per element, before the
 * momentum step: m = fl(m + fl(wd*w)).  wd == 0 forms no decay term, i.e. it is exactly
 * gdraa_sgd_step.  Arguments and errors as gdraa_sgd_step; wd must be finite.
 */
int gdraa_sgd_step_ex(float *w, const void *g, float *v, float lr, float mom, float wd,
                      gdraa_stream_t s);

/*
 * gdraa_sgd_step_mp -- mixed-precision variant: the fp32 master
 * weights are sharded like the momentum, and the broadcast carries a bf16 model
 * copy, cutting the all-gather bytes per element from 4 to 2.
 *   w_master: f32 device buffer, n elements, rank-local (not registered); only the owner
 *             shard [off_r, off_r + len_r) is read and written.
 *   w_model:  registered GDRAA_BF16 buffer, n elements; after the call every rank holds
 *             bf16 RNE(w') of every shard (w' = the updated fp32 master values).
 *   g, v, lr, mom, wd: as gdraa_sgd_step_ex (g's dtype is f32 or bf16).
 * Errors: EINVAL, ENOTREG, ESTATE, ETIMEOUT (sticky), ECUDA.
 */
int gdraa_sgd_step_mp(float *w_master, void *w_model, const void *g, float *v, float lr,
                      float mom, float wd, gdraa_stream_t s);

/*
 * Bucketed calls ("synchronizations ... as late as the DL needs",
 * P:189): the same collectives on the element range [first, first + count) of the
 * registered buffers, so a caller can reduce and apply each gradient bucket as soon as
 * the backward pass has produced it, on a side stream, overlapping the rest of the
 * backward.  Every rank must issue the same sequence of ranges.  The owner partition
 * (gdraa_shard) applies to the range: rank r owns [first + off_r, first + off_r + len_r)
 * with off_r/len_r = gdraa_shard(world, r, count) -- so v (and w_master) must be stepped
 * with the same bucketing every iteration.
 *   w, g, v, buf, w_master, w_model: the base pointers as registered / allocated.
 *   first: multiple of 8 (16-byte aligned for bf16 too); count >= 1; first + count <= n.
 * Errors as the whole-buffer calls, plus EINVAL for a bad range.  GDRAA_MAX_CTAS caps
 * the CTAs per call so that bucket kernels leave SMs to the concurrent backward.
 */
int gdraa_allreduce_mean_range(void *buf, size_t first, size_t count, gdraa_stream_t s);
int gdraa_sgd_step_range(float *w, const void *g, float *v, size_t first, size_t count,
                         float lr, float mom, float wd, gdraa_stream_t s);
int gdraa_sgd_step_mp_range(float *w_master, void *w_model, const void *g, float *v,
                            size_t first, size_t count, float lr, float mom, float wd,
                            gdraa_stream_t s);

/*
 * Bucket sets (SURVEY §8(f) NEXT-3 "keeping two syncs per bucket-set"; P:189 the
 * synchronizations come "as late as the DL needs"; Alg. 1 line 153 = the 1st
 * synchronization, line 166 = the 2nd).  The calls of one iteration's buckets each need
 * their own 2nd synchronization -- bucket k may be reduced only once every rank's
 * backward has produced it -- but the 1st (every peer's broadcast into our buffers has
 * landed, every peer has finished reading our g) is needed only before the next forward
 * pass reads w and the next backward overwrites g.  Between gdraa_bucket_set_begin and
 * gdraa_bucket_set_end every collective call (whole-buffer or _range, any mode) runs its
 * 2nd synchronization and its data movement as usual but defers its 1st; _end performs
 * one 1st synchronization for all of them.  A set of K two-shot calls thus counts K + 1
 * device barriers in sync_waits instead of 2K (small-message calls, which carry both
 * synchronisations with their data, are unchanged).
 *
 * gdraa_bucket_set_begin -- open a set (local, host only; enqueues nothing).
 * Errors: ESTATE (not initialised, or a set is already open).
 *
 * gdraa_bucket_set_end -- close the set (collective: every rank closes it after the same
 * calls).  Enqueues on s, ordered after every call of the set (the cross-stream rule
 * above), one small kernel: a system-scope fence of the set's pushes, one exit flag to
 * each peer, a wait for each peer's.  Nothing is enqueued at world 1.  Work after it on
 * s sees every result of the set on every rank.
 * Errors: ESTATE (no set open), ETIMEOUT (sticky), ECUDA.
 *
 * Inside a set:
 *  - The results of a call (w / buf / w_model over its range; v and w_master on the
 *    owner shard) are complete on every rank only after gdraa_bucket_set_end; do not
 *    read them, or pass them to another call, before that.
 *  - The calls of one set must write disjoint element ranges of every destination
 *    buffer (EINVAL otherwise: an overlapping range would read data still in flight).
 *  - g must not be overwritten before gdraa_bucket_set_end has completed (peers may
 *    still be reading it).
 *  - gdraa_finalize with a set still open runs the set's exit barrier first (so that
 *    the peers' gdraa_bucket_set_end completes), then leaves as usual.
 */
int gdraa_bucket_set_begin(void);
int gdraa_bucket_set_end(gdraa_stream_t s);

/*
 * gdraa_bucket_set_begin_streamed -- open a STREAMED bucket set: the same semantics as
 * gdraa_bucket_set_begin (results complete at gdraa_bucket_set_end, disjoint destination
 * ranges), served by ONE persistent kernel instead of one kernel per call.  The set's
 * first call launches that kernel, with `ctas` CTAs per rank, on a stream of the
 * library's own, ordered after the previous collective and after the first call's
 * stream reaches the call (so it holds no SMs before the first bucket is final); each
 * call then only describes
 * its bucket with three stream memory operations (cuStreamWriteValue64) on the caller's
 * stream, which take effect when that stream reaches the call -- i.e. when the bucket's
 * gradient is final -- and the kernel reduces, updates and broadcasts each bucket as its
 * description arrives, in call order, with one entry barrier per bucket and one exit
 * barrier for the set.  No launch, grid drain or exit barrier per bucket.
 *   ctas: >= 1, capped at the co-resident maximum.  The kernel holds these SMs until the
 *         set ends, so they must leave enough SMs to the work that produces the buckets
 *         (e.g. 32 of 148 beside a backward pass).
 * Rules beyond gdraa_bucket_set_begin's:
 *  - every call of the set uses the buffers, mode (mean / sgd / mp), gradient dtype and
 *    lr / mom / wd of its first call (EINVAL otherwise); at most 511 calls per set;
 *  - every call is served by the two-shot data path (the small-message kernels are not
 *    used inside a streamed set); the results are the same bits;
 *  - nothing may wait for the set's completion before gdraa_bucket_set_end has been
 *    issued (the kernel is still waiting for buckets): no cudaDeviceSynchronize, no wait
 *    on the set's streams; gdraa_get_stats returns ESTATE while such a set is open;
 *  - not available in gated mode (ESTATE); world 1 behaves as gdraa_bucket_set_begin;
 *  - not capturable into a CUDA graph (the kernel runs on the library's own stream);
 *  - gdraa_finalize with such a set open closes it on the stream of its last call.
 * Errors: ESTATE (not initialised, set already open, gated), EINVAL (ctas < 1), ECUDA.
 */
int gdraa_bucket_set_begin_streamed(int ctas);

/*
 * gdraa_poly_lr -- the paper's "poly" learning-rate policy with "gamma is 1" read as
 * the power: lr0 * (1 - iter/max_iter)^power, in double, rounded
 * once to float; 0 for iter >= max_iter; -1 if max_iter == 0.  Pure host function.
 */
float gdraa_poly_lr(float lr0, uint64_t iter, uint64_t max_iter, float power);

/*
 * gdraa_shard -- the owner-shard partition ("Divide D(i) by N"; AMB-8):
 *   c = ceil(n/world); len = roundup(c, GDRAA_SHARD_QUANTUM);
 *   off_r = min(rank*len, n); len_r = min(len, n - off_r).
 * Pure host function; usable before gdraa_init.  off/len: host pointers (outputs).
 * Errors: EINVAL (n == 0, world or rank out of range, NULL outputs).
 */
int gdraa_shard(int world, int rank, size_t n, size_t *off, size_t *len);

/*
 * gdraa_small_message_bytes -- the largest gdraa_allreduce_mean payload (n * element
 * size, bytes per rank) served by the small-message path at this world size (SURVEY
 * §8(f) NEXT-2): every rank pushes its whole buffer to every peer as 16-byte entries
 * that carry the call's epoch flag, so the data's arrival is its own synchronisation
 * and no device barrier runs; the fold order and rounding -- hence the result, bit for
 * bit -- are those of the two-shot kernel.  Default 4 MiB / (world - 1) (measured
 * crossover); GDRAA_LL_MAX_BYTES overrides it, 0 disables the path.  Returns 0 for
 * world == 1 or out of range.  Pure host function.
 */
size_t gdraa_small_message_bytes(int world);

/*
 * gdraa_small_step_bytes -- the largest gradient payload (n * sizeof(g), bytes per rank)
 * that gdraa_sgd_step / _ex / _mp (and their _range forms, per range) serve with the
 * small-message SGD kernel at this world size.  That kernel follows the paper's own
 * data flow: every rank pushes block D(r, q) into owner q's receive slot as
 * 16-byte entries carrying the call's epoch flag (Fig. 3a), the owner folds in rank
 * order, divides once, applies the update and pushes the updated block into every
 * rank's slot the same way (Fig. 3b), and every rank copies the blocks it receives into
 * its w.  The arrival of the entries is both synchronisations: no device barrier runs
 * and no rank touches another rank's g or w.  The result -- w' everywhere, v' on the
 * owner shard, g unchanged -- is bitwise the two-shot kernel's.
 *   world: 2..GDRAA_MAX_WORLD (0 otherwise); dtype: of g (GDRAA_F32 / GDRAA_BF16);
 *   mixed: nonzero for gdraa_sgd_step_mp (bf16 broadcast).
 * Default limit 4 MiB / (world - 1) (GDRAA_LL_SGD_MAX_BYTES overrides, 0 disables; a
 * communicator reads it once, at gdraa_init), lowered to what one sender's receive slot
 * (gdraa_small_message_bytes) can hold.  Pure host function (reads the environment).
 */
size_t gdraa_small_step_bytes(int world, int dtype, int mixed);

typedef struct {
    uint64_t calls;            /* collective calls completed on the device (device counter) */
    uint64_t sync_waits;       /* device barrier completions: 2 per call when world >= 2
                                  (1 per call inside a bucket set, + 1 per
                                  gdraa_bucket_set_end)                                      */
    uint64_t rs_bytes_in;      /* algorithmic reduce bytes pulled from peers (Eq. 2)         */
    uint64_t rs_bytes_out;     /* algorithmic reduce bytes peers pulled from us (Eq. 1)      */
    uint64_t ag_bytes_out;     /* algorithmic broadcast bytes pushed to peers                */
    uint64_t ag_bytes_in;      /* algorithmic broadcast bytes peers pushed to us             */
    uint64_t adds;             /* aggregation adds (Eq. 3, first term)                       */
    uint64_t divides;          /* aggregation divides (Eq. 3, second term)                   */
    uint64_t launches;         /* kernels launched by this library                           */
    uint64_t ll_calls;         /* calls served by a small-message path (allreduce_mean below
                                  gdraa_small_message_bytes, sgd_step below
                                  gdraa_small_step_bytes), whose synchronisation travels
                                  with the data (no device barrier; not in sync_waits)       */
    uint64_t iter_done;        /* this rank's "IterDone" flag as the job server sees
                                  it in the shared go/done page: written by the last CTA of
                                  every call's kernel = device calls completed             */
    uint64_t iter_start;       /* this rank's "IterStart" flag in the same page (gated mode
                                  launches call e only once it reads >= e)                 */
} gdraa_stats_t;

/*
 * gdraa_get_stats -- counters of this rank since gdraa_init.  Synchronises the device
 * to read the device-side counters.  out: host pointer.  Errors: EINVAL, ESTATE, ECUDA.
 */
int gdraa_get_stats(gdraa_stats_t *out);

/*
 * gdraa_finalize -- leave the communicator: synchronises the device, unmaps peer
 * buffers, frees the signal pads, tells the job server goodbye.  Returns a sticky
 * error if one is pending (the state is released either way).
 */
int gdraa_finalize(void);

/* Thread-local description of the last error on this thread ("" if none). */
const char *gdraa_last_error(void);

/* Library version string (also names the compile target, e.g. "sm_100a"). */
const char *gdraa_version(void);

/*
 * Virtual ranks on ONE GPU (test and emulation entry points).  The same device code
 * as above runs `world` ranks inside ONE cooperative kernel launch: rank r's CTAs use
 * rank p's buffers through plain device pointers instead of IPC mappings, and the two
 * synchronisations run through per-rank signal pads in local memory.  This is how
 * N > 1 is exercised on a single B200 (profiling guide: never run mutually waiting
 * kernels as separate launches on one GPU).  No gdraa_init is needed.
 *   world: 1..GDRAA_MAX_WORLD; bufs/w/g/v: HOST arrays of `world` device pointers
 *   (rank p's buffer at index p), all distinct, 16-byte aligned, n elements.
 *   Semantics per rank are exactly those of gdraa_allreduce_mean / gdraa_sgd_step.
 * Errors: EINVAL, ECUDA, ETIMEOUT (returned by a later vr call).
 */
int gdraa_vr_allreduce_mean(int world, void *const *bufs, size_t n, int dtype,
                            gdraa_stream_t s);
int gdraa_vr_sgd_step(int world, float *const *w, const void *const *g, float *const *v,
                      size_t n, int dtype, float lr, float mom, gdraa_stream_t s);
int gdraa_vr_sgd_step_ex(int world, float *const *w, const void *const *g, float *const *v,
                         size_t n, int dtype, float lr, float mom, float wd, gdraa_stream_t s);
/* w_master: HOST array of per-rank f32 master buffers; w_model: per-rank bf16 buffers. */
int gdraa_vr_sgd_step_mp(int world, float *const *w_master, void *const *w_model,
                         const void *const *g, float *const *v, size_t n, int dtype, float lr,
                         float mom, float wd, gdraa_stream_t s);

/*
 * Bucketed virtual-rank calls (NEXT-3 on one GPU): the calls above on the element
 * range [first, first + count) of every rank's n-element buffers, with the range's own
 * owner partition (rank r owns [first + off_r, +len_r), off_r/len_r = gdraa_shard(world,
 * r, count)) -- exactly the semantics of gdraa_allreduce_mean_range / gdraa_sgd_step_range
 * / gdraa_sgd_step_mp_range, so the per-range owner rule is testable on one GPU.
 *   first: multiple of 8; count >= 1; first + count <= n.  Other arguments as above.
 * Errors: EINVAL (bad range, null arrays), ECUDA, ETIMEOUT (returned by a later call).
 */
int gdraa_vr_allreduce_mean_range(int world, void *const *bufs, size_t n, int dtype,
                                  size_t first, size_t count, gdraa_stream_t s);
int gdraa_vr_sgd_step_range(int world, float *const *w, const void *const *g, float *const *v,
                            size_t n, int dtype, size_t first, size_t count, float lr, float mom,
                            float wd, gdraa_stream_t s);
int gdraa_vr_sgd_step_mp_range(int world, float *const *w_master, void *const *w_model,
                               const void *const *g, float *const *v, size_t n, int dtype,
                               size_t first, size_t count, float lr, float mom, float wd,
                               gdraa_stream_t s);

/*
 * Bucket sets over virtual ranks (the semantics of gdraa_bucket_set_begin / _end for the
 * gdraa_vr_* calls of this `world` on the current device; one open set per world).
 * Errors: EINVAL (world), ESTATE (set already open / not open), ECUDA, ETIMEOUT.
 */
int gdraa_vr_bucket_set_begin(int world);
int gdraa_vr_bucket_set_end(int world, gdraa_stream_t s);
/* The streamed form for virtual ranks: one cooperative persistent launch of ctas x world
 * CTAs serves the set's gdraa_vr_* calls (rules of gdraa_bucket_set_begin_streamed). */
int gdraa_vr_bucket_set_begin_streamed(int world, int ctas);

#ifdef __cplusplus
}
#endif
#endif /* GDRAA_H */
