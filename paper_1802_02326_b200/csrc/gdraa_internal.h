// gdraa_internal.h -- types shared by the host runtime (gdraa_runtime.cu) and the
// sm_100a kernels (gdraa_kernels.cu).  Not part of the ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "gdraa.h"

namespace gdraa {

constexpr int kMaxWorld = GDRAA_MAX_WORLD;
constexpr uint64_t kQuantum = GDRAA_SHARD_QUANTUM;

// Signal pad of one rank (device memory, exported to peers over CUDA IPC).  Peers write
// only `entry[their rank]` and `exit[their rank]`; everything from `epoch` on is written
// by the owning rank only.  Each array sits on its own 128-byte line.
struct alignas(128) Pad {
    uint64_t entry[kMaxWorld];     // paper "2nd synchronization" (Alg. 1)
    uint64_t _p0[16 - kMaxWorld];
    uint64_t exit[kMaxWorld];      // paper "1st synchronization" (Alg. 1)
    uint64_t _p1[16 - kMaxWorld];
    uint64_t epoch;                // completed collective calls (device-resident)
    uint64_t calls;
    uint64_t sync_waits;
    uint32_t arrive;               // CTA arrival counter of the running call
    uint32_t next;                 // next work chunk of the running call (dynamic schedule)
    uint64_t ll_calls;             // calls served by the small-message (LL) path
    uint64_t mc_calls;             // calls that used the multicast barrier (tools/tune.cu A/B)
    uint64_t _p3[10];
#ifdef GDRAA_EXPERIMENTAL
    // Distributed exit (kFlagDistExit, tools/tune.cu only): every CTA of sender p adds the
    // elements it finished (pulled, folded, pushed) to recv_done[p] of every peer after its
    // fence; the owner's last CTA waits until recv_done[p] reaches recv_expect[p] + len_p.
    uint64_t recv_done[kMaxWorld];     // written by peers (remote atomics)
    uint64_t _p4[16 - kMaxWorld];
    uint64_t recv_expect[kMaxWorld];   // written by the owner's last CTA
    uint64_t _p5[16 - kMaxWorld];
#endif
};
static_assert(sizeof(Pad) % 128 == 0, "pad layout");

// Host-mapped failure record (written by the device on a barrier timeout).
struct ErrBlock {
    volatile int32_t code;                   // 0 or GDRAA_ETIMEOUT
    volatile int32_t phase;                  // 1 = entry barrier, 2 = exit barrier
    volatile uint32_t missing[kMaxWorld];    // missing[p] = 1 if rank p never arrived
    volatile int32_t vrank;                  // the (virtual) rank that timed out
};

// Streamed bucket sets (gdraa_bucket_set_begin_streamed): one persistent kernel serves
// every bucket of the set.  The host describes bucket k with stream memory operations
// on the caller's stream (so they take effect when the caller's stream reaches the call,
// i.e. once the bucket's gradient is final): first[k], count[k], then ready[k] =
// set_tag(gen, k); gdraa_bucket_set_end posts ready[K] = set_close(gen).  Tags carry the
// set's generation, so values left from earlier sets are never mistaken for this one's.
constexpr int kSetMax = 512;
struct SetDesc {
    uint64_t ready[kSetMax];
    uint64_t first[kSetMax];
    uint64_t count[kSetMax];
};
__host__ __device__ constexpr uint64_t set_tag(uint32_t gen, uint32_t k) {
    return (static_cast<uint64_t>(gen) << 32) | (k + 1u);
}
__host__ __device__ constexpr uint64_t set_close(uint32_t gen) {
    return (static_cast<uint64_t>(gen) << 32) | 0xFFFFFFFFu;
}

// Kernel parameters (passed by value).  Row vr describes virtual rank vr: one row in
// multi-process mode (gridDim.y == 1, rank = rank0), `world` rows in the single-GPU
// virtual-rank mode (gridDim.y == world, rank = blockIdx.y).
struct KParams {
    int world;
    int rank0;
    uint64_t n;          // elements
    uint64_t blk;        // shard length (Q-aligned ceil(n/world))
    float lr, mom;
    float wd;            // weight decay (0: no decay term is formed)
    uint64_t timeout_ns;
    const void *src[kMaxWorld][kMaxWorld];   // [vr][p]: rank p's g (or buf) seen from vr
    void *dst[kMaxWorld][kMaxWorld];         // [vr][p]: rank p's w (or buf) seen from vr
    float *v[kMaxWorld];                     // [vr]: local momentum buffer
    float *wm[kMaxWorld];                    // [vr]: local fp32 master weights (kSgdMp)
    Pad *pad[kMaxWorld][kMaxWorld];          // [vr][p]: rank p's pad seen from vr
    // Small-message path (kMean only): rank p's LL receive buffer seen from vr, laid out
    // [2 parities][world senders][ll_pairs] x uint4 {word0, flag, word1, flag}.
    uint4 *ll[kMaxWorld][kMaxWorld];
    uint64_t ll_pairs;                       // capacity in 8-byte payload pairs per sender
    uint32_t ll_sleep_ns;                    // LL poll back-off cap (0 = spin)
    ErrBlock *err;                           // host-mapped (device alias)
    volatile uint64_t *done[kMaxWorld];      // host-mapped done flags (device alias) or null
    const volatile int32_t *abort;           // host-mapped job-server abort flag, or null:
                                             // spins give up early once a rank has died
    uint32_t flags;                          // kFlag* bits (launch-variant switches)
    // streamed bucket set (gdraa_tma_set_kernel only): the bucket descriptors (shared by
    // the virtual ranks of a vr launch), per-row chunk counters [kSetMax], the generation
    const SetDesc *sdesc;
    uint32_t *snext[kMaxWorld];
    uint32_t sgen;
#ifdef GDRAA_EXPERIMENTAL
    // Measured-and-rejected variants of the two-shot TMA kernel, compiled only into
    // tools/tune.cu for the A/B, never into the library.  NVLS multicast:
    // mc_dst[vr] = multicast VA of the broadcast buffer (one multimem.st reaches every
    // member of the group); mc_bar[vr] = multicast VA of a {entry, exit} u64 counter block
    // whose local copy is bar_local[vr] (one multimem.red per rank and barrier).
    void *mc_dst[kMaxWorld];
    uint64_t *mc_bar[kMaxWorld];
    uint64_t *bar_local[kMaxWorld];
#endif
#ifdef GDRAA_TRACE
    uint64_t *trace;                         // tools/tune.cu only: %globaltimer stamps
#endif
};

// kMean: dst = mean (allreduce_mean).  kSgd: dst = w' (fp32, replicated w).
// kSgdMp: fp32 master w sharded like v (p.wm), dst = bf16 RNE(w') model copy (NEXT-1).
enum Mode { kMean = 0, kSgd = 1, kSgdMp = 2 };

// KParams::flags.  kFlagCtaFence: at exit, one fence.acq_rel.sys per CTA after
// __syncthreads() instead of one per thread (default; GDRAA_EXIT_FENCE=thread clears it).
constexpr uint32_t kFlagCtaFence = 1u;
// Experimental (tools/tune.cu only, GDRAA_EXPERIMENTAL): kFlagMcPeersOnly -- the mc_dst
// group holds the N-1 peers only, the own copy is stored locally as well; kFlagDistExit
// -- the exit synchronisation without the last-CTA relay, each CTA telling every peer
// directly how many elements it finished (measured slower: DESIGN.md §11).
constexpr uint32_t kFlagMcPeersOnly = 2u;
constexpr uint32_t kFlagDistExit = 4u;
// kFlagDeferExit: the call is inside a bucket set (gdraa_bucket_set_begin/_end): the
// two-shot kernels skip the exit fence and the exit flag exchange (they still run the
// entry barrier); launch_gdraa_exit performs the set's single 1st synchronization.
constexpr uint32_t kFlagDeferExit = 8u;
uint32_t env_kernel_flags();
constexpr int kModes = 3;

// Launch the fused kernel.  grid_x CTAs per (virtual) rank; vr_rows = gridDim.y.
// cooperative: use cudaLaunchCooperativeKernel (required when vr_rows > 1).
cudaError_t launch_gdraa(const KParams &p, int dtype, int mode, int vr_rows,
                         bool cooperative, cudaStream_t s, int *grid_x_out);

// The deferred exit barrier of a bucket set: fence + exit-flag exchange at the epoch of
// the last call, one 32-thread CTA per (virtual) rank (vr_rows = gridDim.y).
cudaError_t launch_gdraa_exit(const KParams &p, int vr_rows, bool cooperative, cudaStream_t s);

// Max co-resident CTAs of the kernel for (dtype, mode, world) on this device.
int max_ctas(int dtype, int mode, int world);

// The TMA-staged variant of launch_gdraa (same semantics and results).
cudaError_t launch_gdraa_tma(const KParams &p, int dtype, int mode, int vr_rows,
                             bool cooperative, cudaStream_t s, int *grid_x_out);
// The persistent bucket-set kernel (world >= 2, any mode / dtype): p.dst / p.src / p.v /
// p.wm are the BASE pointers of the buffers; buckets arrive through p.sdesc.  ctas: CTAs
// per (virtual) rank (capped at the co-resident maximum).
cudaError_t launch_gdraa_tma_set(const KParams &p, int dtype, int mode, int vr_rows,
                                 bool cooperative, cudaStream_t s, int ctas);
// Whether the runtime launches the TMA-staged kernel for this call (measured choice;
// GDRAA_KERNEL=tma|lsu forces it).
bool use_tma_kernel(int dtype, int mode, int world);

// Small-message allreduce_mean ("LL": data carries its own epoch flags, no barriers).
// Requires n * elem_size <= 8 * p.ll_pairs.
cudaError_t launch_gdraa_ll(const KParams &p, int dtype, int vr_rows, bool cooperative,
                            cudaStream_t s);
// Small-message fused SGD step (kSgd / kSgdMp): gradient blocks and updated blocks travel
// as LL entries through the same receive areas; the data carries both synchronisations.
// Requires ll_sgd_fits(p.blk, ...).
cudaError_t launch_gdraa_ll_sgd(const KParams &p, int dtype, int mode, int vr_rows,
                                bool cooperative, cudaStream_t s);
// Whether a shard of blk elements fits one sender's LL slot (gradient + broadcast part).
bool ll_sgd_fits(uint64_t blk, int dtype, int mode, uint64_t ll_pairs);
// Largest gdraa_sgd_step gradient payload (n * sizeof(g), bytes per rank) served by the
// small-message SGD path (GDRAA_LL_SGD_MAX_BYTES overrides, 0 disables).
uint64_t ll_sgd_limit_bytes(int world);

// Largest allreduce_mean payload (bytes per rank) served by the LL path: the measured
// crossover with the two-shot kernel is ~4 MiB at N=2 and ~1.5 MiB at N=4
// (profiles/r15_sweep*_ll*.jsonl), i.e. ~4 MiB / (N-1) as the LL bytes grow with N-1.
// GDRAA_LL_MAX_BYTES overrides it (0 disables the LL path).
uint64_t ll_limit_bytes(int world);
constexpr uint64_t kLLBaseBytes = 4ull << 20;
constexpr uint64_t kLLSgdBaseBytes = 4ull << 20;

}  // namespace gdraa
