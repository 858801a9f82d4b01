// gdraa_kernels.cu -- sm_100a kernels of the GDRAA hot path (arxiv 1802.02326).
//
// ONE kernel per collective call does the whole of Algorithm 1's communication part
// plus the model update for the shard this rank owns:
//
//   a2  entry barrier   = paper "2nd synchronization" (Alg. 1)
//   a3  reduce          = pull block r of every rank's D(i) over NVLink (Fig. 3a)
//   a4  aggregation     = left fold in ascending rank, one division by N (Eq. 3)
//   a5  update          = momentum SGD on the owner shard      [sgd mode]
//   a6  broadcast       = push the averaged/updated block into every rank (Fig. 3b)
//   a7  exit barrier    = paper "1st synchronization" (Alg. 1)
//
// Rank r's CTAs read every peer's shard r through CUDA-IPC mapped pointers (coalesced
// loads, all N sources in flight per thread), and store the result shard to all N
// ranks with coalesced 128-bit stores (posted NVLink writes).  Every thread owns 4
// consecutive elements per vector, so each warp-level load / store instruction covers
// one contiguous span (256 B of bf16 g, 512 B of fp32 g/w/v): no partial-sector NVLink
// writes.  Shard r is read and written by rank r only, so in-place allreduce is race
// free chunk by chunk.  Every rounding is pinned (__fadd_rn / __fdiv_rn / __fmul_rn /
// __fsub_rn are never contracted into FMA), so the result is bitwise the CPU oracle's.
//
// Tensor cores are not used: there is no contraction on this path.
#include <cuda_bf16.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <utility>

#include "gdraa_internal.h"

namespace gdraa {
namespace {

// ---------------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// The h-th 8-byte half of a bf16 output vector (4 or 8 values).
__device__ __forceinline__ void set_half(uint2 &o, int, uint2 v) { o = v; }
__device__ __forceinline__ void set_half(uint4 &o, int h, uint2 v) {
    if (h == 0) {
        o.x = v.x;
        o.y = v.y;
    } else {
        o.z = v.x;
        o.w = v.y;
    }
}
// NVLS multicast stores (the address is a multicast VA: the switch delivers to every
// member); reached only from the experimental multicast branch (mc_dst != null).
__device__ __forceinline__ void mc_st(uint4 *p, uint4 v) {
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(__uint_as_float(v.x)),
                 "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
                 : "memory");
}
__device__ __forceinline__ void mc_st(uint2 *p, uint2 v) {
    asm volatile("multimem.st.global.v2.bf16x2 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y)
                 : "memory");
}
__device__ __forceinline__ void mc_st_bf16(uint2 *p, uint2 v) { mc_st(p, v); }
__device__ __forceinline__ void mc_st_bf16(uint4 *p, uint4 v) {
    asm volatile("multimem.st.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
#ifdef GDRAA_EXPERIMENTAL   // tools/tune.cu only
__device__ __forceinline__ void red_add_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void mc_red_add_release(uint64_t *p, uint64_t v) {
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
#endif
__device__ __forceinline__ void fence_acq_rel_sys() {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint64_t global_timer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Streaming loads: data is touched once, keep it out of L1.
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_stream(const uint2 *p) {
    uint2 r;
    asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_vec(uint4 *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_vec(uint2 *p, uint2 v) {
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

// Spin until *flag >= target, bounded by timeout_ns of %globaltimer, and abandoned early
// if the job server has flagged a dead rank (host-mapped, read every 4096 polls).
__device__ __forceinline__ bool wait_geq(const uint64_t *flag, uint64_t target,
                                         uint64_t timeout_ns,
                                         const volatile int32_t *abort = nullptr) {
    if (ld_relaxed_sys(flag) < target) {
        const uint64_t t0 = global_timer_ns();
        uint32_t polls = 0;
        while (ld_relaxed_sys(flag) < target) {
            if (global_timer_ns() - t0 > timeout_ns) return false;
            if (abort != nullptr && (++polls & 4095u) == 0 && *abort != 0) return false;
        }
    }
    (void)ld_acquire_sys(flag);   // acquire pattern: orders our later reads after it
    return true;
}

__device__ __forceinline__ void report_timeout(ErrBlock *err, int phase, int peer, int vr) {
    err->missing[peer] = 1u;
    err->phase = phase;
    err->vrank = vr;
    __threadfence_system();
    err->code = GDRAA_ETIMEOUT;
}

// Phase timestamps for tools/tune.cu (compiled out of the library).
#ifdef GDRAA_TRACE
#define GDRAA_STAMP(k)                                                                   \
    do {                                                                                 \
        if (p.trace) p.trace[((epoch % 64) * kMaxWorld + vr) * 8 + (k)] = global_timer_ns(); \
    } while (0)
// slots 5/6: earliest / latest end of any CTA's data loop (atomic min / max), reset with
// the kernel-start stamp
#define GDRAA_STAMP_START()                                                              \
    do {                                                                                 \
        if (p.trace) {                                                                   \
            uint64_t *t_ = p.trace + ((epoch % 64) * kMaxWorld + vr) * 8;                \
            t_[5] = ~0ull;                                                               \
            t_[6] = 0;                                                                   \
            t_[0] = global_timer_ns();                                                   \
        }                                                                                \
    } while (0)
#define GDRAA_STAMP_DONE()                                                               \
    do {                                                                                 \
        __syncthreads();                                                                 \
        if (p.trace && threadIdx.x == 0) {                                               \
            unsigned long long *t_ = reinterpret_cast<unsigned long long *>(             \
                p.trace + ((epoch % 64) * kMaxWorld + vr) * 8);                          \
            const unsigned long long now_ = global_timer_ns();                           \
            atomicMin(t_ + 5, now_);                                                     \
            atomicMax(t_ + 6, now_);                                                     \
        }                                                                                \
    } while (0)
#else
#define GDRAA_STAMP(k) \
    do {               \
    } while (0)
#define GDRAA_STAMP_DONE() \
    do {                   \
    } while (0)
#define GDRAA_STAMP_START() \
    do {                    \
    } while (0)
#endif

// ---------------------------------------------------------------------------------
// Element access: a vector is 4 consecutive elements; Raw is its storage in g / buf.
// ---------------------------------------------------------------------------------
constexpr int E = 4;

template <typename TG> struct Elem;
template <> struct Elem<float> {
    using Raw = uint4;                       // 16 bytes
    __device__ __forceinline__ static void widen(Raw r, float (&f)[E]) {
        f[0] = __uint_as_float(r.x);
        f[1] = __uint_as_float(r.y);
        f[2] = __uint_as_float(r.z);
        f[3] = __uint_as_float(r.w);
    }
    __device__ __forceinline__ static Raw narrow(const float (&f)[E]) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                          __float_as_uint(f[3]));
    }
    __device__ __forceinline__ static float load1(const void *p, uint64_t i) {
        return static_cast<const float *>(p)[i];
    }
    __device__ __forceinline__ static void store1(void *p, uint64_t i, float m) {
        static_cast<float *>(p)[i] = m;
    }
};
template <> struct Elem<__nv_bfloat16> {
    using Raw = uint2;                       // 8 bytes
    // bf16 -> fp32 is exact: the 16 bits become the high half (AMB-13).
    __device__ __forceinline__ static float lo(uint32_t u) { return __uint_as_float(u << 16); }
    __device__ __forceinline__ static float hi(uint32_t u) {
        return __uint_as_float(u & 0xFFFF0000u);
    }
    __device__ __forceinline__ static void widen(Raw r, float (&f)[E]) {
        f[0] = lo(r.x); f[1] = hi(r.x); f[2] = lo(r.y); f[3] = hi(r.y);
    }
    // fp32 -> bf16 round to nearest even (finite values).
    __device__ __forceinline__ static uint32_t pack(float a, float b) {
        const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(a));
        const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(b));
        return l | (h << 16);
    }
    __device__ __forceinline__ static Raw narrow(const float (&f)[E]) {
        return make_uint2(pack(f[0], f[1]), pack(f[2], f[3]));
    }
    __device__ __forceinline__ static float load1(const void *p, uint64_t i) {
        return lo(static_cast<const uint16_t *>(p)[i]);
    }
    __device__ __forceinline__ static void store1(void *p, uint64_t i, float m) {
        static_cast<__nv_bfloat16 *>(p)[i] = __float2bfloat16_rn(m);
    }
};

// Aggregation: s = x_0; s = fl(s + x_p) for p = 1..N-1; m = fl(s / N).
// For N a power of two, fl(s / N) and fl(s * 2^-k) round the same real number s * 2^-k
// once, so they are the same bits; the multiply avoids __fdiv_rn's reciprocal
// refinement (FFMA) and its slow-path call.  Other N: one correctly rounded division.
template <int WORLD>
__device__ __forceinline__ float average(const float (&x)[WORLD]) {
    float s = x[0];
#pragma unroll
    for (int q = 1; q < WORLD; ++q) s = __fadd_rn(s, x[q]);
    if constexpr (WORLD == 1)
        return s;                                   // fl(s / 1) = s
    else if constexpr ((WORLD & (WORLD - 1)) == 0)
        return __fmul_rn(s, 1.0f / static_cast<float>(WORLD));
    else
        return __fdiv_rn(s, static_cast<float>(WORLD));
}

// Update: v = fl(fl(mom*v) + m); w = fl(w - fl(lr*v)).  With weight decay
// (P:246): m is first replaced by fl(m + fl(wd*w)); wd == 0 forms no decay term.
__device__ __forceinline__ void sgd(float m, float lr, float mom, float wd, float &w, float &v) {
    if (wd != 0.0f) m = __fadd_rn(m, __fmul_rn(wd, w));
    const float t = __fmul_rn(mom, v);
    v = __fadd_rn(t, m);
    const float u = __fmul_rn(lr, v);
    w = __fsub_rn(w, u);
}

__device__ __forceinline__ float4 ld_f4(const float *p) {
    const uint4 r = ld_stream(reinterpret_cast<const uint4 *>(p));
    return make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z),
                       __uint_as_float(r.w));
}
__device__ __forceinline__ uint4 as_u4(float a, float b, float c, float d) {
    return make_uint4(__float_as_uint(a), __float_as_uint(b), __float_as_uint(c),
                      __float_as_uint(d));
}

// ---------------------------------------------------------------------------------
// The fused kernel.  TG: gradient / buffer element type; WORLD: N; MODE: kMean or
// kSgd; U: vectors per thread in flight per iteration (memory-level parallelism);
// THREADS x MINB: CTA size and minimum co-resident CTAs per SM (register budget).
// ---------------------------------------------------------------------------------
template <typename TG, int WORLD, int MODE, int U, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
gdraa_kernel(const __grid_constant__ KParams p) {
    using EL = Elem<TG>;
    using Raw = typename EL::Raw;
    const int vr = blockIdx.y;
    const int rank = p.rank0 + vr;
    Pad *mine = p.pad[vr][rank];
    __shared__ int s_abort;
    __shared__ int s_last;

    // All CTAs read the epoch before any of them can arrive at the exit counter, and the
    // last CTA updates it only after every CTA arrived: one consistent value per call.
    // Programmatic dependent launch: this grid may have been scheduled while the previous
    // kernel on the stream was finishing; wait for its completion (a no-op otherwise).
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t epoch = *reinterpret_cast<volatile uint64_t *>(&mine->epoch) + 1;
    if (threadIdx.x == 0) s_abort = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) GDRAA_STAMP_START();

    // a2: "2nd synchronization" -- every peer's D(i) is final (stream-ordered after its
    // backward) before anyone reads it or writes into it.
    if (WORLD > 1) {
        if (blockIdx.x == 0 && threadIdx.x < WORLD && threadIdx.x != rank)
            st_release_sys(&p.pad[vr][threadIdx.x]->entry[rank], epoch);
        __syncthreads();
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            if (!wait_geq(&mine->entry[threadIdx.x], epoch, p.timeout_ns, p.abort)) {
                report_timeout(p.err, 1, threadIdx.x, vr);
                s_abort = 1;
            }
        }
        __syncthreads();
        if (s_abort) return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) GDRAA_STAMP(1);

    // a1: this rank's block D(., r), Q-aligned ceil partition (AMB-8).
    const uint64_t off = min(static_cast<uint64_t>(rank) * p.blk, p.n);
    const uint64_t len = min(p.blk, p.n - off);
    const uint64_t nvec = len / E;

    constexpr bool kUpdate = MODE != kMean;
    const float lr = p.lr, mom = p.mom, wd = p.wd;
    float *const vloc = p.v[vr];
    // the fp32 weights the update reads: the replicated w (kSgd) or the local master
    // shard (kSgdMp, whose broadcast carries only a bf16 model copy)
    float *const wloc = MODE == kSgdMp ? p.wm[vr] : static_cast<float *>(p.dst[vr][rank]);
    const Raw *src[WORLD];
#pragma unroll
    for (int q = 0; q < WORLD; ++q)
        src[q] = reinterpret_cast<const Raw *>(static_cast<const TG *>(p.src[vr][q]) + off);

    // Vectors k0, k0 + THREADS, ..., k0 + (UU-1) * THREADS of the shard.
    auto process = [&](uint64_t k0, auto ucount) {
        constexpr int UU = decltype(ucount)::value;
        Raw raw[UU][WORLD];
        float4 wv[UU], vv[UU];
        // a3: reduce -- all N sources in flight at once (local HBM + N-1 NVLink peers).
#pragma unroll
        for (int u = 0; u < UU; ++u) {
            const uint64_t k = k0 + u * THREADS;
#pragma unroll
            for (int q = 0; q < WORLD; ++q) raw[u][q] = ld_stream(src[q] + k);
            if (kUpdate) {
                wv[u] = ld_f4(wloc + off + k * E);
                vv[u] = ld_f4(vloc + off + k * E);
            }
        }
        // a4 (+ a5): aggregate (and update) in registers; a6: push to every rank.
#pragma unroll
        for (int u = 0; u < UU; ++u) {
            const uint64_t e0 = off + (k0 + u * THREADS) * E;
            float x[WORLD][E];
#pragma unroll
            for (int q = 0; q < WORLD; ++q) EL::widen(raw[u][q], x[q]);
            float m[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                float col[WORLD];
#pragma unroll
                for (int q = 0; q < WORLD; ++q) col[q] = x[q][e];
                m[e] = average<WORLD>(col);
            }
            if (kUpdate) {
                float4 w = wv[u], v = vv[u];
                sgd(m[0], lr, mom, wd, w.x, v.x);
                sgd(m[1], lr, mom, wd, w.y, v.y);
                sgd(m[2], lr, mom, wd, w.z, v.z);
                sgd(m[3], lr, mom, wd, w.w, v.w);
                st_vec(reinterpret_cast<uint4 *>(vloc + e0), as_u4(v.x, v.y, v.z, v.w));
                if (MODE == kSgd) {
                    const uint4 o = as_u4(w.x, w.y, w.z, w.w);
#pragma unroll
                    for (int j = 1; j <= WORLD; ++j) {   // own copy last
                        const int q = (rank + j) % WORLD;
                        st_vec(reinterpret_cast<uint4 *>(static_cast<float *>(p.dst[vr][q]) + e0),
                               o);
                    }
                } else {   // kSgdMp: master shard stays local, bf16 copy to every rank
                    st_vec(reinterpret_cast<uint4 *>(wloc + e0), as_u4(w.x, w.y, w.z, w.w));
                    const float wf[E] = {w.x, w.y, w.z, w.w};
                    const uint2 o = Elem<__nv_bfloat16>::narrow(wf);
#pragma unroll
                    for (int j = 1; j <= WORLD; ++j) {
                        const int q = (rank + j) % WORLD;
                        st_vec(reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(p.dst[vr][q]) + e0),
                               o);
                    }
                }
            } else {
                const Raw o = EL::narrow(m);
#pragma unroll
                for (int j = 1; j <= WORLD; ++j) {
                    const int q = (rank + j) % WORLD;
                    st_vec(reinterpret_cast<Raw *>(static_cast<TG *>(p.dst[vr][q]) + e0), o);
                }
            }
        }
    };

    // Dynamic schedule: CTAs take chunks from a per-rank counter (the next index is
    // fetched while the current chunk is in flight).  A static grid-stride split left
    // the slowest CTA finishing 41 us after CTA 0 at R50 / N=2 (profiles/r07_trace_n2).
    // Big chunks (THREADS*U vectors) first; the last ~2 waves use THREADS-vector chunks
    // so the CTAs finish close together.
    const uint64_t big = static_cast<uint64_t>(THREADS) * U;
    const uint64_t tailv = 2ull * gridDim.x * THREADS;
    const uint64_t nbig = nvec > tailv ? (nvec - tailv) / big : 0;
    const uint64_t small0 = nbig * big;
    const uint64_t nchunks = nbig + (nvec - small0 + THREADS - 1) / THREADS;
    __shared__ uint32_t s_chunk[2];
    if (threadIdx.x == 0) s_chunk[0] = atomicAdd(&mine->next, 1u);
    __syncthreads();
    uint32_t c = s_chunk[0];
    int slot = 0;
    while (c < nchunks) {
        if (threadIdx.x == 0) s_chunk[slot ^ 1] = atomicAdd(&mine->next, 1u);
        if (c < nbig) {
            process(c * big + threadIdx.x, std::integral_constant<int, U>{});
        } else {
            const uint64_t k = small0 + (c - nbig) * THREADS + threadIdx.x;
            if (k < nvec) process(k, std::integral_constant<int, 1>{});
        }
        __syncthreads();
        c = s_chunk[slot ^ 1];
        slot ^= 1;
    }

    // Ragged tail of the last non-empty shard (len % 4 elements), scalar.
    if (blockIdx.x == gridDim.x - 1) {
        for (uint64_t t = nvec * E + threadIdx.x; t < len; t += THREADS) {
            const uint64_t e = off + t;
            float col[WORLD];
#pragma unroll
            for (int q = 0; q < WORLD; ++q) col[q] = EL::load1(p.src[vr][q], e);
            const float m = average<WORLD>(col);
            if (kUpdate) {
                float w = wloc[e], v = vloc[e];
                sgd(m, lr, mom, wd, w, v);
                vloc[e] = v;
                if (MODE == kSgd) {
                    for (int j = 1; j <= WORLD; ++j)
                        static_cast<float *>(p.dst[vr][(rank + j) % WORLD])[e] = w;
                } else {
                    wloc[e] = w;
                    for (int j = 1; j <= WORLD; ++j)
                        Elem<__nv_bfloat16>::store1(p.dst[vr][(rank + j) % WORLD], e, w);
                }
            } else {
                for (int j = 1; j <= WORLD; ++j) EL::store1(p.dst[vr][(rank + j) % WORLD], e, m);
            }
        }
    }

    // a7: "1st synchronization" -- our pushes are performed system-wide, then the last
    // CTA of this rank tells every peer and waits until every peer has done the same.
    if (blockIdx.x == 0 && threadIdx.x == 0) GDRAA_STAMP(2);
    GDRAA_STAMP_DONE();
    // Let the next kernel on the stream start launching; it waits for our completion
    // (griddepcontrol.wait above) before touching anything.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // Our pushes must be performed system-wide before the peers hear of them.  Either
    // every thread fences its own stores, or (kFlagCtaFence) the CTA synchronises and
    // one thread fences for all of them (release cumulativity over bar.sync).
    // N = 1: the kernel boundary orders our stores.  A call inside a bucket set
    // (kFlagDeferExit) leaves both the fence and the flag exchange to the set's
    // gdraa_exit_kernel.
    const bool defer = (p.flags & kFlagDeferExit) != 0;
    const bool cta_fence = (p.flags & kFlagCtaFence) != 0;
    if (WORLD > 1 && !cta_fence && !defer) fence_acq_rel_sys();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (WORLD > 1 && cta_fence && !defer) fence_acq_rel_sys();
        const unsigned prev = atomicAdd(&mine->arrive, 1u);
        s_last = (prev == gridDim.x - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x == 0) GDRAA_STAMP(3);
    if (WORLD > 1 && !defer) {
        if (threadIdx.x < WORLD && threadIdx.x != rank)
            st_release_sys(&p.pad[vr][threadIdx.x]->exit[rank], epoch);
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            if (!wait_geq(&mine->exit[threadIdx.x], epoch, p.timeout_ns, p.abort)) {
                report_timeout(p.err, 2, threadIdx.x, vr);
                s_abort = 1;
            }
        }
        __syncthreads();
        if (s_abort) return;
    }
    if (threadIdx.x == 0) {
        GDRAA_STAMP(4);
        mine->arrive = 0;
        mine->next = 0;
        mine->calls += 1;
        if (WORLD > 1) mine->sync_waits += defer ? 1 : 2;
        mine->epoch = epoch;
        if (p.done[vr] != nullptr) *p.done[vr] = epoch;   // job-server "IterDone" flag
    }
}

// ---------------------------------------------------------------------------------
// Small-message allreduce_mean (the latency path).  Below ~256 KiB
// the two device barriers and the pull round trip dominate, so every rank PUSHES its
// whole buffer into every peer's receive slot as 16-byte entries {word, flag, word, flag}
// ("LL" format: the epoch flag travels with the data, so the data's arrival is its own
// 2nd synchronization), then folds the N contributions in ascending rank and divides
// once -- bitwise the same result as the two-shot kernel (and the oracle).  Receive slots
// alternate by epoch parity: a rank cannot overwrite slot parity e before every peer
// finished call e-2, so no exit barrier is needed (the 1st synchronization is implied by
// the next call's data).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void st_ll(uint4 *p, uint4 v) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const uint4 *p) {
    uint4 r;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
    return r;
}

// Poll one LL entry until both flag words carry `flag`.  Bounded by timeout_ns; the
// host-mapped abort flag is read only every 1024 polls (a read per poll from thousands
// of polling threads would queue on PCIe and serialise the whole kernel).  A thread whose
// entry is not there yet backs off with __nanosleep (doubling up to max_sleep_ns; 0 = spin)
// so that tens of thousands of waiting threads do not flood L2 with polls while the
// peers' NVLink writes are trying to land there.
__device__ __forceinline__ uint4 ll_wait(const uint4 *src, uint32_t flag, uint64_t timeout_ns,
                                         const volatile int32_t *abort, uint32_t max_sleep_ns,
                                         bool &ok) {
    uint4 r = ld_ll(src);
    if (r.y == flag && r.w == flag) return r;
    const uint64_t t0 = global_timer_ns();
    uint32_t polls = 0, sleep_ns = 32;
    do {
        if (max_sleep_ns != 0) {
            __nanosleep(sleep_ns);
            sleep_ns = sleep_ns * 2 > max_sleep_ns ? max_sleep_ns : sleep_ns * 2;
        }
        r = ld_ll(src);
        if ((++polls & 1023u) == 0 &&
            (global_timer_ns() - t0 > timeout_ns || (abort != nullptr && *abort != 0))) {
            ok = false;
            break;
        }
    } while (r.y != flag || r.w != flag);
    return r;
}

// 8 payload bytes of the buffer at pair j (fewer at the ragged end; the rest is 0).
__device__ __forceinline__ uint2 load_pair(const void *buf, uint64_t j, uint64_t nbytes) {
    const uint64_t b0 = j * 8;
    if (b0 + 8 <= nbytes) return *reinterpret_cast<const uint2 *>(static_cast<const char *>(buf) + b0);
    uint32_t w[2] = {0u, 0u};
    const uint16_t *h = static_cast<const uint16_t *>(buf);   // n*s is a multiple of 2
    for (uint64_t b = b0; b < nbytes; b += 2) {
        const uint32_t k = static_cast<uint32_t>((b - b0) / 2);
        w[k / 2] |= static_cast<uint32_t>(h[b / 2]) << (16 * (k % 2));
    }
    return make_uint2(w[0], w[1]);
}
__device__ __forceinline__ void store_pair(void *buf, uint64_t j, uint64_t nbytes, uint2 v) {
    const uint64_t b0 = j * 8;
    if (b0 + 8 <= nbytes) {
        *reinterpret_cast<uint2 *>(static_cast<char *>(buf) + b0) = v;
        return;
    }
    const uint32_t w[2] = {v.x, v.y};
    uint16_t *h = static_cast<uint16_t *>(buf);
    for (uint64_t b = b0; b < nbytes; b += 2) {
        const uint32_t k = static_cast<uint32_t>((b - b0) / 2);
        h[b / 2] = static_cast<uint16_t>(w[k / 2] >> (16 * (k % 2)));
    }
}

// Fold one 32-bit word position across ranks: one fp32 element or two bf16 elements.
template <typename TG, int WORLD> struct WordMean;
template <int WORLD> struct WordMean<float, WORLD> {
    __device__ __forceinline__ static uint32_t run(const uint32_t (&x)[WORLD]) {
        float c[WORLD];
#pragma unroll
        for (int q = 0; q < WORLD; ++q) c[q] = __uint_as_float(x[q]);
        return __float_as_uint(average<WORLD>(c));
    }
};
template <int WORLD> struct WordMean<__nv_bfloat16, WORLD> {
    __device__ __forceinline__ static uint32_t run(const uint32_t (&x)[WORLD]) {
        float lo[WORLD], hi[WORLD];
#pragma unroll
        for (int q = 0; q < WORLD; ++q) {
            lo[q] = Elem<__nv_bfloat16>::lo(x[q]);
            hi[q] = Elem<__nv_bfloat16>::hi(x[q]);
        }
        return Elem<__nv_bfloat16>::pack(average<WORLD>(lo), average<WORLD>(hi));
    }
};

template <typename TG, int WORLD>
__global__ void __launch_bounds__(512)
gdraa_ll_kernel(const __grid_constant__ KParams p) {
    const int vr = blockIdx.y;
    const int rank = p.rank0 + vr;
    Pad *mine = p.pad[vr][rank];
    __shared__ int s_last;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t epoch = *reinterpret_cast<volatile uint64_t *>(&mine->epoch) + 1;
    const uint32_t flag = static_cast<uint32_t>(epoch);
    const uint64_t par = epoch & 1u;
    const uint64_t nbytes = p.n * sizeof(TG);
    const uint64_t npairs = (nbytes + 7) / 8;
    void *const buf = p.dst[vr][rank];
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    bool ok = true;
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < npairs;
         j += stride) {
        const uint2 mine_pair = load_pair(buf, j, nbytes);
        const uint4 entry = make_uint4(mine_pair.x, flag, mine_pair.y, flag);
#pragma unroll
        for (int k = 1; k < WORLD; ++k) {   // push to every peer's slot [par][rank]
            const int q = (rank + k) % WORLD;
            st_ll(p.ll[vr][q] + (par * WORLD + rank) * p.ll_pairs + j, entry);
        }
        uint32_t w0[WORLD], w1[WORLD];
#pragma unroll
        for (int q = 0; q < WORLD; ++q) {
            if (q == rank) {
                w0[q] = mine_pair.x;
                w1[q] = mine_pair.y;
                continue;
            }
            const uint4 *src = p.ll[vr][rank] + (par * WORLD + q) * p.ll_pairs + j;
            const uint4 r = ll_wait(src, flag, p.timeout_ns, p.abort, p.ll_sleep_ns, ok);
            if (!ok) {
                report_timeout(p.err, 1, q, vr);
                break;
            }
            w0[q] = r.x;
            w1[q] = r.z;
        }
        if (!ok) break;
        store_pair(buf, j, nbytes,
                   make_uint2(WordMean<TG, WORLD>::run(w0), WordMean<TG, WORLD>::run(w1)));
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&mine->arrive, 1u);
        s_last = (prev == gridDim.x - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        mine->arrive = 0;
        mine->calls += 1;
        mine->ll_calls += 1;
        mine->epoch = epoch;
        if (p.done[vr] != nullptr) *p.done[vr] = epoch;
    }
}

// ---------------------------------------------------------------------------------
// Small-message fused SGD step (the latency path of gdraa_sgd_step / _mp).  The
// momentum is owner-sharded (AMB-19), so the one-shot scheme above cannot serve it; this
// kernel keeps the two-shot structure of Algorithm 1 but lets the data carry the
// synchronisations, as the paper's RDMA writes into the receive buffer RB do:
//   A  "Reduce": rank r PUSHES its block D(r, q) into owner q's receive slot [par][r]
//      as LL entries {word, flag, word, flag} (Fig. 3a);
//   B  "Aggregation" + update: the owner polls the N-1 entries of each position (its
//      own block comes from local HBM), folds them in ascending rank, divides once, and
//      applies the momentum step; it stores v', w' locally and pushes w'
//      (bf16 RNE(w') for _mp) into every peer's slot [par][r] behind the RS part
//      (Fig. 3b);
//   C  every rank polls the broadcast entries of each peer's block and writes them into
//      its own w (or bf16 model copy).
// Arrival of an entry is the 2nd synchronisation for that position; the arrival of the
// last broadcast entry is the 1st.  No rank ever reads or writes another rank's g or w,
// so neither barrier of the two-shot kernel is needed.  Slot reuse: rank 0 owns a
// non-empty block whenever n >= 1, so finishing call e-1 means having received rank 0's
// broadcast, which rank 0 sent after receiving every rank's call e-1 block, which every
// rank sent after finishing call e-2 -- so parity (e & 1) is free again at call e.
// Slot layout per sender: pairs [0, rs_cap) = the sender's gradient block, pairs
// [rs_cap, rs_cap + ag_cap) = the sender's updated block (caps from the padded shard).
// Work unit of phase B: 4 consecutive elements = 16 (fp32) / 8 (bf16) gradient bytes.
// ---------------------------------------------------------------------------------
template <typename TG, int WORLD, int MODE>
__global__ void __launch_bounds__(512, 2)
gdraa_ll_sgd_kernel(const __grid_constant__ KParams p) {
    using EL = Elem<TG>;
    using Raw = typename EL::Raw;
    constexpr uint64_t SG = sizeof(TG);
    constexpr uint64_t SW = MODE == kSgdMp ? 2 : 4;          // broadcast bytes / element
    constexpr int RS_PAIRS = static_cast<int>(SG * E / 8);    // 2 (fp32) or 1 (bf16)
    constexpr int AG_PAIRS = static_cast<int>(SW * E / 8);    // 2 (fp32 w') or 1 (bf16)
    const int vr = blockIdx.y;
    const int rank = p.rank0 + vr;
    Pad *mine = p.pad[vr][rank];
    __shared__ int s_last;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t epoch = *reinterpret_cast<volatile uint64_t *>(&mine->epoch) + 1;
    const uint32_t flag = static_cast<uint32_t>(epoch);
    const uint64_t par = epoch & 1u;
    const uint64_t rs_cap = (p.blk * SG + 7) / 8;   // the runtime checks rs + ag caps fit
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    auto shard = [&](int q, uint64_t &o, uint64_t &l) {
        o = min(static_cast<uint64_t>(q) * p.blk, p.n);
        l = min(p.blk, p.n - o);
    };
    const TG *const gl = static_cast<const TG *>(p.src[vr][rank]);
    // our receive slot from sender q, and sender rank's slot in peer q's area
    auto rx = [&](int q) { return p.ll[vr][rank] + (par * WORLD + q) * p.ll_pairs; };
    auto tx = [&](int q) { return p.ll[vr][q] + (par * WORLD + rank) * p.ll_pairs; };
    // poll one entry until it carries this call's flag (bounded; abandons on abort)
    bool ok = true;
    auto poll = [&](const uint4 *src, int q, int phase) -> uint2 {
        const uint4 r = ll_wait(src, flag, p.timeout_ns, p.abort, p.ll_sleep_ns, ok);
        if (!ok) report_timeout(p.err, phase, q, vr);
        return make_uint2(r.x, r.z);
    };

    // A: push block D(rank, q) to every owner q != rank.
#pragma unroll 1
    for (int k = 1; k < WORLD; ++k) {
        const int q = (rank + k) % WORLD;
        uint64_t oq, lq;
        shard(q, oq, lq);
        const uint64_t nb = lq * SG, np = (nb + 7) / 8;
        const void *base = gl + oq;
        uint4 *dstq = tx(q);
        for (uint64_t j = tid; j < np; j += stride) {
            const uint2 w = load_pair(base, j, nb);
            st_ll(dstq + j, make_uint4(w.x, flag, w.y, flag));
        }
    }

    // B: fold + update our block, push w' to every peer.
    uint64_t off, len;
    shard(rank, off, len);
    float *const vloc = p.v[vr];
    float *const wloc = MODE == kSgdMp ? p.wm[vr] : static_cast<float *>(p.dst[vr][rank]);
    const float lr = p.lr, mom = p.mom, wd = p.wd;
    const uint64_t nunits = (len + E - 1) / E;
    for (uint64_t u = tid; ok && u < nunits; u += stride) {
        const uint64_t i0 = u * E;                       // first element (shard-relative)
        const int cnt = static_cast<int>(len - i0 < E ? len - i0 : E);
        const int rs_n = static_cast<int>((cnt * SG + 7) / 8);   // RS pairs of this unit
        float x[WORLD][E];
#pragma unroll
        for (int q = 0; q < WORLD; ++q) {
            if (q == rank) {
                for (int e = 0; e < E; ++e) x[q][e] = e < cnt ? EL::load1(gl, off + i0 + e) : 0.f;
                continue;
            }
            uint32_t wd4[4] = {0u, 0u, 0u, 0u};
            const uint4 *src = rx(q) + u * RS_PAIRS;
            for (int h = 0; h < rs_n; ++h) {
                const uint2 pr = poll(src + h, q, 1);
                wd4[2 * h] = pr.x;
                wd4[2 * h + 1] = pr.y;
            }
            Raw raw;
            if constexpr (std::is_same<TG, float>::value)
                raw = make_uint4(wd4[0], wd4[1], wd4[2], wd4[3]);
            else
                raw = make_uint2(wd4[0], wd4[1]);
            EL::widen(raw, x[q]);
        }
        if (!ok) break;
        float wv[E], vv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (e < cnt) {
                float col[WORLD];
#pragma unroll
                for (int q = 0; q < WORLD; ++q) col[q] = x[q][e];
                const float m = average<WORLD>(col);
                wv[e] = wloc[off + i0 + e];
                vv[e] = vloc[off + i0 + e];
                sgd(m, lr, mom, wd, wv[e], vv[e]);
                vloc[off + i0 + e] = vv[e];
                wloc[off + i0 + e] = wv[e];
                if (MODE == kSgdMp)
                    Elem<__nv_bfloat16>::store1(p.dst[vr][rank], off + i0 + e, wv[e]);
            } else {
                wv[e] = 0.f;
            }
        }
        // broadcast entries of this unit (fp32 w': 2 pairs, bf16 copy: 1 pair)
        uint32_t ow[4];
        if (MODE == kSgdMp) {
            const uint2 b = Elem<__nv_bfloat16>::narrow(wv);
            ow[0] = b.x; ow[1] = b.y; ow[2] = 0u; ow[3] = 0u;
        } else {
            ow[0] = __float_as_uint(wv[0]); ow[1] = __float_as_uint(wv[1]);
            ow[2] = __float_as_uint(wv[2]); ow[3] = __float_as_uint(wv[3]);
        }
        const int ag_n = static_cast<int>((cnt * SW + 7) / 8);
#pragma unroll
        for (int k = 1; k < WORLD; ++k) {
            uint4 *dstq = tx((rank + k) % WORLD) + rs_cap + u * AG_PAIRS;
            for (int h = 0; h < ag_n; ++h)
                st_ll(dstq + h, make_uint4(ow[2 * h], flag, ow[2 * h + 1], flag));
        }
    }

    // C: receive every peer's updated block into our w (or bf16 model copy).
    void *const wdst = p.dst[vr][rank];
#pragma unroll 1
    for (int k = 1; ok && k < WORLD; ++k) {
        const int q = (rank + k) % WORLD;
        uint64_t oq, lq;
        shard(q, oq, lq);
        const uint64_t nb = lq * SW, np = (nb + 7) / 8;
        void *base = static_cast<char *>(wdst) + oq * SW;
        const uint4 *src = rx(q) + rs_cap;
        for (uint64_t j = tid; j < np; j += stride) {
            const uint2 w = poll(src + j, q, 2);
            if (!ok) break;
            store_pair(base, j, nb, w);
        }
    }

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&mine->arrive, 1u);
        s_last = (prev == gridDim.x - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        mine->arrive = 0;
        mine->calls += 1;
        mine->ll_calls += 1;
        mine->epoch = epoch;
        if (p.done[vr] != nullptr) *p.done[vr] = epoch;
    }
}

// ---------------------------------------------------------------------------------
// TMA-staged variant of the two-shot kernel (same a2..a7 steps, same arithmetic, same
// barriers).  One producer thread per CTA streams each chunk of the owner shard -- the
// N ranks' gradient blocks (NVLink for peers) plus the local w and v -- into a
// STAGES-deep shared-memory ring with 1-D bulk copies (cp.async.bulk, completion on an
// mbarrier); 8 consumer warps fold, update and push from shared memory.  Bytes in
// flight per SM no longer depend on registers, so a few dozen SMs drive NVLink at full
// rate (profiles/r19_nvlink_probe_n2_ctas.jsonl: bulk pulls reach 615 GB/s from 16 SMs)
// and the rest stay free for a concurrent backward pass (NEXT-3).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Stage = one chunk of CH elements of every source (+ w, v): about STAGE_KB per stage.
// 16 consumer warps: same rate as 8 on the full grid, and 607 GB/s (full rate) from only
// 64 SMs at N=2 vs 595 for 8 warps (profiles/r21_ctas_n2.jsonl).
// End game: the last ~2 waves of chunks are CH / TAILDIV elements, and while they are
// handed out a producer keeps at most TDEPTH of them in flight (so no CTA sits on a
// deep private queue while others have run dry).
// ROT: the producer issues the N gradient copies of a chunk starting at its own rank
// (rank, rank+1, ...) instead of rank 0 (the fold order is unaffected).
template <typename TG, int WORLD, int MODE, int CW_ = 16, int ST_ = 4, int TAILDIV_ = 4,
          int TDEPTH_ = ST_, int ROT_ = 0, int STAGE_KB = 40>
struct TmaCfg {
    static constexpr int TAILDIV = TAILDIV_;
    static constexpr bool ROT = ROT_ != 0;
    static constexpr int TDEPTH = TDEPTH_ < ST_ ? TDEPTH_ : ST_;
    static constexpr int SG = sizeof(TG);
    static constexpr bool UPD = MODE != kMean;
    static constexpr int PER_EL = WORLD * SG + (UPD ? 8 : 0);      // smem bytes / element
    static constexpr int BUDGET = STAGE_KB * 1024;
    // 4096-element chunks only for stage budgets above the library's 40 KB (tune sweeps)
    static constexpr int CH = (STAGE_KB > 40 && BUDGET / PER_EL >= 4096) ? 4096
                              : (BUDGET / PER_EL >= 2048 ? 2048 : (BUDGET / PER_EL >= 1024 ? 1024 : 512));
    static constexpr int STAGES = ST_;
    static constexpr int CW = CW_;                                 // consumer warps
    static constexpr int THREADS = 32 * (CW + 1);
    static constexpr int STAGE_BYTES = CH * PER_EL;
    static constexpr int SMEM = STAGES * STAGE_BYTES;
};

// a4 fold (+ a5 update) of one chunk that the TMA producer staged in shared memory, and
// the a6 push; shared by gdraa_tma_kernel and gdraa_tma_set_kernel.  stage: the chunk's
// stage (the N ranks' gradient blocks of CH elements, then w and v); g0c: index of the
// chunk's first element relative to the base pointers p.dst[vr][*], vloc and wloc.
template <typename C, typename TG, int WORLD, int MODE, int VE>
__device__ __forceinline__ void tma_consume(const KParams &p, int vr, int rank,
                                            const unsigned char *stage, uint64_t g0c,
                                            uint32_t n_el, int ct, float *vloc, float *wloc,
                                            float lr, float mom, float wd, void *mcd,
                                            bool mc_self) {
    using EL = Elem<TG>;
    using Raw = typename EL::Raw;
    constexpr bool kUpdate = C::UPD;
    constexpr int H = VE / E;
    using BfOut = typename std::conditional<H == 2, uint4, uint2>::type;   // VE bf16 values
    auto src = [&](int q) { return reinterpret_cast<const TG *>(stage) + q * C::CH; };
    const float *sw = reinterpret_cast<const float *>(stage + WORLD * C::SG * C::CH);
    const float *sv = sw + C::CH;
    for (uint32_t k = ct * VE; k < n_el; k += C::CW * 32 * VE) {
        float m[H][E];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            float x[WORLD][E];
#pragma unroll
            for (int q = 0; q < WORLD; ++q)
                EL::widen(*reinterpret_cast<const Raw *>(src(q) + k + h * E), x[q]);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                float col[WORLD];
#pragma unroll
                for (int q = 0; q < WORLD; ++q) col[q] = x[q][e];
                m[h][e] = average<WORLD>(col);
            }
        }
        const uint64_t g0 = g0c + k;
        if (kUpdate) {
            float4 w[H];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                w[h] = *reinterpret_cast<const float4 *>(sw + k + h * E);
                float4 v = *reinterpret_cast<const float4 *>(sv + k + h * E);
                sgd(m[h][0], lr, mom, wd, w[h].x, v.x);
                sgd(m[h][1], lr, mom, wd, w[h].y, v.y);
                sgd(m[h][2], lr, mom, wd, w[h].z, v.z);
                sgd(m[h][3], lr, mom, wd, w[h].w, v.w);
                st_vec(reinterpret_cast<uint4 *>(vloc + g0 + h * E), as_u4(v.x, v.y, v.z, v.w));
            }
            if (MODE == kSgd) {
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const uint4 o = as_u4(w[h].x, w[h].y, w[h].z, w[h].w);
                    const uint64_t gh = g0 + h * E;
                    if (mcd != nullptr) {
                        mc_st(reinterpret_cast<uint4 *>(static_cast<float *>(mcd) + gh), o);
                        if (mc_self)
                            st_vec(reinterpret_cast<uint4 *>(static_cast<float *>(p.dst[vr][rank]) + gh), o);
                    } else {
#pragma unroll
                        for (int j = 1; j <= WORLD; ++j) {
                            const int q = (rank + j) % WORLD;
                            st_vec(reinterpret_cast<uint4 *>(static_cast<float *>(p.dst[vr][q]) + gh), o);
                        }
                    }
                }
            } else {   // kSgdMp: fp32 master shard stays local, bf16 copy to every rank
                BfOut o;
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    st_vec(reinterpret_cast<uint4 *>(wloc + g0 + h * E),
                           as_u4(w[h].x, w[h].y, w[h].z, w[h].w));
                    const float wf[E] = {w[h].x, w[h].y, w[h].z, w[h].w};
                    set_half(o, h, Elem<__nv_bfloat16>::narrow(wf));
                }
                if (mcd != nullptr) {
                    mc_st_bf16(reinterpret_cast<BfOut *>(static_cast<__nv_bfloat16 *>(mcd) + g0), o);
                    if (mc_self)
                        st_vec(reinterpret_cast<BfOut *>(static_cast<__nv_bfloat16 *>(p.dst[vr][rank]) + g0), o);
                } else {
#pragma unroll
                    for (int j = 1; j <= WORLD; ++j) {
                        const int q = (rank + j) % WORLD;
                        st_vec(reinterpret_cast<BfOut *>(static_cast<__nv_bfloat16 *>(p.dst[vr][q]) + g0), o);
                    }
                }
            }
        } else if constexpr (std::is_same<TG, float>::value) {
            const Raw o = EL::narrow(m[0]);
#pragma unroll
            for (int j = 1; j <= WORLD; ++j) {
                const int q = (rank + j) % WORLD;
                st_vec(reinterpret_cast<Raw *>(static_cast<TG *>(p.dst[vr][q]) + g0), o);
            }
        } else {   // bf16 mean: VE elements -> one store per destination
            BfOut o;
#pragma unroll
            for (int h = 0; h < H; ++h) set_half(o, h, EL::narrow(m[h]));
#pragma unroll
            for (int j = 1; j <= WORLD; ++j) {
                const int q = (rank + j) % WORLD;
                st_vec(reinterpret_cast<BfOut *>(static_cast<TG *>(p.dst[vr][q]) + g0), o);
            }
        }
    }
}

// Scalar a3-a6 for elements e = lo, lo + stride, ... < hi (a shard's ragged tail of
// len % 8 elements, which no 16-byte bulk copy covers), reading the ranks' gradients
// directly; indices relative to the base pointers.
template <typename TG, int WORLD, int MODE>
__device__ __forceinline__ void tail_scalar(const KParams &p, int vr, int rank, uint64_t lo,
                                            uint64_t hi, int stride, float *vloc, float *wloc,
                                            float lr, float mom, float wd) {
    using EL = Elem<TG>;
    for (uint64_t e = lo; e < hi; e += stride) {
        float col[WORLD];
#pragma unroll
        for (int q = 0; q < WORLD; ++q) col[q] = EL::load1(p.src[vr][q], e);
        const float m = average<WORLD>(col);
        if (MODE != kMean) {
            float w = wloc[e], v = vloc[e];
            sgd(m, lr, mom, wd, w, v);
            vloc[e] = v;
            if (MODE == kSgd) {
                for (int j = 1; j <= WORLD; ++j)
                    static_cast<float *>(p.dst[vr][(rank + j) % WORLD])[e] = w;
            } else {
                wloc[e] = w;
                for (int j = 1; j <= WORLD; ++j)
                    Elem<__nv_bfloat16>::store1(p.dst[vr][(rank + j) % WORLD], e, w);
            }
        } else {
            for (int j = 1; j <= WORLD; ++j)
                EL::store1(p.dst[vr][(rank + j) % WORLD], e, m);
        }
    }
}

// VE_: elements per consumer thread per step (0 = 8 when the broadcast is bf16 -- the bf16
// mean and the mixed-precision model copy -- so that every destination gets one 16-byte
// store per thread and step, else 4).
template <typename TG, int WORLD, int MODE, int CW_ = 16, int ST_ = 4, int TAILDIV_ = 4,
          int TDEPTH_ = ST_, int ROT_ = 0, int VE_ = 0, int SKB_ = 40>
__global__ void __launch_bounds__(TmaCfg<TG, WORLD, MODE, CW_, ST_, TAILDIV_, TDEPTH_, ROT_, SKB_>::THREADS, 1)
gdraa_tma_kernel(const __grid_constant__ KParams p) {
    using C = TmaCfg<TG, WORLD, MODE, CW_, ST_, TAILDIV_, TDEPTH_, ROT_, SKB_>;
    using EL = Elem<TG>;
    using Raw = typename EL::Raw;
    constexpr bool kUpdate = C::UPD;
    constexpr bool kBfOut = MODE == kSgdMp || (MODE == kMean && !std::is_same<TG, float>::value);
    constexpr int VE = VE_ != 0 ? VE_ : (kBfOut ? 8 : 4);
    constexpr int H = VE / E;                 // 4-element vectors per thread and step
    static_assert(H == 1 || (H == 2 && kBfOut), "VE = 8 only for bf16 broadcasts");
    using BfOut = typename std::conditional<H == 2, uint4, uint2>::type;   // VE bf16 values
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[C::STAGES], empty[C::STAGES];
    __shared__ uint32_t s_chunk[C::STAGES];
    __shared__ int s_abort, s_last;

    const int vr = blockIdx.y;
    const int rank = p.rank0 + vr;
    Pad *mine = p.pad[vr][rank];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t epoch = *reinterpret_cast<volatile uint64_t *>(&mine->epoch) + 1;
    if (threadIdx.x == 0) {
        s_abort = 0;
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) GDRAA_STAMP_START();
#ifdef GDRAA_EXPERIMENTAL
    // multicast barrier variant: counters reach (mc_calls + 1) * N once every rank arrived
    const bool mcb = WORLD > 1 && p.mc_bar[vr] != nullptr;
    const uint64_t mc_target =
        mcb ? (*reinterpret_cast<volatile uint64_t *>(&mine->mc_calls) + 1) * WORLD : 0;
#else
    constexpr bool mcb = false;
#endif
    // a2: "2nd synchronization"
#ifdef GDRAA_EXPERIMENTAL
    if (WORLD > 1 && mcb) {
        if (blockIdx.x == 0 && threadIdx.x == 0) mc_red_add_release(p.mc_bar[vr], 1);
        __syncthreads();
        if (threadIdx.x == 0 && !wait_geq(p.bar_local[vr], mc_target, p.timeout_ns, p.abort)) {
            report_timeout(p.err, 1, rank, vr);
            s_abort = 1;
        }
    } else
#endif
    if (WORLD > 1) {
        if (blockIdx.x == 0 && threadIdx.x < WORLD && threadIdx.x != rank)
            st_release_sys(&p.pad[vr][threadIdx.x]->entry[rank], epoch);
        __syncthreads();
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            if (!wait_geq(&mine->entry[threadIdx.x], epoch, p.timeout_ns, p.abort)) {
                report_timeout(p.err, 1, threadIdx.x, vr);
                s_abort = 1;
            }
        }
    }
    __syncthreads();
    if (s_abort) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) GDRAA_STAMP(1);

    const uint64_t off = min(static_cast<uint64_t>(rank) * p.blk, p.n);
    const uint64_t len = min(p.blk, p.n - off);
    const uint64_t lenv = len & ~7ull;                  // bulk copies: 16-byte multiples
    // Chunks of CH elements, the last ~2 waves of CH/TAILDIV so the CTAs finish together
    // (the end-game of the LSU kernel); chunk c -> (e0, n_el) is a pure function.
    constexpr uint64_t CHS = C::CH / C::TAILDIV;
    const uint64_t tailv = 2ull * gridDim.x * CHS;
    const uint64_t nbig = lenv > tailv ? (lenv - tailv) / C::CH : 0;
    const uint64_t small0 = nbig * C::CH;
    const uint64_t nchunks = nbig + (lenv - small0 + CHS - 1) / CHS;
    auto chunk = [&](uint32_t c, uint64_t &e0, uint32_t &n_el) {
        if (c < nbig) {
            e0 = static_cast<uint64_t>(c) * C::CH;
            n_el = C::CH;
        } else {
            e0 = small0 + (c - nbig) * CHS;
            n_el = static_cast<uint32_t>(lenv - e0 < CHS ? lenv - e0 : CHS);
        }
    };
    const float lr = p.lr, mom = p.mom, wd = p.wd;
    float *const vloc = p.v[vr];
    float *const wloc = MODE == kSgdMp ? p.wm[vr] : static_cast<float *>(p.dst[vr][rank]);

    auto stage_src = [&](int s, int q) {
        return reinterpret_cast<TG *>(smem + s * C::STAGE_BYTES) + q * C::CH;
    };
    auto stage_w = [&](int s) {
        return reinterpret_cast<float *>(smem + s * C::STAGE_BYTES + WORLD * C::SG * C::CH);
    };
    auto stage_v = [&](int s) { return stage_w(s) + C::CH; };

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint64_t my_elems = 0;   // thread 0: elements of the chunks this CTA claimed (dist exit)
    if (warp == 0) {
        // producer: a3 loads (and the local w, v) of one chunk per stage
        if (lane == 0) {
            // The entry barrier's acquire (generic proxy) must also order the bulk copies
            // (async proxy) that read the peers' gradients after it.
            asm volatile("fence.proxy.async.global;" ::: "memory");
            bool tail = false;
            for (uint32_t it = 0;; ++it) {
                const int s = it % C::STAGES;
                if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
                if (C::TDEPTH < C::STAGES && tail && it >= C::TDEPTH) {
                    // end game: wait until stage it - TDEPTH has been consumed
                    const uint32_t j = it - C::TDEPTH;
                    mbar_wait(&empty[j % C::STAGES], (j / C::STAGES) & 1);
                }
                const uint32_t c = atomicAdd(&mine->next, 1u);
                tail = c >= nbig;
                if (c >= nchunks) {
                    s_chunk[s] = 0xFFFFFFFFu;
                    mbar_arrive(&full[s]);
                    break;
                }
                s_chunk[s] = c;
                uint64_t e0;
                uint32_t n_el;
                chunk(c, e0, n_el);
                my_elems += n_el;
                mbar_arrive_tx(&full[s], n_el * C::PER_EL);
#pragma unroll
                for (int k = 0; k < WORLD; ++k) {
                    const int q = C::ROT ? (rank + k) % WORLD : k;
                    bulk_g2s(stage_src(s, q), static_cast<const TG *>(p.src[vr][q]) + off + e0,
                             n_el * C::SG, &full[s]);
                }
                if (kUpdate) {
                    bulk_g2s(stage_w(s), wloc + off + e0, n_el * 4, &full[s]);
                    bulk_g2s(stage_v(s), vloc + off + e0, n_el * 4, &full[s]);
                }
            }
        }
    } else {
        // consumers: a4 fold (+ a5 update) from shared memory, a6 push
        const int ct = threadIdx.x - 32;
#ifdef GDRAA_EXPERIMENTAL
        void *const mcd = WORLD > 1 ? p.mc_dst[vr] : nullptr;   // multicast broadcast (A/B)
#else
        void *const mcd = nullptr;
#endif
        const bool mc_self = (p.flags & kFlagMcPeersOnly) != 0;
        for (uint32_t it = 0;; ++it) {
            const int s = it % C::STAGES;
            mbar_wait(&full[s], (it / C::STAGES) & 1);
            const uint32_t c = s_chunk[s];
            if (c == 0xFFFFFFFFu) break;
            uint64_t e0;
            uint32_t n_el;
            chunk(c, e0, n_el);
            tma_consume<C, TG, WORLD, MODE, VE>(p, vr, rank, smem + s * C::STAGE_BYTES, off + e0,
                                                n_el, ct, vloc, wloc, lr, mom, wd, mcd, mc_self);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        // ragged tail (len % 8 elements) by the last CTA's consumers, scalar
        if (blockIdx.x == gridDim.x - 1)
            tail_scalar<TG, WORLD, MODE>(p, vr, rank, off + lenv + ct, off + len, C::CW * 32,
                                         vloc, wloc, lr, mom, wd);
    }

    // a7: "1st synchronization" (as in gdraa_kernel)
    if (blockIdx.x == 0 && threadIdx.x == 0) GDRAA_STAMP(2);
    GDRAA_STAMP_DONE();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef GDRAA_EXPERIMENTAL
    const bool dist = WORLD > 1 && !mcb && (p.flags & kFlagDistExit) != 0;
#else
    constexpr bool dist = false;
#endif
    const bool defer = (p.flags & kFlagDeferExit) != 0 && !dist && !mcb;   // bucket set
    const bool cta_fence = (p.flags & kFlagCtaFence) != 0 || dist;
    if (WORLD > 1 && !cta_fence && !defer) fence_acq_rel_sys();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (WORLD > 1 && cta_fence && !defer) fence_acq_rel_sys();
#ifdef GDRAA_EXPERIMENTAL
        if (dist) {
            if (blockIdx.x == gridDim.x - 1) my_elems += len - lenv;   // the ragged tail
#pragma unroll 1
            for (int j = 1; j < WORLD; ++j) {
                const int q = (rank + j) % WORLD;
                red_add_release_sys(&p.pad[vr][q]->recv_done[rank], my_elems);
            }
        }
#endif
        const unsigned prev = atomicAdd(&mine->arrive, 1u);
        s_last = (prev == gridDim.x - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x == 0) GDRAA_STAMP(3);
#ifdef GDRAA_EXPERIMENTAL
    if (dist) {
        // every CTA of every peer q has finished (its pulls of our g done, its pushes into
        // our w performed) once recv_done[q] covers q's whole shard
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            const int q = threadIdx.x;
            const uint64_t oq = min(static_cast<uint64_t>(q) * p.blk, p.n);
            const uint64_t target = mine->recv_expect[q] + min(p.blk, p.n - oq);
            if (!wait_geq(&mine->recv_done[q], target, p.timeout_ns, p.abort)) {
                report_timeout(p.err, 2, q, vr);
                s_abort = 1;
            } else {
                mine->recv_expect[q] = target;
            }
        }
        __syncthreads();
        if (s_abort) return;
    } else if (WORLD > 1 && mcb) {
        if (threadIdx.x == 0) {
            mc_red_add_release(p.mc_bar[vr] + 1, 1);
            if (!wait_geq(p.bar_local[vr] + 1, mc_target, p.timeout_ns, p.abort)) {
                report_timeout(p.err, 2, rank, vr);
                s_abort = 1;
            }
        }
        __syncthreads();
        if (s_abort) return;
    } else
#endif
    if (WORLD > 1 && !defer) {
        if (threadIdx.x < WORLD && threadIdx.x != rank)
            st_release_sys(&p.pad[vr][threadIdx.x]->exit[rank], epoch);
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            if (!wait_geq(&mine->exit[threadIdx.x], epoch, p.timeout_ns, p.abort)) {
                report_timeout(p.err, 2, threadIdx.x, vr);
                s_abort = 1;
            }
        }
        __syncthreads();
        if (s_abort) return;
    }
    if (threadIdx.x == 0) {
        GDRAA_STAMP(4);
        mine->arrive = 0;
        mine->next = 0;
        mine->calls += 1;
        if (WORLD > 1) mine->sync_waits += defer ? 1 : 2;
        if (mcb) mine->mc_calls += 1;
        mine->epoch = epoch;
        if (p.done[vr] != nullptr) *p.done[vr] = epoch;
    }
}

// ---------------------------------------------------------------------------------
// Streamed bucket set (gdraa_bucket_set_begin_streamed): ONE
// persistent grid serves every bucket of an iteration, so a bucket costs neither a launch
// nor a grid drain nor an exit barrier, and a CTA that runs out of work in bucket k moves
// straight on to bucket k+1.  Per bucket k (descriptors written by stream memory
// operations on the caller's stream when the bucket's gradient is final, see SetDesc):
//   a2  the producer of every CTA waits for ready[k]; CTA 0 then stores epoch e_k into
//       every peer's pad and every producer waits for every peer's e_k (the same flags as
//       the per-call kernel, one epoch per bucket);
//   a3-a6 chunks of the bucket's owner shard are claimed from next[k] and staged, folded,
//       updated and pushed exactly as in gdraa_tma_kernel (tma_consume; the shard's
//       ragged tail is one extra "chunk" done by scalar loads, tail_scalar);
// and once the close marker arrives: a7 once for the whole set (per-CTA fence, the last
// CTA exchanges exit flags at the last bucket's epoch).  Same arithmetic, same bits.
// ---------------------------------------------------------------------------------
template <typename TG, int WORLD, int MODE>
__global__ void __launch_bounds__(TmaCfg<TG, WORLD, MODE>::THREADS, 1)
gdraa_tma_set_kernel(const __grid_constant__ KParams p) {
    using C = TmaCfg<TG, WORLD, MODE>;
    constexpr bool kUpdate = C::UPD;
    constexpr bool kBfOut = MODE == kSgdMp || (MODE == kMean && !std::is_same<TG, float>::value);
    constexpr int VE = kBfOut ? 8 : 4;
    constexpr uint32_t kDone = 0xFFFFFFFFu;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[C::STAGES], empty[C::STAGES];
    __shared__ uint32_t s_bk[C::STAGES], s_chunk[C::STAGES];
    __shared__ uint64_t s_first[C::STAGES], s_count[C::STAGES];
    __shared__ int s_abort, s_last;
    __shared__ uint32_t s_nb;

    const int vr = blockIdx.y;
    const int rank = p.rank0 + vr;
    Pad *mine = p.pad[vr][rank];
    const uint64_t epoch0 = *reinterpret_cast<volatile uint64_t *>(&mine->epoch);
    if (threadIdx.x == 0) {
        s_abort = 0;
        s_nb = 0;
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    float *const vloc = p.v[vr];
    float *const wloc = MODE == kSgdMp ? p.wm[vr] : static_cast<float *>(p.dst[vr][rank]);
    constexpr uint64_t CHS = C::CH / C::TAILDIV;
    // the owner shard of a bucket of `count` elements and its chunking (as gdraa_tma_kernel)
    struct Geo {
        uint64_t off, len, lenv, nbig, small0, nchunks;
    };
    auto geo = [&](uint64_t count) {
        Geo g;
        const uint64_t c = (count + WORLD - 1) / WORLD;
        const uint64_t blk = (c + 63) / 64 * 64;
        g.off = min(static_cast<uint64_t>(rank) * blk, count);
        g.len = min(blk, count - g.off);
        g.lenv = g.len & ~7ull;
        const uint64_t tailv = 2ull * gridDim.x * CHS;
        g.nbig = g.lenv > tailv ? (g.lenv - tailv) / C::CH : 0;
        g.small0 = g.nbig * C::CH;
        g.nchunks = g.nbig + (g.lenv - g.small0 + CHS - 1) / CHS;
        return g;
    };
    auto chunk = [&](const Geo &g, uint32_t c, uint64_t &e0, uint32_t &n_el) {
        if (c < g.nbig) {
            e0 = static_cast<uint64_t>(c) * C::CH;
            n_el = C::CH;
        } else {
            e0 = g.small0 + (c - g.nbig) * CHS;
            n_el = static_cast<uint32_t>(g.lenv - e0 < CHS ? g.lenv - e0 : CHS);
        }
    };
    auto stage_src = [&](int s, int q) {
        return reinterpret_cast<TG *>(smem + s * C::STAGE_BYTES) + q * C::CH;
    };
    auto stage_w = [&](int s) {
        return reinterpret_cast<float *>(smem + s * C::STAGE_BYTES + WORLD * C::SG * C::CH);
    };

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        if (lane == 0) {
            // producer
            const SetDesc *sd = p.sdesc;
            uint32_t *next = p.snext[vr];
            const uint64_t want_close = set_close(p.sgen);
            uint32_t it = 0;
            bool have_stage = false;
            for (uint32_t b = 0; b < kSetMax; ++b) {
                // bucket b described and its gradient final on this rank (or the set closed)
                const uint64_t want = set_tag(p.sgen, b);
                uint64_t r = ld_relaxed_sys(&sd->ready[b]);
                if (r != want && r != want_close) {
                    const uint64_t t0 = global_timer_ns();
                    uint32_t polls = 0;
                    while ((r = ld_relaxed_sys(&sd->ready[b])) != want && r != want_close) {
                        if (global_timer_ns() - t0 > p.timeout_ns ||
                            (p.abort != nullptr && (++polls & 4095u) == 0 && *p.abort != 0)) {
                            report_timeout(p.err, 1, rank, vr);
                            s_abort = 1;
                            break;
                        }
                    }
                    if (s_abort) break;
                }
                (void)ld_acquire_sys(&sd->ready[b]);
                if (r == want_close) {
                    s_nb = b;
                    break;
                }
                const uint64_t first = *reinterpret_cast<const volatile uint64_t *>(&sd->first[b]);
                const uint64_t count = *reinterpret_cast<const volatile uint64_t *>(&sd->count[b]);
                // a2 for bucket b
                const uint64_t e = epoch0 + 1 + b;
                if (WORLD > 1) {
                    if (blockIdx.x == 0)
                        for (int q = 0; q < WORLD; ++q)
                            if (q != rank) st_release_sys(&p.pad[vr][q]->entry[rank], e);
                    for (int q = 0; q < WORLD && !s_abort; ++q)
                        if (q != rank && !wait_geq(&mine->entry[q], e, p.timeout_ns, p.abort)) {
                            report_timeout(p.err, 1, q, vr);
                            s_abort = 1;
                        }
                    if (s_abort) break;
                }
                asm volatile("fence.proxy.async.global;" ::: "memory");
                const Geo g = geo(count);
                const uint32_t total = static_cast<uint32_t>(g.nchunks + (g.len > g.lenv ? 1 : 0));
                for (;;) {
                    const int s = it % C::STAGES;
                    if (!have_stage) {
                        if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
                        have_stage = true;
                    }
                    const uint32_t c = atomicAdd(&next[b], 1u);
                    if (c >= total) break;               // bucket b done: keep the stage
                    s_bk[s] = b;
                    s_chunk[s] = c;
                    s_first[s] = first;
                    s_count[s] = count;
                    if (c == g.nchunks) {
                        mbar_arrive(&full[s]);            // ragged tail: no bulk copy
                    } else {
                        uint64_t e0;
                        uint32_t n_el;
                        chunk(g, c, e0, n_el);
                        const uint64_t base = first + g.off + e0;
                        mbar_arrive_tx(&full[s], n_el * C::PER_EL);
#pragma unroll
                        for (int q = 0; q < WORLD; ++q)
                            bulk_g2s(stage_src(s, q), static_cast<const TG *>(p.src[vr][q]) + base,
                                     n_el * C::SG, &full[s]);
                        if (kUpdate) {
                            bulk_g2s(stage_w(s), wloc + base, n_el * 4, &full[s]);
                            bulk_g2s(stage_w(s) + C::CH, vloc + base, n_el * 4, &full[s]);
                        }
                    }
                    ++it;
                    have_stage = false;
                }
            }
            // no more work: the consumers' stop sentinel
            const int s = it % C::STAGES;
            if (!have_stage && it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
            s_chunk[s] = kDone;
            mbar_arrive(&full[s]);
        }
    } else {
        const int ct = threadIdx.x - 32;
        for (uint32_t it = 0;; ++it) {
            const int s = it % C::STAGES;
            mbar_wait(&full[s], (it / C::STAGES) & 1);
            const uint32_t c = s_chunk[s];
            if (c == kDone) break;
            const uint64_t first = s_first[s];
            const Geo g = geo(s_count[s]);
            if (c == g.nchunks) {
                tail_scalar<TG, WORLD, MODE>(p, vr, rank, first + g.off + g.lenv + ct,
                                             first + g.off + g.len, C::CW * 32, vloc, wloc,
                                             p.lr, p.mom, p.wd);
            } else {
                uint64_t e0;
                uint32_t n_el;
                chunk(g, c, e0, n_el);
                tma_consume<C, TG, WORLD, MODE, VE>(p, vr, rank, smem + s * C::STAGE_BYTES,
                                                    first + g.off + e0, n_el, ct, vloc, wloc,
                                                    p.lr, p.mom, p.wd, nullptr, false);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }

    // a7 once for the set: our pushes performed, then the last CTA of this rank exchanges
    // exit flags at the last bucket's epoch
    __syncthreads();
    if (threadIdx.x == 0) {
        if (WORLD > 1) fence_acq_rel_sys();
        const unsigned prev = atomicAdd(&mine->arrive, 1u);
        s_last = (prev == gridDim.x - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    // every CTA's producer saw the same close index; take it from this one (or, after an
    // abort, report nothing further: the error block already names the missing rank)
    if (s_abort) return;
    const uint32_t nb = s_nb;
    const uint64_t e_last = epoch0 + nb;
    if (WORLD > 1) {
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            st_release_sys(&p.pad[vr][threadIdx.x]->exit[rank], e_last);
            if (!wait_geq(&mine->exit[threadIdx.x], e_last, p.timeout_ns, p.abort)) {
                report_timeout(p.err, 2, threadIdx.x, vr);
                s_abort = 1;
            }
        }
        __syncthreads();
        if (s_abort) return;
    }
    // reset the chunk counters this set used, for the next set
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) p.snext[vr][b] = 0;
    if (threadIdx.x == 0) {
        mine->arrive = 0;
        mine->calls += nb;
        if (WORLD > 1) mine->sync_waits += nb + 1;
        mine->epoch = e_last;
        if (p.done[vr] != nullptr) *p.done[vr] = e_last;
    }
}

// ---------------------------------------------------------------------------------
// The deferred 1st synchronization of a bucket set (gdraa_bucket_set_end; SURVEY §8(f)
// NEXT-3, "as late as the DL needs").  The set's two-shot calls ran their entry
// barrier and data movement but neither fenced nor exchanged exit flags; this grid,
// stream-ordered after all of them, performs both once: every pushing thread of those
// kernels has finished (kernel boundary), a system-scope fence makes their stores
// performed, and each rank tells every peer and waits for every peer with the epoch of
// the set's last call (exit flags are monotone, so the skipped epochs need no flag of
// their own).  One CTA of 32 threads per (virtual) rank; the epoch is not advanced.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(32) gdraa_exit_kernel(const __grid_constant__ KParams p) {
    const int vr = blockIdx.y;
    const int rank = p.rank0 + vr;
    Pad *mine = p.pad[vr][rank];
    __shared__ int s_abort;
    if (threadIdx.x == 0) s_abort = 0;
    const uint64_t epoch = *reinterpret_cast<volatile uint64_t *>(&mine->epoch);
    __syncthreads();
    const int q = threadIdx.x;
    if (q < p.world && q != rank) {
        fence_acq_rel_sys();
        st_release_sys(&p.pad[vr][q]->exit[rank], epoch);
        if (!wait_geq(&mine->exit[q], epoch, p.timeout_ns, p.abort)) {
            report_timeout(p.err, 2, q, vr);
            s_abort = 1;
        }
    }
    __syncthreads();
    if (s_abort) return;
    if (threadIdx.x == 0) mine->sync_waits += 1;
}

using KernelFnLL = void (*)(KParams);

// Programmatic stream serialization hides the launch gap between back-to-back
// collectives (GDRAA_PDL=0 launches plainly).
cudaError_t launch_pdl(void (*fn)(KParams), dim3 grid, dim3 block, cudaStream_t s,
                       const KParams &p) {
    static const bool pdl = [] {
        const char *e = std::getenv("GDRAA_PDL");
        return e == nullptr || e[0] != '0';
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, p);
}

template <typename TG>
KernelFnLL pick_ll_t(int world) {
    switch (world) {
        case 2: return gdraa_ll_kernel<TG, 2>;
        case 3: return gdraa_ll_kernel<TG, 3>;
        case 4: return gdraa_ll_kernel<TG, 4>;
        case 5: return gdraa_ll_kernel<TG, 5>;
        case 6: return gdraa_ll_kernel<TG, 6>;
        case 7: return gdraa_ll_kernel<TG, 7>;
        case 8: return gdraa_ll_kernel<TG, 8>;
        default: return nullptr;
    }
}

struct TmaLaunch {
    KernelFnLL fn;
    int threads;
    int smem;
    int ch;
};

// SET: the persistent bucket-set kernel (world >= 2) instead of the per-call one
template <typename TG, int MODE, int WORLD, bool SET>
TmaLaunch pick_tma_w() {
    using C = TmaCfg<TG, WORLD, MODE>;
    if constexpr (SET) {
        if constexpr (WORLD < 2) return {nullptr, 0, 0, 0};
        else return {gdraa_tma_set_kernel<TG, WORLD, MODE>, C::THREADS, C::SMEM, C::CH};
    } else {
        return {gdraa_tma_kernel<TG, WORLD, MODE>, C::THREADS, C::SMEM, C::CH};
    }
}

template <typename TG, int MODE, bool SET>
TmaLaunch pick_tma_m(int world) {
    switch (world) {
        case 1: return pick_tma_w<TG, MODE, 1, SET>();
        case 2: return pick_tma_w<TG, MODE, 2, SET>();
        case 3: return pick_tma_w<TG, MODE, 3, SET>();
        case 4: return pick_tma_w<TG, MODE, 4, SET>();
        case 5: return pick_tma_w<TG, MODE, 5, SET>();
        case 6: return pick_tma_w<TG, MODE, 6, SET>();
        case 7: return pick_tma_w<TG, MODE, 7, SET>();
        case 8: return pick_tma_w<TG, MODE, 8, SET>();
        default: return {nullptr, 0, 0, 0};
    }
}

template <typename TG, bool SET = false>
TmaLaunch pick_tma_t(int mode, int world) {
    switch (mode) {
        case kMean: return pick_tma_m<TG, kMean, SET>(world);
        case kSgd: return pick_tma_m<TG, kSgd, SET>(world);
        case kSgdMp: return pick_tma_m<TG, kSgdMp, SET>(world);
        default: return {nullptr, 0, 0, 0};
    }
}

// Grid sizing for shards smaller than a full wave: one CTA per end-game (small) chunk, so
// a mid-size call spreads over every SM instead of one CTA per big chunk (a CTA moves
// only ~5 GB/s over NVLink, so few CTAs make a mid-size call latency-bound).
// GDRAA_GRID_SMALL=0 sizes by big chunks (the earlier rule; A/B measurements only).
bool grid_by_small_chunks() {
    static const bool v = [] {
        const char *e = std::getenv("GDRAA_GRID_SMALL");
        return e == nullptr || e[0] != '0';
    }();
    return v;
}

int env_max_ctas() {
    static const int v = [] {
        const char *e = std::getenv("GDRAA_MAX_CTAS");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// ---------------------------------------------------------------------------------
// Launch shapes (measured on B200): vectors in flight per
// thread U, CTA size and CTAs per SM.
// ---------------------------------------------------------------------------------
// N <= 2 (profiles/r04_tune*.jsonl): 1024 threads x U=2 is the best or within 1% of it
// for both dtypes and modes (N=1 sgd 87.9 us vs 97.6 us for 512 x U=4; N=2 sgd 174.0 us).
// N = 4 (profiles/r06_tune_n4.jsonl): 2 CTAs x 512 threads x U=2 is best for all four
// (f32 sgd 247.9 us vs 252.5 us at 1 CTA/SM).  N > 4 keeps 2 x 512 with U=1 so that N
// sources in flight still fit the 64 registers of two 512-thread CTAs per SM.
// N = 1 with the dynamic schedule (profiles/r09_tune_n1.jsonl): 2 x 512 threads, U=1 is
// best (84.1 us = 6081 GB/s vs 88.2 us for 1024 x U=2).
// N = 1 (the local fused SGD): once the division by N = 1 compiles to nothing, the
// round-1 shape (U1 x 512 x 2/SM) pipelines into 58 registers and 2 CTAs per SM, 2%
// slower than at 36 registers (profiles/r65_ab_mc_ve_dist.json); re-swept
// (profiles/r66_tune_n1_lsu.jsonl, tools/tune lsu): U4 x 512 x 1/SM is the fastest.
// GDRAA_N1_U / _THREADS / _MINB override it at compile time (A/B builds only).
#ifndef GDRAA_N1_U
#define GDRAA_N1_U 4
#define GDRAA_N1_THREADS 512
#define GDRAA_N1_MINB 1
#endif
template <typename TG, int WORLD, int MODE> struct Shape {
    static constexpr int U = WORLD == 1 ? GDRAA_N1_U : (WORLD <= 4 ? 2 : 1);
    static constexpr int THREADS = WORLD == 1 ? GDRAA_N1_THREADS : (WORLD == 2 ? 1024 : 512);
    static constexpr int MINB = WORLD == 1 ? GDRAA_N1_MINB : (WORLD == 2 ? 1 : 2);
};

using KernelFn = void (*)(KParams);

struct Launch {
    KernelFn fn;
    int threads;
    int u;
};

template <typename TG, int MODE, int WORLD>
Launch pick_w() {
    using S = Shape<TG, WORLD, MODE>;
    return {gdraa_kernel<TG, WORLD, MODE, S::U, S::THREADS, S::MINB>, S::THREADS, S::U};
}

template <typename TG, int MODE>
Launch pick_m(int world) {
    switch (world) {
        case 1: return pick_w<TG, MODE, 1>();
        case 2: return pick_w<TG, MODE, 2>();
        case 3: return pick_w<TG, MODE, 3>();
        case 4: return pick_w<TG, MODE, 4>();
        case 5: return pick_w<TG, MODE, 5>();
        case 6: return pick_w<TG, MODE, 6>();
        case 7: return pick_w<TG, MODE, 7>();
        case 8: return pick_w<TG, MODE, 8>();
        default: return {nullptr, 0, 0};
    }
}

template <typename TG>
Launch pick_t(int mode, int world) {
    switch (mode) {
        case kMean: return pick_m<TG, kMean>(world);
        case kSgd: return pick_m<TG, kSgd>(world);
        case kSgdMp: return pick_m<TG, kSgdMp>(world);
        default: return {nullptr, 0, 0};
    }
}

Launch pick(int dtype, int mode, int world) {
    return dtype == GDRAA_F32 ? pick_t<float>(mode, world) : pick_t<__nv_bfloat16>(mode, world);
}

}  // namespace

cudaError_t launch_gdraa_exit(const KParams &p, int vr_rows, bool cooperative, cudaStream_t s) {
    dim3 grid(1, vr_rows), block(32);
    if (cooperative) {
        void *args[] = {const_cast<KParams *>(&p)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(gdraa_exit_kernel),
                                           grid, block, args, 0, s);
    }
    gdraa_exit_kernel<<<grid, block, 0, s>>>(p);
    return cudaGetLastError();
}

int max_ctas(int dtype, int mode, int world) {
    Launch l = pick(dtype, mode, world);
    if (l.fn == nullptr) return 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    // co-resident CTAs per device and kernel, queried once (it is on the launch path)
    static int cache[64][2][kModes][kMaxWorld + 1];
    int &c = cache[dev][dtype == GDRAA_F32 ? 0 : 1][mode][world];
    if (c == 0) {
        int sms = 0, per_sm = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            return 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, l.fn, l.threads, 0) !=
            cudaSuccess)
            return 0;
        c = sms * per_sm;
    }
    return c;
}

cudaError_t launch_gdraa(const KParams &p, int dtype, int mode, int vr_rows, bool cooperative,
                         cudaStream_t s, int *grid_x_out) {
    Launch l = pick(dtype, mode, p.world);
    if (l.fn == nullptr) return cudaErrorInvalidValue;
    // GDRAA_MAX_CTAS (tuning only): cap the grid, e.g. to leave SMs to a concurrent
    // backward pass when buckets are reduced on a side stream (NEXT-3).
    const int env_cap = env_max_ctas();
    int cap = max_ctas(dtype, mode, p.world) / vr_rows;
    if (env_cap > 0 && env_cap < cap) cap = env_cap;
    if (cap < 1) return cudaErrorInvalidConfiguration;
    const uint64_t nvec = (p.blk + E - 1) / E;
    const uint64_t per_chunk =
        static_cast<uint64_t>(l.threads) * (grid_by_small_chunks() ? 1 : l.u);
    const uint64_t want = (nvec + per_chunk - 1) / per_chunk;   // chunks of the largest shard
    int gx = static_cast<int>(want < static_cast<uint64_t>(cap) ? want : cap);
    if (gx < 1) gx = 1;
    if (grid_x_out) *grid_x_out = gx;
    dim3 grid(gx, vr_rows), block(l.threads);
    if (cooperative) {
        void *args[] = {const_cast<KParams *>(&p)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(l.fn), grid, block,
                                           args, 0, s);
    }
    return launch_pdl(l.fn, grid, block, s, p);
}

cudaError_t launch_gdraa_ll(const KParams &p, int dtype, int vr_rows, bool cooperative,
                            cudaStream_t s) {
    KernelFnLL fn = dtype == GDRAA_F32 ? pick_ll_t<float>(p.world)
                                       : pick_ll_t<__nv_bfloat16>(p.world);
    if (fn == nullptr) return cudaErrorInvalidValue;
    const uint64_t es = dtype == GDRAA_F32 ? 4 : 2;
    if (p.n * es > 8 * p.ll_pairs) return cudaErrorInvalidValue;
    constexpr int kT = 512;
    const uint64_t npairs = (p.n * es + 7) / 8;   // one thread per 8-byte payload pair
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    uint64_t gx = (npairs + kT - 1) / kT;
    // all resident (2 CTAs of 512 per SM); GDRAA_MAX_CTAS caps it further, e.g. to leave
    // SMs to a concurrent backward pass -- the grid-stride loop is correct at any size
    uint64_t cap = static_cast<uint64_t>(sms) * 2 / vr_rows;
    const int env_cap = env_max_ctas();
    if (env_cap > 0 && static_cast<uint64_t>(env_cap) < cap) cap = env_cap;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    dim3 grid(static_cast<unsigned>(gx), vr_rows), block(kT);
    if (cooperative) {
        void *args[] = {const_cast<KParams *>(&p)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(fn), grid, block, args,
                                           0, s);
    }
    return launch_pdl(fn, grid, block, s, p);
}

namespace {
template <typename TG, int MODE>
KernelFnLL pick_ll_sgd_m(int world) {
    switch (world) {
        case 2: return gdraa_ll_sgd_kernel<TG, 2, MODE>;
        case 3: return gdraa_ll_sgd_kernel<TG, 3, MODE>;
        case 4: return gdraa_ll_sgd_kernel<TG, 4, MODE>;
        case 5: return gdraa_ll_sgd_kernel<TG, 5, MODE>;
        case 6: return gdraa_ll_sgd_kernel<TG, 6, MODE>;
        case 7: return gdraa_ll_sgd_kernel<TG, 7, MODE>;
        case 8: return gdraa_ll_sgd_kernel<TG, 8, MODE>;
        default: return nullptr;
    }
}
}  // namespace

bool ll_sgd_fits(uint64_t blk, int dtype, int mode, uint64_t ll_pairs) {
    const uint64_t sg = dtype == GDRAA_F32 ? 4 : 2, sw = mode == kSgdMp ? 2 : 4;
    return (blk * sg + 7) / 8 + (blk * sw + 7) / 8 <= ll_pairs;
}

cudaError_t launch_gdraa_ll_sgd(const KParams &p, int dtype, int mode, int vr_rows,
                                bool cooperative, cudaStream_t s) {
    KernelFnLL fn = nullptr;
    if (mode == kSgd)
        fn = dtype == GDRAA_F32 ? pick_ll_sgd_m<float, kSgd>(p.world)
                                : pick_ll_sgd_m<__nv_bfloat16, kSgd>(p.world);
    else if (mode == kSgdMp)
        fn = dtype == GDRAA_F32 ? pick_ll_sgd_m<float, kSgdMp>(p.world)
                                : pick_ll_sgd_m<__nv_bfloat16, kSgdMp>(p.world);
    if (fn == nullptr) return cudaErrorInvalidValue;
    if (!ll_sgd_fits(p.blk, dtype, mode, p.ll_pairs)) return cudaErrorInvalidValue;
    constexpr int kT = 512;
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kT, 0);
    if (e != cudaSuccess) return e;
    // every CTA polls entries other CTAs (and peers) produce: the grid must be resident
    const uint64_t es = dtype == GDRAA_F32 ? 4 : 2;
    const uint64_t rs_pairs = (p.blk * es + 7) / 8, units = (p.blk + E - 1) / E;
    const uint64_t work = rs_pairs > units ? rs_pairs : units;
    uint64_t gx = (work + kT - 1) / kT;
    // GDRAA_MAX_CTAS caps it further (a smaller grid is resident all the more; every
    // phase is a grid-stride loop)
    uint64_t cap = static_cast<uint64_t>(sms) * per_sm / vr_rows;
    const int env_cap = env_max_ctas();
    if (env_cap > 0 && static_cast<uint64_t>(env_cap) < cap) cap = env_cap;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    dim3 grid(static_cast<unsigned>(gx), vr_rows), block(kT);
    if (cooperative) {
        void *args[] = {const_cast<KParams *>(&p)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(fn), grid, block, args,
                                           0, s);
    }
    return launch_pdl(fn, grid, block, s, p);
}

// Which data-movement variant serves a call (both produce the same bits): the TMA-staged
// kernel at every N >= 2.  Round 1 kept the LSU kernel for bf16 at N <= 2 (1-2.6% faster
// then, profiles/r23_bench_kernel_choice.json); with the per-CTA exit fence the TMA kernel
// wins every bf16 mode at N = 2 and 4 as well (profiles/r66_tune_choice.jsonl: sgd
// 123.5 vs 124.9 us, mean 87.9 vs 89.3, _mp 88.8 vs 90.7 at N = 2; 182.7 vs 188.1, 128.0
// vs 132.9, 128.9 vs 133.6 at N = 4).  N = 1 has no peers: the LSU kernel.
// GDRAA_KERNEL=lsu|tma forces one.
bool use_tma_kernel(int dtype, int mode, int world) {
    static const int forced = [] {
        const char *e = std::getenv("GDRAA_KERNEL");
        if (e == nullptr) return -1;
        return std::string(e) == "tma" ? 1 : (std::string(e) == "lsu" ? 0 : -1);
    }();
    (void)dtype;
    (void)mode;
    if (forced >= 0) return forced == 1;
    return world >= 2;
}

// Opt a TMA kernel in to > 48 KiB of dynamic shared memory (once per device and kernel)
// and return its co-resident CTAs per SM.
static cudaError_t tma_prepare(const TmaLaunch &l, int dev, int *per_sm) {
    static std::mutex mu;
    static std::map<std::pair<int, void *>, int> occ;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(dev, reinterpret_cast<void *>(l.fn));
    auto it = occ.find(key);
    if (it == occ.end()) {
        cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(l.fn),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, l.smem);
        if (e != cudaSuccess) return e;
        int n = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l.fn, l.threads, l.smem);
        if (e != cudaSuccess) return e;
        it = occ.emplace(key, n).first;
    }
    *per_sm = it->second;
    return cudaSuccess;
}

cudaError_t launch_gdraa_tma_set(const KParams &p, int dtype, int mode, int vr_rows,
                                 bool cooperative, cudaStream_t s, int ctas) {
    TmaLaunch l = dtype == GDRAA_F32 ? pick_tma_t<float, true>(mode, p.world)
                                     : pick_tma_t<__nv_bfloat16, true>(mode, p.world);
    if (l.fn == nullptr) return cudaErrorInvalidValue;
    int dev = 0, per_sm = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = tma_prepare(l, dev, &per_sm);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    int cap = sms * per_sm / vr_rows;
    if (ctas > 0 && ctas < cap) cap = ctas;
    if (cap < 1) return cudaErrorInvalidConfiguration;
    dim3 grid(cap, vr_rows), block(l.threads);
    if (cooperative) {
        void *args[] = {const_cast<KParams *>(&p)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(l.fn), grid, block,
                                           args, l.smem, s);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = l.smem;
    cfg.stream = s;
    return cudaLaunchKernelEx(&cfg, l.fn, p);
}

cudaError_t launch_gdraa_tma(const KParams &p, int dtype, int mode, int vr_rows,
                             bool cooperative, cudaStream_t s, int *grid_x_out) {
    TmaLaunch l = dtype == GDRAA_F32 ? pick_tma_t<float>(mode, p.world)
                                     : pick_tma_t<__nv_bfloat16>(mode, p.world);
    if (l.fn == nullptr) return cudaErrorInvalidValue;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int per_sm = 0, sms = 0;
    e = tma_prepare(l, dev, &per_sm);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    int cap = sms * per_sm / vr_rows;
    const int env_cap = env_max_ctas();
    if (env_cap > 0 && env_cap < cap) cap = env_cap;
    if (cap < 1) return cudaErrorInvalidConfiguration;
    const uint64_t ch = grid_by_small_chunks() ? l.ch / 4 : l.ch;   // end-game chunk: CH/4
    const uint64_t want = ((p.blk & ~7ull) + ch - 1) / ch;   // chunks of the largest shard
    int gx = static_cast<int>(want < static_cast<uint64_t>(cap) ? want : cap);
    if (gx < 1) gx = 1;
    if (grid_x_out) *grid_x_out = gx;
    dim3 grid(gx, vr_rows), block(l.threads);
    if (cooperative) {
        void *args[] = {const_cast<KParams *>(&p)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(l.fn), grid, block,
                                           args, l.smem, s);
    }
    static const bool pdl = [] {
        const char *x = std::getenv("GDRAA_PDL");
        return x == nullptr || x[0] != '0';
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = l.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, l.fn, p);
}

}  // namespace gdraa
