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
// 128-bit loads, all N sources in flight per thread), and store the result shard to
// all N ranks with 128-bit stores (posted NVLink writes).  Shard r is read and written
// by rank r only, so in-place allreduce is race free chunk by chunk.  The rounding of
// every operation is pinned (__fadd_rn / __fdiv_rn / __fmul_rn / __fsub_rn: never
// contracted into FMA), so the result is bitwise that of the CPU oracle.
//
// Tensor cores are not used: there is no contraction on this path.
#include <cuda_bf16.h>

#include <type_traits>

#include "gdraa_internal.h"

namespace gdraa {
namespace {

constexpr int kThreads = 512;

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
__device__ __forceinline__ void fence_acq_rel_sys() {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint64_t global_timer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Streaming 128-bit load: data is touched once, keep it out of L1.
__device__ __forceinline__ uint4 ld_stream(const void *p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_v4(void *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Spin until *flag >= target, bounded by timeout_ns of %globaltimer.
__device__ __forceinline__ bool wait_geq(const uint64_t *flag, uint64_t target,
                                         uint64_t timeout_ns) {
    if (ld_relaxed_sys(flag) < target) {
        const uint64_t t0 = global_timer_ns();
        while (ld_relaxed_sys(flag) < target) {
            if (global_timer_ns() - t0 > timeout_ns) return false;
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

// ---------------------------------------------------------------------------------
// Element access: 16 bytes of g per source per vector.
// ---------------------------------------------------------------------------------
template <typename TG> struct Elem;
template <> struct Elem<float> {
    static constexpr int E = 4;
    __device__ __forceinline__ static void widen(uint4 r, float (&f)[E]) {
        f[0] = __uint_as_float(r.x);
        f[1] = __uint_as_float(r.y);
        f[2] = __uint_as_float(r.z);
        f[3] = __uint_as_float(r.w);
    }
    __device__ __forceinline__ static uint4 narrow(const float (&f)[E]) {
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
    static constexpr int E = 8;
    __device__ __forceinline__ static float lo(uint32_t u) { return __uint_as_float(u << 16); }
    __device__ __forceinline__ static float hi(uint32_t u) {
        return __uint_as_float(u & 0xFFFF0000u);
    }
    __device__ __forceinline__ static void widen(uint4 r, float (&f)[E]) {
        f[0] = lo(r.x); f[1] = hi(r.x); f[2] = lo(r.y); f[3] = hi(r.y);
        f[4] = lo(r.z); f[5] = hi(r.z); f[6] = lo(r.w); f[7] = hi(r.w);
    }
    __device__ __forceinline__ static uint32_t pack(float a, float b) {
        const uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(a));
        const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(b));
        return l | (h << 16);
    }
    __device__ __forceinline__ static uint4 narrow(const float (&f)[E]) {
        return make_uint4(pack(f[0], f[1]), pack(f[2], f[3]), pack(f[4], f[5]), pack(f[6], f[7]));
    }
    __device__ __forceinline__ static float load1(const void *p, uint64_t i) {
        return lo(static_cast<const uint16_t *>(p)[i]);
    }
    __device__ __forceinline__ static void store1(void *p, uint64_t i, float m) {
        static_cast<__nv_bfloat16 *>(p)[i] = __float2bfloat16_rn(m);
    }
};

// Aggregation: s = x_0; s = fl(s + x_p) for p = 1..N-1; m = fl(s / N).
template <int WORLD>
__device__ __forceinline__ float average(const float (&x)[WORLD]) {
    float s = x[0];
#pragma unroll
    for (int q = 1; q < WORLD; ++q) s = __fadd_rn(s, x[q]);
    return __fdiv_rn(s, static_cast<float>(WORLD));
}

// Update: v = fl(fl(mom*v) + m); w = fl(w - fl(lr*v)).
__device__ __forceinline__ void sgd(float m, float lr, float mom, float &w, float &v) {
    const float t = __fmul_rn(mom, v);
    v = __fadd_rn(t, m);
    const float u = __fmul_rn(lr, v);
    w = __fsub_rn(w, u);
}

// ---------------------------------------------------------------------------------
// The fused kernel.  TG: gradient / buffer element type; WORLD: N; MODE: kMean or
// kSgd; U: vectors per thread in flight per iteration (memory-level parallelism).
// ---------------------------------------------------------------------------------
template <typename TG, int WORLD, int MODE, int U>
__global__ void __launch_bounds__(kThreads)
gdraa_kernel(const __grid_constant__ KParams p) {
    using EL = Elem<TG>;
    constexpr int E = EL::E;
    const int vr = blockIdx.y;
    const int rank = p.rank0 + vr;
    Pad *mine = p.pad[vr][rank];
    __shared__ int s_abort;
    __shared__ int s_last;

    // All CTAs read the epoch before any of them can arrive at the exit counter, and the
    // last CTA updates it only after every CTA arrived: one consistent value per call.
    const uint64_t epoch = *reinterpret_cast<volatile uint64_t *>(&mine->epoch) + 1;
    if (threadIdx.x == 0) s_abort = 0;

    // a2: "2nd synchronization" -- every peer's D(i) is final (stream-ordered after its
    // backward) before anyone reads it or writes into it.
    if (WORLD > 1) {
        if (blockIdx.x == 0 && threadIdx.x < WORLD && threadIdx.x != rank)
            st_release_sys(&p.pad[vr][threadIdx.x]->entry[rank], epoch);
        __syncthreads();
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            if (!wait_geq(&mine->entry[threadIdx.x], epoch, p.timeout_ns)) {
                report_timeout(p.err, 1, threadIdx.x, vr);
                s_abort = 1;
            }
        }
        __syncthreads();
        if (s_abort) return;
    }

    // a1: this rank's block D(., r), Q-aligned ceil partition (AMB-8).
    const uint64_t off = min(static_cast<uint64_t>(rank) * p.blk, p.n);
    const uint64_t len = min(p.blk, p.n - off);
    const uint64_t nvec = len / E;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
    uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;

    const float lr = p.lr, mom = p.mom;
    float *const vloc = p.v[vr];
    void *const wloc = p.dst[vr][rank];

    auto process = [&](uint64_t i0, auto ucount) {
        constexpr int UU = decltype(ucount)::value;
        uint4 raw[UU][WORLD];
        float wv[UU][E], vv[UU][E];
        // a3: reduce -- all N sources in flight at once (local HBM + N-1 NVLink peers).
#pragma unroll
        for (int u = 0; u < UU; ++u) {
            const uint64_t e0 = off + (i0 + u * stride) * E;
#pragma unroll
            for (int q = 0; q < WORLD; ++q)
                raw[u][q] = ld_stream(static_cast<const TG *>(p.src[vr][q]) + e0);
            if (MODE == kSgd) {
#pragma unroll
                for (int k = 0; k < E / 4; ++k) {
                    const float4 a = *reinterpret_cast<const float4 *>(
                        static_cast<const float *>(wloc) + e0 + 4 * k);
                    const float4 b = *reinterpret_cast<const float4 *>(vloc + e0 + 4 * k);
                    wv[u][4 * k + 0] = a.x; wv[u][4 * k + 1] = a.y;
                    wv[u][4 * k + 2] = a.z; wv[u][4 * k + 3] = a.w;
                    vv[u][4 * k + 0] = b.x; vv[u][4 * k + 1] = b.y;
                    vv[u][4 * k + 2] = b.z; vv[u][4 * k + 3] = b.w;
                }
            }
        }
        // a4 (+ a5): aggregate (and update) in registers.
        float out[UU][E];
#pragma unroll
        for (int u = 0; u < UU; ++u) {
            float x[WORLD][E];
#pragma unroll
            for (int q = 0; q < WORLD; ++q) EL::widen(raw[u][q], x[q]);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                float col[WORLD];
#pragma unroll
                for (int q = 0; q < WORLD; ++q) col[q] = x[q][e];
                const float m = average<WORLD>(col);
                if (MODE == kSgd) {
                    sgd(m, lr, mom, wv[u][e], vv[u][e]);
                    out[u][e] = wv[u][e];
                } else {
                    out[u][e] = m;
                }
            }
        }
        // a6: broadcast -- push the block to every rank (own copy last).
#pragma unroll
        for (int u = 0; u < UU; ++u) {
            const uint64_t e0 = off + (i0 + u * stride) * E;
            if (MODE == kSgd) {
#pragma unroll
                for (int k = 0; k < E / 4; ++k)
                    *reinterpret_cast<float4 *>(vloc + e0 + 4 * k) =
                        make_float4(vv[u][4 * k], vv[u][4 * k + 1], vv[u][4 * k + 2],
                                    vv[u][4 * k + 3]);
#pragma unroll
                for (int k = 0; k < E / 4; ++k) {
                    const uint4 o = make_uint4(
                        __float_as_uint(out[u][4 * k]), __float_as_uint(out[u][4 * k + 1]),
                        __float_as_uint(out[u][4 * k + 2]), __float_as_uint(out[u][4 * k + 3]));
#pragma unroll
                    for (int j = 1; j <= WORLD; ++j) {
                        const int q = (rank + j) % WORLD;
                        st_v4(static_cast<float *>(p.dst[vr][q]) + e0 + 4 * k, o);
                    }
                }
            } else {
                const uint4 o = EL::narrow(out[u]);
#pragma unroll
                for (int j = 1; j <= WORLD; ++j) {
                    const int q = (rank + j) % WORLD;
                    st_v4(static_cast<TG *>(p.dst[vr][q]) + e0, o);
                }
            }
        }
    };

    if (U > 1) {
        for (; i + (U - 1) * stride < nvec; i += U * stride)
            process(i, std::integral_constant<int, U>{});
    }
    for (; i < nvec; i += stride) process(i, std::integral_constant<int, 1>{});

    // Ragged tail of the last non-empty shard (len % E elements), scalar.
    if (blockIdx.x == gridDim.x - 1) {
        for (uint64_t t = nvec * E + threadIdx.x; t < len; t += kThreads) {
            const uint64_t e = off + t;
            float col[WORLD];
#pragma unroll
            for (int q = 0; q < WORLD; ++q) col[q] = EL::load1(p.src[vr][q], e);
            const float m = average<WORLD>(col);
            if (MODE == kSgd) {
                float w = static_cast<const float *>(wloc)[e], v = vloc[e];
                sgd(m, lr, mom, w, v);
                vloc[e] = v;
                for (int j = 1; j <= WORLD; ++j)
                    static_cast<float *>(p.dst[vr][(rank + j) % WORLD])[e] = w;
            } else {
                for (int j = 1; j <= WORLD; ++j) EL::store1(p.dst[vr][(rank + j) % WORLD], e, m);
            }
        }
    }

    // a7: "1st synchronization" -- our pushes are performed system-wide, then the last
    // CTA of this rank tells every peer and waits until every peer has done the same.
    fence_acq_rel_sys();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&mine->arrive, 1u);
        s_last = (prev == gridDim.x - 1);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    if (WORLD > 1) {
        if (threadIdx.x < WORLD && threadIdx.x != rank)
            st_release_sys(&p.pad[vr][threadIdx.x]->exit[rank], epoch);
        if (threadIdx.x < WORLD && threadIdx.x != rank) {
            if (!wait_geq(&mine->exit[threadIdx.x], epoch, p.timeout_ns)) {
                report_timeout(p.err, 2, threadIdx.x, vr);
                s_abort = 1;
            }
        }
        __syncthreads();
        if (s_abort) return;
    }
    if (threadIdx.x == 0) {
        mine->arrive = 0;
        mine->calls += 1;
        if (WORLD > 1) mine->sync_waits += 2;
        mine->epoch = epoch;
        if (p.done[vr] != nullptr) *p.done[vr] = epoch;   // job-server "IterDone" flag
    }
}

// ---------------------------------------------------------------------------------
// Dispatch
// ---------------------------------------------------------------------------------
// Vectors in flight per thread: enough 16-byte loads to cover NVLink latency without
// spilling (bf16 vectors expand to 8 fp32 values each, so they get half the depth).
template <typename TG, int WORLD> constexpr int unroll_for() {
    return sizeof(TG) == 4 ? (WORLD <= 2 ? 4 : (WORLD <= 4 ? 2 : 1)) : (WORLD <= 2 ? 2 : 1);
}

using KernelFn = void (*)(KParams);

template <typename TG, int MODE, int WORLD>
KernelFn pick_w() { return gdraa_kernel<TG, WORLD, MODE, unroll_for<TG, WORLD>()>; }

template <typename TG, int MODE>
KernelFn pick_m(int world) {
    switch (world) {
        case 1: return pick_w<TG, MODE, 1>();
        case 2: return pick_w<TG, MODE, 2>();
        case 3: return pick_w<TG, MODE, 3>();
        case 4: return pick_w<TG, MODE, 4>();
        case 5: return pick_w<TG, MODE, 5>();
        case 6: return pick_w<TG, MODE, 6>();
        case 7: return pick_w<TG, MODE, 7>();
        case 8: return pick_w<TG, MODE, 8>();
        default: return nullptr;
    }
}

KernelFn pick(int dtype, int mode, int world) {
    if (dtype == GDRAA_F32)
        return mode == kSgd ? pick_m<float, kSgd>(world) : pick_m<float, kMean>(world);
    return mode == kSgd ? pick_m<__nv_bfloat16, kSgd>(world) : pick_m<__nv_bfloat16, kMean>(world);
}

}  // namespace

int max_ctas(int dtype, int mode, int world) {
    KernelFn fn = pick(dtype, mode, world);
    if (fn == nullptr) return 0;
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess)
        return 0;
    return sms * per_sm;
}

cudaError_t launch_gdraa(const KParams &p, int dtype, int mode, int vr_rows, bool cooperative,
                         cudaStream_t s, int *grid_x_out) {
    KernelFn fn = pick(dtype, mode, p.world);
    if (fn == nullptr) return cudaErrorInvalidValue;
    const int cap = max_ctas(dtype, mode, p.world) / vr_rows;
    if (cap < 1) return cudaErrorInvalidConfiguration;
    const int E = dtype == GDRAA_F32 ? 4 : 8;
    const uint64_t nvec = (p.blk + E - 1) / E;
    const uint64_t want = (nvec + kThreads - 1) / kThreads;
    int gx = static_cast<int>(want < static_cast<uint64_t>(cap) ? want : cap);
    if (gx < 1) gx = 1;
    if (grid_x_out) *grid_x_out = gx;
    dim3 grid(gx, vr_rows), block(kThreads);
    if (cooperative) {
        void *args[] = {const_cast<KParams *>(&p)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(fn), grid, block, args,
                                           0, s);
    }
    fn<<<grid, block, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace gdraa
