// nvlink_probe.cu -- microbenchmark of SM-driven NVLink traffic between two B200s
// (single process, cudaDeviceEnablePeerAccess), to choose the data movement of the
// GDRAA kernel: peer loads (pull) vs peer stores (push) vs 1-D TMA bulk copies, run in
// both directions at once as the allreduce does.  Prints one JSON line per variant.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe nvlink_probe.cu
//   ./nvlink_probe [MiB per direction]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x,               \
                         cudaGetErrorString(e));                                         \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)

__device__ __forceinline__ uint4 ldg_na(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// dst[i] = src[i], U vectors per thread in flight.
template <int U>
__global__ void copy_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_na(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n; i += stride) dst[i] = ldg_na(src + i);
}

// 256-bit variant (sm_100 LDG.E.ENL2.256 / STG.E.ENL2.256): 32 bytes per thread.
struct alignas(32) V8 {
    uint32_t a[8];
};
__device__ __forceinline__ V8 ld8(const V8 *p) {
    V8 r;
    asm volatile("ld.global.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.a[0]), "=r"(r.a[1]), "=r"(r.a[2]), "=r"(r.a[3]), "=r"(r.a[4]),
                   "=r"(r.a[5]), "=r"(r.a[6]), "=r"(r.a[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(V8 *p, const V8 &v) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.a[0]),
                 "r"(v.a[1]), "r"(v.a[2]), "r"(v.a[3]), "r"(v.a[4]), "r"(v.a[5]), "r"(v.a[6]),
                 "r"(v.a[7])
                 : "memory");
}
template <int U>
__global__ void copy8_kernel(const V8 *__restrict__ src, V8 *__restrict__ dst, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        V8 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld8(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) st8(dst + i + u * stride, v[u]);
    }
}

// sum of two sources (one remote) into dst (the pull-reduce of the current kernel).
template <int U>
__global__ void pull_reduce_push(const uint4 *__restrict__ local, const uint4 *__restrict__ remote,
                                 uint4 *__restrict__ dst_local, uint4 *__restrict__ dst_remote,
                                 size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = ldg_na(local + i + u * stride);
            b[u] = ldg_na(remote + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float4 x = *reinterpret_cast<float4 *>(&a[u]), y = *reinterpret_cast<float4 *>(&b[u]);
            float4 s = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
            dst_local[i + u * stride] = *reinterpret_cast<uint4 *>(&s);
            dst_remote[i + u * stride] = *reinterpret_cast<uint4 *>(&s);
        }
    }
}

// 1-D TMA bulk copy global(remote) -> shared, then shared -> global(local) by the CTA.
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem), "r"(bytes),
                 "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *gmem, const void *smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(gmem), "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read(int) { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// TMA pull: STAGES x CHUNK bytes in flight per CTA; thread 0 issues, all threads copy
// smem -> local global (or the bulk store does it when kBulkStore).
template <int STAGES, int CHUNK, bool kBulkStore>
__global__ void tma_pull(const char *__restrict__ remote, char *__restrict__ dst, size_t bytes) {
    extern __shared__ __align__(128) char smem[];
    __shared__ uint64_t bars[STAGES];
    const size_t nchunks = bytes / CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    size_t c0 = blockIdx.x;
    const size_t step = gridDim.x;
    // prologue
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            size_t c = c0 + s * step;
            if (c < nchunks) {
                mbar_expect_tx(&bars[s], CHUNK);
                bulk_g2s(smem + s * CHUNK, remote + c * CHUNK, CHUNK, &bars[s]);
            }
        }
    }
    uint32_t phase[STAGES] = {};
    int s = 0;
    for (size_t it = 0;; ++it) {
        size_t c = c0 + it * step;
        if (c >= nchunks) break;
        mbar_wait(&bars[s], phase[s]);
        phase[s] ^= 1;
        if (kBulkStore) {
            if (threadIdx.x == 0) {
                bulk_s2g(dst + c * CHUNK, smem + s * CHUNK, CHUNK);
                bulk_commit();
                bulk_wait_read(0);
            }
        } else {
            const uint4 *sp = reinterpret_cast<const uint4 *>(smem + s * CHUNK);
            uint4 *dp = reinterpret_cast<uint4 *>(dst + c * CHUNK);
            for (int k = threadIdx.x; k < CHUNK / 16; k += blockDim.x) dp[k] = sp[k];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            size_t cn = c + STAGES * step;
            if (cn < nchunks) {
                mbar_expect_tx(&bars[s], CHUNK);
                bulk_g2s(smem + s * CHUNK, remote + cn * CHUNK, CHUNK, &bars[s]);
            }
        }
        s = (s + 1) % STAGES;
    }
    if (kBulkStore && threadIdx.x == 0) bulk_wait_all();
}

// TMA push: local global -> smem -> remote global (bulk store to the peer).
template <int STAGES, int CHUNK>
__global__ void tma_push(const char *__restrict__ src, char *__restrict__ remote, size_t bytes) {
    extern __shared__ __align__(128) char smem[];
    __shared__ uint64_t bars[STAGES];
    const size_t nchunks = bytes / CHUNK;
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase[STAGES] = {};
    size_t it = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        int s = it % STAGES;
        if (it >= STAGES) {  // wait until the bulk store that used this stage has read smem
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
        }
        mbar_expect_tx(&bars[s], CHUNK);
        bulk_g2s(smem + s * CHUNK, src + c * CHUNK, CHUNK, &bars[s]);
        mbar_wait(&bars[s], phase[s]);
        phase[s] ^= 1;
        bulk_s2g(remote + c * CHUNK, smem + s * CHUNK, CHUNK);
        bulk_commit();
    }
    bulk_wait_all();
}

struct Pair {
    char *buf[2][3];   // per device: 3 buffers
};

static int g_sms = 148;

template <typename Launch>
double run_bidir(const char *name, size_t bytes, Launch launch, int iters = 20) {
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaStreamCreate(&st[d]));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
    }
    for (int w = 0; w < 3; ++w)
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            launch(d, st[d]);
        }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
    for (int i = 0; i < iters; ++i)
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            launch(d, st[d]);
        }
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], st[d])); }
    float ms[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        CK(cudaEventElapsedTime(&ms[d], e0[d], e1[d]));
        CK(cudaGetLastError());
    }
    double t = (ms[0] > ms[1] ? ms[0] : ms[1]) / iters;
    double gbs = bytes / (t * 1e-3) / 1e9;
    std::printf("{\"variant\": \"%s\", \"bytes_per_dir\": %zu, \"ms\": %.4f, \"gbs_per_dir\": %.1f}\n",
                name, bytes, t, gbs);
    std::fflush(stdout);
    return gbs;
}

int main(int argc, char **argv) {
    size_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 256;
    size_t bytes = mib << 20;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
        std::fprintf(stderr, "need 2 GPUs\n");
        return 1;
    }
    Pair p;
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        for (int b = 0; b < 3; ++b) {
            CK(cudaMalloc(&p.buf[d][b], bytes));
            CK(cudaMemset(p.buf[d][b], 1, bytes));
        }
    }
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t n16 = bytes / 16;
    // local HBM copy reference
    for (int grid_mult : {2, 4}) {
        char name[64];
        std::snprintf(name, sizeof name, "local_copy_u4_g%d", grid_mult);
        run_bidir(name, bytes, [&](int d, cudaStream_t s) {
            copy_kernel<4><<<g_sms * grid_mult, 512, 0, s>>>((const uint4 *)p.buf[d][0], (uint4 *)p.buf[d][1], n16);
        });
    }
    // pull: each device reads the peer's buffer into its own
    for (int grid_mult : {1, 2, 4})
        for (int u : {1, 4}) {
            char name[64];
            std::snprintf(name, sizeof name, "pull_u%d_g%d", u, grid_mult);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                if (u == 1)
                    copy_kernel<1><<<g_sms * grid_mult, 512, 0, s>>>((const uint4 *)p.buf[1 - d][0], (uint4 *)p.buf[d][1], n16);
                else
                    copy_kernel<4><<<g_sms * grid_mult, 512, 0, s>>>((const uint4 *)p.buf[1 - d][0], (uint4 *)p.buf[d][1], n16);
            });
        }
    // push: each device writes its buffer into the peer's
    for (int grid_mult : {1, 2, 4})
        for (int u : {1, 4}) {
            char name[64];
            std::snprintf(name, sizeof name, "push_u%d_g%d", u, grid_mult);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                if (u == 1)
                    copy_kernel<1><<<g_sms * grid_mult, 512, 0, s>>>((const uint4 *)p.buf[d][0], (uint4 *)p.buf[1 - d][2], n16);
                else
                    copy_kernel<4><<<g_sms * grid_mult, 512, 0, s>>>((const uint4 *)p.buf[d][0], (uint4 *)p.buf[1 - d][2], n16);
            });
        }
    // 256-bit pull / push
    for (int grid_mult : {1, 2}) {
        char name[64];
        std::snprintf(name, sizeof name, "pull_v8_u2_g%d", grid_mult);
        run_bidir(name, bytes, [&](int d, cudaStream_t s) {
            copy8_kernel<2><<<g_sms * grid_mult, 512, 0, s>>>((const V8 *)p.buf[1 - d][0], (V8 *)p.buf[d][1], bytes / 32);
        });
        std::snprintf(name, sizeof name, "push_v8_u2_g%d", grid_mult);
        run_bidir(name, bytes, [&](int d, cudaStream_t s) {
            copy8_kernel<2><<<g_sms * grid_mult, 512, 0, s>>>((const V8 *)p.buf[d][0], (V8 *)p.buf[1 - d][2], bytes / 32);
        });
    }
    // one-directional references (only device 0 moves data)
    {
        auto one = [&](const char *name, auto fn) {
            cudaEvent_t a, b;
            CK(cudaSetDevice(0));
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            for (int i = 0; i < 3; ++i) fn();
            CK(cudaEventRecord(a));
            for (int i = 0; i < 20; ++i) fn();
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            std::printf("{\"variant\": \"%s\", \"bytes_per_dir\": %zu, \"ms\": %.4f, \"gbs_per_dir\": %.1f}\n",
                        name, bytes, ms / 20, bytes / (ms / 20 * 1e-3) / 1e9);
            std::fflush(stdout);
        };
        one("oneway_push_u4", [&] { copy_kernel<4><<<g_sms * 2, 512>>>((const uint4 *)p.buf[0][0], (uint4 *)p.buf[1][2], n16); });
        one("oneway_pull_u4", [&] { copy_kernel<4><<<g_sms * 2, 512>>>((const uint4 *)p.buf[1][0], (uint4 *)p.buf[0][2], n16); });
        one("oneway_memcpy_peer", [&] { CK(cudaMemcpyPeerAsync(p.buf[1][2], 1, p.buf[0][0], 0, bytes, 0)); });
    }
    // pull-reduce-push (the current fused kernel's traffic at N=2 on half the bytes each way)
    for (int grid_mult : {1, 2, 4}) {
        char name[64];
        std::snprintf(name, sizeof name, "pull_reduce_push_u4_g%d", grid_mult);
        run_bidir(name, bytes, [&](int d, cudaStream_t s) {
            pull_reduce_push<4><<<g_sms * grid_mult, 512, 0, s>>>(
                (const uint4 *)p.buf[d][0], (const uint4 *)p.buf[1 - d][0], (uint4 *)p.buf[d][1],
                (uint4 *)p.buf[1 - d][2], n16 / 2);
        });
    }
    // TMA pull into smem
    {
        constexpr int ST = 4, CH = 16384;
        auto k1 = tma_pull<ST, CH, false>;
        auto k2 = tma_pull<ST, CH, true>;
        CK(cudaSetDevice(0)); CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
        CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
        CK(cudaSetDevice(1)); CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
        CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
        for (int grid_mult : {1, 2, 3}) {
            char name[64];
            std::snprintf(name, sizeof name, "tma_pull_st%d_ch%d_g%d", ST, CH, grid_mult);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                k1<<<g_sms * grid_mult, 256, ST * CH, s>>>(p.buf[1 - d][0], p.buf[d][1], bytes);
            });
            std::snprintf(name, sizeof name, "tma_pull_bulkstore_st%d_ch%d_g%d", ST, CH, grid_mult);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                k2<<<g_sms * grid_mult, 256, ST * CH, s>>>(p.buf[1 - d][0], p.buf[d][1], bytes);
            });
        }
    }
    {
        constexpr int ST = 4, CH = 16384;
        auto k = tma_push<ST, CH>;
        for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH)); }
        for (int grid_mult : {1, 2, 3}) {
            char name[64];
            std::snprintf(name, sizeof name, "tma_push_st%d_ch%d_g%d", ST, CH, grid_mult);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                k<<<g_sms * grid_mult, 32, ST * CH, s>>>(p.buf[d][0], p.buf[1 - d][2], bytes);
            });
        }
    }
    // How many SMs does each mechanism need?  (bidirectional, fixed per-CTA shapes)
    {
        constexpr int ST = 8, CH = 16384;
        auto kp = tma_pull<ST, CH, true>;
        auto ks = tma_push<ST, CH>;
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
            CK(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH));
        }
        for (int grid : {8, 16, 32, 64, 96, 148}) {
            char name[64];
            std::snprintf(name, sizeof name, "ctas%03d_pull_u4_1024thr", grid);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                copy_kernel<4><<<grid, 1024, 0, s>>>((const uint4 *)p.buf[1 - d][0], (uint4 *)p.buf[d][1], n16);
            });
            std::snprintf(name, sizeof name, "ctas%03d_push_u4_1024thr", grid);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                copy_kernel<4><<<grid, 1024, 0, s>>>((const uint4 *)p.buf[d][0], (uint4 *)p.buf[1 - d][2], n16);
            });
            std::snprintf(name, sizeof name, "ctas%03d_tma_pull_st8", grid);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                kp<<<grid, 32, ST * CH, s>>>(p.buf[1 - d][0], p.buf[d][1], bytes);
            });
            std::snprintf(name, sizeof name, "ctas%03d_tma_push_st8", grid);
            run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                ks<<<grid, 32, ST * CH, s>>>(p.buf[d][0], p.buf[1 - d][2], bytes);
            });
        }
    }
    // cudaMemcpyPeerAsync reference
    run_bidir("memcpy_peer", bytes, [&](int d, cudaStream_t s) {
        CK(cudaMemcpyPeerAsync(p.buf[1 - d][2], 1 - d, p.buf[d][0], d, bytes, s));
    });
    // Hybrid: can copy engines carry part of the traffic while SMs carry the rest, and
    // does the mix beat the SM-only ceiling?  Each device moves `bytes` per direction in
    // total: a fraction f by SM kernel (pull or push) on stream s, the rest by a
    // copy-engine push on a side stream, concurrently.
    {
        cudaStream_t side[2];
        cudaEvent_t fork[2], join[2];
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaStreamCreateWithFlags(&side[d], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&fork[d], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&join[d], cudaEventDisableTiming));
        }
        for (int pct : {25, 50, 75}) {
            const size_t sm_b = bytes / 100 * pct / 256 * 256, ce_b = bytes - sm_b;
            for (int kind = 0; kind < 2; ++kind) {   // 0: SM pull, 1: SM push
                for (int grid : {32, 0}) {
                    char name[96];
                    std::snprintf(name, sizeof name, "hybrid_sm%s%d_ctas%s_ce_push%d",
                                  kind ? "push" : "pull", pct, grid ? "032" : "all", 100 - pct);
                    run_bidir(name, bytes, [&](int d, cudaStream_t s) {
                        CK(cudaEventRecord(fork[d], s));
                        CK(cudaStreamWaitEvent(side[d], fork[d], 0));
                        CK(cudaMemcpyPeerAsync(p.buf[1 - d][2] + sm_b, 1 - d, p.buf[d][0] + sm_b, d,
                                               ce_b, side[d]));
                        const int gx = grid ? grid : g_sms;
                        if (kind == 0)
                            copy_kernel<4><<<gx, 1024, 0, s>>>((const uint4 *)p.buf[1 - d][0],
                                                               (uint4 *)p.buf[d][1], sm_b / 16);
                        else
                            copy_kernel<4><<<gx, 1024, 0, s>>>((const uint4 *)p.buf[d][0],
                                                               (uint4 *)p.buf[1 - d][1], sm_b / 16);
                        CK(cudaEventRecord(join[d], side[d]));
                        CK(cudaStreamWaitEvent(s, join[d], 0));
                    });
                }
            }
        }
    }
    return 0;
}
