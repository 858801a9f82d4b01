// nvls_probe.cu -- NVLS in-switch reduction (multimem.ld_reduce) as the reduce step of the
// GDRAA iteration ("multimem.ld_reduce for the RS is excluded unless
// proven deterministic").  Two questions, one process, one device per rank:
//
//  1. Bits.  Every rank reads the whole gradient buffer through the multicast address with
//     multimem.ld_reduce.add.f32 (the switch returns the sum over the N ranks' copies).
//     Is that sum (a) the same on every rank and on a repeated run, and (b) equal to the
//     oracle's rank-ordered left fold fl(fl(g0 + g1) + g2) ... (O3)?  Every left-fold
//     permutation and the balanced trees are scored so the switch's order can be named.
//  2. Rate.  The data movement of allreduce_mean (RS + mean + AG of the mean) three ways,
//     back-to-back on all devices, max over devices:
//       unicast : the library's pattern -- pull the shard from every peer (ld.global),
//                 fold, divide, store the mean to every rank (N-1 peer stores)
//       nvls_uc : ld_reduce the shard through the switch, divide, unicast stores to every rank
//       nvls_mc : ld_reduce, divide, one multimem.st (the switch writes every rank's copy)
//     and the reduce half alone (nvls_rs: ld_reduce + local store).  Reported as µs and as
//     NCCL busBW = 2(N-1)/N * L * 4 / t.
//
// Inputs are gradient-like fp32 (random sign, exponents over 2^-24..2^0, full mantissas),
// generated on the host with a counter-based splitmix64 (no method arithmetic).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/nvls_probe \
//        tools/nvls_probe.cu -lcuda
//   tools/nvls_probe [N] [L] [iters]
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            std::printf("{\"error\": \"%s:%d %s\"}\n", __FILE__, __LINE__,               \
                        cudaGetErrorString(e_));                                         \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)
#define CU(x)                                                                            \
    do {                                                                                 \
        CUresult r_ = (x);                                                               \
        if (r_ != CUDA_SUCCESS) {                                                        \
            const char *s_ = nullptr;                                                    \
            cuGetErrorString(r_, &s_);                                                   \
            std::printf("{\"error\": \"%s:%d %s: %s\"}\n", __FILE__, __LINE__, #x,       \
                        s_ ? s_ : "?");                                                  \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)

constexpr int kMax = 8;

__device__ __forceinline__ float4 ld_reduce4(const float *mc) {
    float4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(mc)
                 : "memory");
    return r;
}
__device__ __forceinline__ void mc_st4(float *mc, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc),
                 "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ float4 ld_nc4(const float *p) {
    float4 r;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

struct Ptrs {
    const float *g[kMax];   // every rank's gradient (unicast VA, peer-accessible)
    float *w[kMax];         // every rank's output buffer (unicast VA)
    const float *mcg;       // this device's multicast VA of the gradient buffers
    float *mcw;             // this device's multicast VA of the output buffers
};

// 1. the switch's sum of the whole buffer into a local array
__global__ void reduce_all(const float *mcg, float *out, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x)
        reinterpret_cast<float4 *>(out)[i] = ld_reduce4(mcg + 4 * i);
}

// 2. data movement of allreduce_mean on this rank's shard [off, off + len), len % 4 == 0
template <int MODE>   // 0 unicast, 1 nvls_uc, 2 nvls_mc, 3 nvls_rs
__global__ void __launch_bounds__(512) step(Ptrs p, int n, int rank, size_t off, size_t len4) {
    const float inv = 1.0f / n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len4;
         i += (size_t)gridDim.x * blockDim.x) {
        const size_t e = off + 4 * i;
        float4 s;
        if (MODE == 0) {
            float4 x[kMax];
#pragma unroll
            for (int q = 0; q < kMax; ++q)
                if (q < n) x[q] = ld_nc4(p.g[q] + e);
            s = x[0];
#pragma unroll
            for (int q = 1; q < kMax; ++q)
                if (q < n) {
                    s.x += x[q].x; s.y += x[q].y; s.z += x[q].z; s.w += x[q].w;
                }
        } else {
            s = ld_reduce4(p.mcg + e);
        }
        s.x *= inv; s.y *= inv; s.z *= inv; s.w *= inv;
        if (MODE == 2) {
            mc_st4(p.mcw + e, s);
        } else if (MODE == 3) {
            *reinterpret_cast<float4 *>(p.w[rank] + e) = s;
        } else {
#pragma unroll
            for (int j = 1; j <= kMax; ++j)
                if (j <= n)
                    *reinterpret_cast<float4 *>(p.w[(rank + j) % n] + e) = s;
        }
    }
}

static uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static float grad_value(int rank, size_t i) {
    const uint64_t h = splitmix((static_cast<uint64_t>(rank) << 40) ^ i ^ 0x5EEDull);
    const uint32_t mant = static_cast<uint32_t>(h) & 0x7FFFFFu;
    const int ex = static_cast<int>((h >> 23) % 25);   // 2^-24 .. 2^0
    const uint32_t sign = static_cast<uint32_t>((h >> 40) & 1u) << 31;
    const uint32_t bits = sign | (static_cast<uint32_t>(127 - ex) << 23) | mant;
    float f;
    std::memcpy(&f, &bits, 4);
    return f;
}
static uint32_t bits_of(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

struct Multicast {
    std::vector<float *> local, mcva;
};

// One multicast object over n devices; each device binds `bytes` of its own VMM memory
// (accessible from every device, so unicast peer loads / stores work on the same memory).
static Multicast make_multicast(int n, size_t bytes) {
    CUmulticastObjectProp prop = {};
    prop.numDevices = n;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    prop.size = bytes;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t sz = (bytes + gran - 1) / gran * gran;
    prop.size = sz;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &prop));
    for (int d = 0; d < n; ++d) {
        CUdevice dev;
        CU(cuDeviceGet(&dev, d));
        CU(cuMulticastAddDevice(mc, dev));
    }
    std::vector<CUmemAccessDesc> acc(n);
    for (int q = 0; q < n; ++q) {
        acc[q] = {};
        acc[q].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[q].location.id = q;
        acc[q].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    Multicast m;
    m.local.resize(n);
    m.mcva.resize(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CUmemAllocationProp ap = {};
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = d;
        CUmemGenericAllocationHandle ph;
        CU(cuMemCreate(&ph, sz, &ap, 0));
        CU(cuMulticastBindMem(mc, 0, ph, 0, sz, 0));
        CUdeviceptr va = 0, mva = 0;
        CU(cuMemAddressReserve(&va, sz, 0, 0, 0));
        CU(cuMemMap(va, sz, 0, ph, 0));
        CU(cuMemSetAccess(va, sz, acc.data(), n));
        CU(cuMemAddressReserve(&mva, sz, 0, 0, 0));
        CU(cuMemMap(mva, sz, 0, mc, 0));
        CU(cuMemSetAccess(mva, sz, &acc[d], 1));
        CK(cudaMemset(reinterpret_cast<void *>(va), 0, sz));
        CK(cudaDeviceSynchronize());
        m.local[d] = reinterpret_cast<float *>(va);
        m.mcva[d] = reinterpret_cast<float *>(mva);
    }
    return m;
}

int main(int argc, char **argv) {
    CU(cuInit(0));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    const int n = argc > 1 ? std::atoi(argv[1]) : ndev;
    const size_t L = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 25557032ull;
    const int iters = argc > 3 ? std::atoi(argv[3]) : 50;
    if (n < 2 || n > ndev || n > kMax) {
        std::printf("{\"error\": \"need 2..%d devices, have %d\"}\n", kMax, ndev);
        return 1;
    }
    const size_t Lp = (L + 255) / 256 * 256;   // padded so every shard is whole float4s
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < n; ++q)
            if (q != d) {
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, d, q));
                if (ok) CK(cudaDeviceEnablePeerAccess(q, 0));
            }
    }
    Multicast G = make_multicast(n, Lp * 4), Wb = make_multicast(n, Lp * 4);

    // gradient-like inputs, rank r on device r
    std::vector<std::vector<float>> gh(n, std::vector<float>(Lp, 0.0f));
    for (int r = 0; r < n; ++r) {
        for (size_t i = 0; i < L; ++i) gh[r][i] = grad_value(r, i);
        CK(cudaSetDevice(r));
        CK(cudaMemcpy(G.local[r], gh[r].data(), Lp * 4, cudaMemcpyHostToDevice));
    }

    // ---- 1. bits -----------------------------------------------------------------------
    const size_t NB = std::min<size_t>(Lp, 1u << 22);   // 4 Mi elements checked bit by bit
    std::vector<std::vector<uint32_t>> got(n, std::vector<uint32_t>(NB));
    std::vector<uint32_t> again(NB);
    std::vector<float *> outd(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMalloc(&outd[d], NB * 4));
        reduce_all<<<592, 512>>>(G.mcva[d], outd[d], NB / 4);
        CK(cudaGetLastError());
    }
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(got[d].data(), outd[d], NB * 4, cudaMemcpyDeviceToHost));
    }
    CK(cudaSetDevice(0));
    reduce_all<<<592, 512>>>(G.mcva[0], outd[0], NB / 4);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(again.data(), outd[0], NB * 4, cudaMemcpyDeviceToHost));
    size_t cross = 0, rerun = 0;
    for (size_t i = 0; i < NB; ++i) {
        for (int d = 1; d < n; ++d) cross += got[d][i] != got[0][i];
        rerun += again[i] != got[0][i];
    }
    std::printf("{\"probe\": \"nvls_bits_determinism\", \"n\": %d, \"elements\": %zu, "
                "\"mismatch_across_ranks\": %zu, \"mismatch_rerun\": %zu}\n", n, NB, cross, rerun);

    // candidate orders: every left-fold permutation, and (n = 4) the three balanced trees
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    struct Cand { std::string name; size_t match; };
    std::vector<Cand> cands;
    auto score = [&](const std::string &name, auto sum_fn) {
        size_t m = 0;
        for (size_t i = 0; i < NB; ++i) m += bits_of(sum_fn(i)) == got[0][i];
        cands.push_back({name, m});
    };
    do {
        std::string name = "left";
        for (int q : perm) name += std::to_string(q);
        const std::vector<int> pm = perm;
        score(name, [&](size_t i) {
            float s = gh[pm[0]][i];
            for (int k = 1; k < n; ++k) s = s + gh[pm[k]][i];
            return s;
        });
    } while (std::next_permutation(perm.begin(), perm.end()));
    if (n == 4) {
        const int pairs[3][4] = {{0, 1, 2, 3}, {0, 2, 1, 3}, {0, 3, 1, 2}};
        for (const auto &pr : pairs) {
            std::string name = "tree(" + std::to_string(pr[0]) + std::to_string(pr[1]) + ")(" +
                               std::to_string(pr[2]) + std::to_string(pr[3]) + ")";
            score(name, [&](size_t i) {
                const float a = gh[pr[0]][i] + gh[pr[1]][i];
                const float b = gh[pr[2]][i] + gh[pr[3]][i];
                return a + b;
            });
        }
    }
    // exact sum rounded once (double is exact for 4 terms of these magnitudes only
    // approximately; reported as a reference point)
    score("fl(exact)", [&](size_t i) {
        double s = 0;
        for (int q = 0; q < n; ++q) s += gh[q][i];
        return static_cast<float>(s);
    });
    std::sort(cands.begin(), cands.end(), [](const Cand &a, const Cand &b) { return a.match > b.match; });
    const size_t oracle_match = [&] {
        for (const auto &c : cands) {
            std::string want = "left";
            for (int q = 0; q < n; ++q) want += std::to_string(q);
            if (c.name == want) return c.match;
        }
        return size_t(0);
    }();
    std::printf("{\"probe\": \"nvls_bits_order\", \"n\": %d, \"elements\": %zu, "
                "\"oracle_left_fold_match\": %zu, \"oracle_left_fold_mismatch_frac\": %.6f, "
                "\"best\": [", n, NB, oracle_match, 1.0 - double(oracle_match) / NB);
    for (size_t k = 0; k < std::min<size_t>(cands.size(), 6); ++k)
        std::printf("%s{\"order\": \"%s\", \"match_frac\": %.6f}", k ? ", " : "",
                    cands[k].name.c_str(), double(cands[k].match) / NB);
    std::printf("]}\n");
    std::fflush(stdout);

    // ---- 2. rate -----------------------------------------------------------------------
    const size_t c = (Lp + n - 1) / n;
    const size_t blk = (c + 63) / 64 * 64;
    std::vector<Ptrs> P(n);
    for (int d = 0; d < n; ++d) {
        for (int q = 0; q < n; ++q) {
            P[d].g[q] = G.local[q];
            P[d].w[q] = Wb.local[q];
        }
        P[d].mcg = G.mcva[d];
        P[d].mcw = Wb.mcva[d];
    }
    const char *names[4] = {"unicast", "nvls_uc", "nvls_mc", "nvls_rs"};
    for (int rep = 0; rep < 2; ++rep) {
        for (int mode = 0; mode < 4; ++mode) {
            std::vector<cudaEvent_t> a(n), b(n);
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaDeviceSynchronize());
            }
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventCreate(&a[d]));
                CK(cudaEventCreate(&b[d]));
                const size_t off = std::min(d * blk, Lp), len = std::min(blk, Lp - off);
                auto launch = [&] {
                    switch (mode) {
                        case 0: step<0><<<296, 512>>>(P[d], n, d, off, len / 4); break;
                        case 1: step<1><<<296, 512>>>(P[d], n, d, off, len / 4); break;
                        case 2: step<2><<<296, 512>>>(P[d], n, d, off, len / 4); break;
                        default: step<3><<<296, 512>>>(P[d], n, d, off, len / 4); break;
                    }
                };
                for (int k = 0; k < 3; ++k) launch();
                CK(cudaEventRecord(a[d]));
                for (int k = 0; k < iters; ++k) launch();
                CK(cudaEventRecord(b[d]));
                CK(cudaGetLastError());
            }
            float worst = 0.f;
            for (int d = 0; d < n; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventSynchronize(b[d]));
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, a[d], b[d]));
                worst = std::max(worst, ms);
            }
            const double us = worst * 1e3 / iters;
            const double busbw = 2.0 * (n - 1) / n * L * 4 / (us * 1e-6) / 1e9;
            std::printf("{\"probe\": \"nvls_rate\", \"mode\": \"%s\", \"rep\": %d, \"n\": %d, "
                        "\"L\": %zu, \"us\": %.2f, \"busbw_gbs\": %.1f}\n",
                        names[mode], rep, n, L, us, busbw);
            std::fflush(stdout);
        }
    }
    // the nvls_mc output must equal the mean of the switch's sum on every rank (sanity)
    std::vector<uint32_t> wv(NB);
    size_t bad = 0;
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMemcpy(wv.data(), Wb.local[d], NB * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < NB; ++i) {
            float s;
            std::memcpy(&s, &got[0][i], 4);
            bad += wv[i] != bits_of(s * (1.0f / n));
        }
    }
    std::printf("{\"probe\": \"nvls_output_check\", \"n\": %d, \"mismatch\": %zu}\n", n, bad);
    return 0;
}
