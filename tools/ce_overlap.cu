// ce_overlap.cu -- NEXT-3 probe (DESIGN.md §11/§12): does a copy-engine data path overlap a
// backward pass better than an SM-driven one?  The paper moves its blocks with the NIC's
// RDMA engine, i.e. with no SM involvement; on B200 the copy engines are
// that engine.  SM-driven collectives (the library's kernels, NCCL) take SMs from the
// backward's GEMMs; copy engines do not.
//
// Single process, two devices (peer access), cross-device order by events (no flag
// barriers, identical for both paths, so the comparison isolates the data mover).
// A synthetic backward of K compute-bound kernels (FMA loops on every SM) produces the
// gradient buffer bucket by bucket, last bucket first; after kernel k both devices' bucket
// k is "final".  Each bucket is then reduced (mean of the two ranks, owner shard), applied
// (momentum SGD) and broadcast by
//   sm : one fused kernel per bucket with C CTAs: pull the peer's shard, fold, update,
//        push w' to the peer (the library's data flow, LSU-style)
//   ce : cudaMemcpyAsync of the peer's shard into a receive buffer (copy engine), a
//        fold+update kernel with C CTAs from local HBM, cudaMemcpyAsync of w' to the peer
// Prints per mode: backward alone, buckets alone, serial, overlapped (us, max over
// devices).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ce_overlap tools/ce_overlap.cu
//   ./tools/ce_overlap [L=25557032] [K=4] [spin_iters] [iters=20]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
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

// compute-bound stand-in for one backward GEMM: every thread runs `iters` dependent FMAs
__global__ void spin(float *sink, int iters) {
    float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
        a = fmaf(a, b, c);
        b = fmaf(b, 0.99999f, c);
    }
    if (a == 12345.f) sink[threadIdx.x] = a + b;
}

// mean of own and peer g (N = 2: an exact multiply), v = 0.9 v + m, w = w - 0.1 v;
// PUSH: also store w' into the peer's w
// U vectors per thread in flight (all loads before any use), as the library's LSU kernel
template <bool PULL, bool PUSH, int U = 4>
__global__ void fold_update(const float4 *__restrict__ own, const float4 *__restrict__ other,
                            float4 *__restrict__ w, float4 *__restrict__ v,
                            float4 *__restrict__ peer_w, size_t n4, int own_first) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i0 < n4; i0 += U * stride) {
        float4 o[U], r[U], ww[U], vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = i0 + u * stride;
            if (i < n4) {
                o[u] = own[i];
                r[u] = other[i];   // PULL: `other` is the peer's g (NVLink)
                ww[u] = w[i];
                vv[u] = v[i];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = i0 + u * stride;
            if (i >= n4) break;
            const float4 a = own_first ? o[u] : r[u], b = own_first ? r[u] : o[u];
            float m;
#define UPD(c)                                                                           \
    m = __fmul_rn(__fadd_rn(a.c, b.c), 0.5f);                                            \
    vv[u].c = __fadd_rn(__fmul_rn(0.9f, vv[u].c), m);                                    \
    ww[u].c = __fsub_rn(ww[u].c, __fmul_rn(0.1f, vv[u].c));
            UPD(x) UPD(y) UPD(z) UPD(w)
#undef UPD
            w[i] = ww[u];
            v[i] = vv[u];
            if (PUSH) peer_w[i] = ww[u];
        }
    }
    (void)PULL;
}

struct Dev {
    float *g, *w, *v, *rb, *sink;
    cudaStream_t comp, comm, srs, sag;
    std::vector<cudaEvent_t> ready, done;
    cudaEvent_t t0, t1, j;
    int sms;
};

int main(int argc, char **argv) {
    const size_t L = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 25557032;
    const int K = argc > 2 ? std::atoi(argv[2]) : 4;
    int spin_iters = argc > 3 ? std::atoi(argv[3]) : 0;
    const int iters = argc > 4 ? std::atoi(argv[4]) : 20;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
        std::printf("{\"error\": \"need 2 GPUs\"}\n");
        return 1;
    }
    Dev D[2];
    const size_t Lp = (L + 255) / 256 * 256;
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&D[d].g, Lp * 4));
        CK(cudaMalloc(&D[d].w, Lp * 4));
        CK(cudaMalloc(&D[d].v, Lp * 4));
        CK(cudaMalloc(&D[d].rb, Lp * 4));
        CK(cudaMalloc(&D[d].sink, 4096));
        CK(cudaMemset(D[d].g, 0, Lp * 4));
        CK(cudaMemset(D[d].w, 0, Lp * 4));
        CK(cudaMemset(D[d].v, 0, Lp * 4));
        for (cudaStream_t *s : {&D[d].comp, &D[d].comm, &D[d].srs, &D[d].sag})
            CK(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
        D[d].ready.resize(K);
        D[d].done.resize(K);
        for (int k = 0; k < K; ++k) {
            CK(cudaEventCreateWithFlags(&D[d].ready[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&D[d].done[k], cudaEventDisableTiming));
        }
        CK(cudaEventCreate(&D[d].t0));
        CK(cudaEventCreate(&D[d].t1));
        CK(cudaEventCreateWithFlags(&D[d].j, cudaEventDisableTiming));
        CK(cudaDeviceGetAttribute(&D[d].sms, cudaDevAttrMultiProcessorCount, d));
    }
    // buckets: K equal ranges (multiples of 256 elements), last first
    std::vector<std::pair<size_t, size_t>> B;
    for (int k = K - 1; k >= 0; --k) {
        const size_t a = Lp * k / K / 256 * 256, b = Lp * (k + 1) / K / 256 * 256;
        B.push_back({a, b - a});
    }
    auto shard = [&](size_t count, int r, size_t &off, size_t &len) {
        const size_t blk = ((count + 1) / 2 + 63) / 64 * 64;
        off = std::min(r * blk, count);
        len = std::min(blk, count - off);
    };
    auto bwd_piece = [&](int d) {
        spin<<<D[d].sms * 4, 256, 0, D[d].comp>>>(D[d].sink, spin_iters);
        CK(cudaGetLastError());
    };
    // one bucket on device d, after both devices' ready[k]; records done[k] on its last stream
    auto bucket = [&](int d, int k, const std::string &mode, int ctas) {
        const int p = 1 - d;
        size_t off, len;
        shard(B[k].second, d, off, len);
        const size_t a = B[k].first + off;
        if (mode == "sm") {
            CK(cudaStreamWaitEvent(D[d].comm, D[d].ready[k], 0));
            CK(cudaStreamWaitEvent(D[d].comm, D[p].ready[k], 0));
            fold_update<true, true><<<ctas, 512, 0, D[d].comm>>>(
                reinterpret_cast<const float4 *>(D[d].g + a), reinterpret_cast<const float4 *>(D[p].g + a),
                reinterpret_cast<float4 *>(D[d].w + a), reinterpret_cast<float4 *>(D[d].v + a),
                reinterpret_cast<float4 *>(D[p].w + a), len / 4, d == 0);
            CK(cudaGetLastError());
            CK(cudaEventRecord(D[d].done[k], D[d].comm));
        } else {
            CK(cudaStreamWaitEvent(D[d].srs, D[d].ready[k], 0));
            CK(cudaStreamWaitEvent(D[d].srs, D[p].ready[k], 0));
            CK(cudaMemcpyAsync(D[d].rb + a, D[p].g + a, len * 4, cudaMemcpyDeviceToDevice, D[d].srs));
            fold_update<false, false><<<ctas, 512, 0, D[d].srs>>>(
                reinterpret_cast<const float4 *>(D[d].g + a), reinterpret_cast<const float4 *>(D[d].rb + a),
                reinterpret_cast<float4 *>(D[d].w + a), reinterpret_cast<float4 *>(D[d].v + a),
                nullptr, len / 4, d == 0);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(D[p].w + a, D[d].w + a, len * 4, cudaMemcpyDeviceToDevice, D[d].srs));
            CK(cudaEventRecord(D[d].done[k], D[d].srs));
        }
    };
    // what = 0 backward alone, 1 buckets alone, 2 serial, 3 overlapped
    auto run = [&](int what, const std::string &mode, int ctas) {
        auto once = [&]() {
            for (int k = 0; k < K; ++k)
                for (int d = 0; d < 2; ++d) {
                    CK(cudaSetDevice(d));
                    if (what != 1) bwd_piece(d);
                    CK(cudaEventRecord(D[d].ready[k], D[d].comp));
                }
            if (what == 0) return;
            if (what == 2)   // serial: the buckets start after the whole backward
                for (int d = 0; d < 2; ++d) {
                    CK(cudaSetDevice(d));
                    CK(cudaEventRecord(D[d].j, D[d].comp));
                }
            for (int k = 0; k < K; ++k)
                for (int d = 0; d < 2; ++d) {
                    CK(cudaSetDevice(d));
                    if (what == 2) {
                        CK(cudaStreamWaitEvent(mode == "sm" ? D[d].comm : D[d].srs, D[0].j, 0));
                        CK(cudaStreamWaitEvent(mode == "sm" ? D[d].comm : D[d].srs, D[1].j, 0));
                    }
                    bucket(d, k, mode, ctas);
                }
            // the iteration ends when both devices' last buckets are done (the exit sync)
            for (int d = 0; d < 2; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaStreamWaitEvent(D[d].comp, D[0].done[K - 1], 0));
                CK(cudaStreamWaitEvent(D[d].comp, D[1].done[K - 1], 0));
            }
        };
        for (int i = 0; i < 3; ++i) once();
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(D[d].t0, D[d].comp));
        }
        for (int i = 0; i < iters; ++i) once();
        float worst = 0.f;
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventRecord(D[d].t1, D[d].comp));
            CK(cudaEventSynchronize(D[d].t1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, D[d].t0, D[d].t1));
            worst = ms > worst ? ms : worst;
        }
        return worst * 1e3 / iters;
    };
    if (spin_iters == 0) {   // calibrate: K pieces ~ 150 us in total
        spin_iters = 1000;
        for (;;) {
            const double us = run(0, "sm", 0);
            if (us >= 150.0 || spin_iters > 10000000) break;
            spin_iters = static_cast<int>(spin_iters * 150.0 / (us > 1 ? us : 1) * 1.05) + 1;
        }
    }
    const double bwd = run(0, "sm", 0);
    for (const char *mode : {"sm", "ce"})
        for (int ctas : {16, 32, 64, 148}) {
            const double alone = run(1, mode, ctas), serial = run(2, mode, ctas),
                         over = run(3, mode, ctas);
            std::printf("{\"probe\": \"ce_overlap\", \"L\": %zu, \"buckets\": %d, \"mode\": \"%s\", "
                        "\"ctas\": %d, \"spin_iters\": %d, \"bwd_us\": %.1f, \"buckets_alone_us\": %.1f, "
                        "\"serial_us\": %.1f, \"overlap_us\": %.1f}\n",
                        L, K, mode, ctas, spin_iters, bwd, alone, serial, over);
            std::fflush(stdout);
        }
    return 0;
}
