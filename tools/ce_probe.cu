// ce_probe.cu -- upper bound of a copy-engine-driven GDRAA step: could the
// copy engines, which move ~760 GB/s of data per direction against ~700 for SM-issued
// NVLink traffic, carry the step's reduce-scatter and all-gather while the SMs only fold
// and update from local HBM?
//
// Single process, two devices (peer access).  Per device d and chunk k of its shard
// (K chunks), all on d's own streams:
//   rs[k]:  cudaMemcpyAsync  peer g shard chunk k  -> local receive buffer   (CE pull)
//   red[k]: a fold + momentum-SGD kernel over chunk k (own g, received chunk, w, v)
//   ag[k]:  cudaMemcpyAsync  local w' chunk k      -> peer w                 (CE push)
// with events rs[k] -> red[k] -> ag[k]; rs copies on one stream, kernels on another, ag
// copies on a third, so chunk k's reduce overlaps chunk k+1's pull and chunk k-1's push.
// No cross-device synchronisation is modelled (it would only add to the time), so the
// result is a LOWER bound on a CE-driven step.  Prints one JSON line per (L, K).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ce_probe tools/ce_probe.cu
//   ./tools/ce_probe [L=25557032] [iters=20]
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

// m = (g_own + g_rx) / 2 (N = 2: an exact multiply), v = mom v + m, w = w - lr v
__global__ void fold_update(const float4 *__restrict__ own, const float4 *__restrict__ rx,
                            float4 *__restrict__ w, float4 *__restrict__ v, size_t n4, int own_first) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
         i += (size_t)gridDim.x * blockDim.x) {
        const float4 a = own_first ? own[i] : rx[i], b = own_first ? rx[i] : own[i];
        float4 ww = w[i], vv = v[i];
        float m;
#define UPD(c)                                                                           \
    m = __fmul_rn(__fadd_rn(a.c, b.c), 0.5f);                                            \
    vv.c = __fadd_rn(__fmul_rn(0.9f, vv.c), m);                                          \
    ww.c = __fsub_rn(ww.c, __fmul_rn(0.1f, vv.c));
        UPD(x) UPD(y) UPD(z) UPD(w)
#undef UPD
        w[i] = ww;
        v[i] = vv;
    }
}

int main(int argc, char **argv) {
    const size_t L = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 25557032;
    const int iters = argc > 2 ? std::atoi(argv[2]) : 20;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
        std::printf("{\"error\": \"need 2 GPUs\"}\n");
        return 1;
    }
    const size_t shard = ((L + 1) / 2 + 63) / 64 * 64;   // elements per rank's shard
    struct Dev {
        float *g, *w, *v, *rb;
        cudaStream_t srs, sred, sag;
        int sms;
    } D[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&D[d].g, 2 * shard * 4));
        CK(cudaMalloc(&D[d].w, 2 * shard * 4));
        CK(cudaMalloc(&D[d].v, 2 * shard * 4));
        CK(cudaMalloc(&D[d].rb, shard * 4));
        CK(cudaMemset(D[d].g, 0, 2 * shard * 4));
        CK(cudaMemset(D[d].w, 0, 2 * shard * 4));
        CK(cudaMemset(D[d].v, 0, 2 * shard * 4));
        CK(cudaStreamCreateWithFlags(&D[d].srs, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&D[d].sred, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&D[d].sag, cudaStreamNonBlocking));
        CK(cudaDeviceGetAttribute(&D[d].sms, cudaDevAttrMultiProcessorCount, d));
    }
    for (int K : {1, 4, 8, 16, 32, 64}) {
        const size_t ch = (shard + K - 1) / K / 64 * 64 + 64;   // chunk elements
        std::vector<std::vector<cudaEvent_t>> ers(2), ered(2);
        std::vector<cudaEvent_t> t0(2), t1(2), join_rs(2), join_ag(2);
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            ers[d].resize(K);
            ered[d].resize(K);
            for (int k = 0; k < K; ++k) {
                CK(cudaEventCreateWithFlags(&ers[d][k], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ered[d][k], cudaEventDisableTiming));
            }
            CK(cudaEventCreate(&t0[d]));
            CK(cudaEventCreate(&t1[d]));
            CK(cudaEventCreateWithFlags(&join_rs[d], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&join_ag[d], cudaEventDisableTiming));
        }
        auto step = [&](int d) {
            const int p = 1 - d;
            // rank d owns shard d: pull the peer's g shard d, push w' shard d into the peer
            const float *peer_g = D[p].g + d * shard;
            float *peer_w = D[p].w + d * shard;
            for (int k = 0; k < K; ++k) {
                const size_t a = k * ch, n = a >= shard ? 0 : (shard - a < ch ? shard - a : ch);
                if (n == 0) break;
                CK(cudaMemcpyAsync(D[d].rb + a, peer_g + a, n * 4, cudaMemcpyDeviceToDevice, D[d].srs));
                CK(cudaEventRecord(ers[d][k], D[d].srs));
                CK(cudaStreamWaitEvent(D[d].sred, ers[d][k], 0));
                fold_update<<<D[d].sms * 2, 512, 0, D[d].sred>>>(
                    reinterpret_cast<const float4 *>(D[d].g + d * shard + a),
                    reinterpret_cast<const float4 *>(D[d].rb + a),
                    reinterpret_cast<float4 *>(D[d].w + d * shard + a),
                    reinterpret_cast<float4 *>(D[d].v + d * shard + a), n / 4, d == 0);
                CK(cudaGetLastError());
                CK(cudaEventRecord(ered[d][k], D[d].sred));
                CK(cudaStreamWaitEvent(D[d].sag, ered[d][k], 0));
                CK(cudaMemcpyAsync(peer_w + a, D[d].w + d * shard + a, n * 4,
                                   cudaMemcpyDeviceToDevice, D[d].sag));
            }
            // the step ends when all three streams are done
            CK(cudaEventRecord(join_rs[d], D[d].sag));
            CK(cudaStreamWaitEvent(D[d].srs, join_rs[d], 0));
        };
        // warm-up
        for (int it = 0; it < 3; ++it)
            for (int d = 0; d < 2; ++d) {
                CK(cudaSetDevice(d));
                step(d);
            }
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaDeviceSynchronize());
        }
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventRecord(t0[d], D[d].srs));
            CK(cudaStreamWaitEvent(D[d].sred, t0[d], 0));
            CK(cudaStreamWaitEvent(D[d].sag, t0[d], 0));
        }
        for (int it = 0; it < iters; ++it)
            for (int d = 0; d < 2; ++d) {
                CK(cudaSetDevice(d));
                step(d);
            }
        float worst = 0.f;
        for (int d = 0; d < 2; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventRecord(t1[d], D[d].srs));
            CK(cudaEventSynchronize(t1[d]));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, t0[d], t1[d]));
            worst = ms > worst ? ms : worst;
        }
        const double us = worst * 1e3 / iters;
        const double bnv = 2.0 * shard * 4;   // per direction: pulled g shard + pushed w' shard
        std::printf("{\"probe\": \"ce_step\", \"L\": %zu, \"K\": %d, \"us_per_step\": %.2f, "
                    "\"bus_gbs_per_direction\": %.1f, \"frac_of_770\": %.3f}\n",
                    L, K, us, bnv / (us * 1e-6) / 1e9, bnv / (us * 1e-6) / 1e9 / 770.0);
        std::fflush(stdout);
    }
    return 0;
}
