// mc_probe.cu -- can this box's NVSwitch do multicast (NVLS), and what does a device
// barrier cost with one multicast reduction per rank (an O(1)-message
// signal pad) versus N-1 unicast flag stores per rank (the library's barrier)?
//
// Single process, one device per rank, all devices of the box (or argv[1]).  Each rank
// runs one kernel of K back-to-back barrier rounds (one CTA; thread 0 signals, polls):
//   unicast:   st.release.sys of epoch e into every peer's slot[rank]; poll own slots
//   multicast: multimem.red.release.sys.global.add.u64 [mc], 1 (the switch adds 1 into
//              every rank's copy); poll own copy >= e * N
// and prints the per-round time (max over ranks).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mc_probe \
//        tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
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

__device__ __forceinline__ uint64_t ld_acq(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// The library's scheme: thread q (q != rank) stores into peer q's slot and polls our slot q,
// in parallel, then the CTA synchronises.
__global__ void unicast_rounds(uint64_t *const *peer_slots, uint64_t *mine, int rank, int n,
                               int rounds) {
    const int q = threadIdx.x;
    for (uint64_t e = 1; e <= static_cast<uint64_t>(rounds); ++e) {
        if (q < n && q != rank) {
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_slots[q] + rank),
                         "l"(e)
                         : "memory");
            while (ld_acq(mine + q) < e) {
            }
        }
        __syncthreads();
    }
}

__global__ void multicast_rounds(uint64_t *mc, const uint64_t *mine, int n, int rounds) {
    if (threadIdx.x != 0) return;
    for (uint64_t e = 1; e <= static_cast<uint64_t>(rounds); ++e) {
        asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc), "l"(1ull)
                     : "memory");
        while (ld_acq(mine) < e * n) {
        }
    }
}

int main(int argc, char **argv) {
    CU(cuInit(0));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    int n = argc > 1 ? std::atoi(argv[1]) : ndev;
    const int rounds = argc > 2 ? std::atoi(argv[2]) : 10000;
    if (n < 2 || n > ndev || n > kMax) {
        std::printf("{\"error\": \"need 2..%d devices, have %d\"}\n", kMax, ndev);
        return 1;
    }
    int mc_ok = 1;
    for (int d = 0; d < n; ++d) {
        CUdevice dev;
        CU(cuDeviceGet(&dev, d));
        int v = 0;
        CU(cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
        mc_ok &= v;
    }
    std::printf("{\"probe\": \"multicast_supported\", \"n\": %d, \"value\": %d}\n", n, mc_ok);
    std::fflush(stdout);

    // --- unicast barrier (the library's scheme) -------------------------------------
    std::vector<uint64_t *> slots(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < n; ++q)
            if (q != d) CK(cudaDeviceEnablePeerAccess(q, 0));
        CK(cudaMalloc(&slots[d], kMax * sizeof(uint64_t)));
        CK(cudaMemset(slots[d], 0, kMax * sizeof(uint64_t)));
    }
    std::vector<uint64_t **> tab(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMalloc(&tab[d], n * sizeof(uint64_t *)));
        CK(cudaMemcpy(tab[d], slots.data(), n * sizeof(uint64_t *), cudaMemcpyHostToDevice));
        CK(cudaDeviceSynchronize());
    }
    auto time_all = [&](auto launch) {
        std::vector<cudaEvent_t> a(n), b(n);
        for (int d = 0; d < n; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventCreate(&a[d]));
            CK(cudaEventCreate(&b[d]));
            CK(cudaEventRecord(a[d]));
            launch(d);
            CK(cudaEventRecord(b[d]));
        }
        float worst = 0.f;
        for (int d = 0; d < n; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventSynchronize(b[d]));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, a[d], b[d]));
            worst = ms > worst ? ms : worst;
        }
        return worst;
    };
    const float uni_ms = time_all([&](int d) {
        unicast_rounds<<<1, 32>>>(tab[d], slots[d], d, n, rounds);
        CK(cudaGetLastError());
    });
    std::printf("{\"probe\": \"unicast_barrier\", \"n\": %d, \"rounds\": %d, \"us_per_round\": %.3f}\n",
                n, rounds, uni_ms * 1e3 / rounds);
    std::fflush(stdout);
    if (!mc_ok) return 0;

    // --- multicast barrier -----------------------------------------------------------
    CUmulticastObjectProp prop = {};
    prop.numDevices = n;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    prop.size = 1;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    prop.size = gran;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &prop));
    for (int d = 0; d < n; ++d) {
        CUdevice dev;
        CU(cuDeviceGet(&dev, d));
        CU(cuMulticastAddDevice(mc, dev));
    }
    std::vector<uint64_t *> uc(n), mcp(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        CUdevice dev;
        CU(cuDeviceGet(&dev, d));
        CUmemAllocationProp ap = {};
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = d;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        size_t ag = 0;
        CU(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
        const size_t sz = gran > ag ? gran : ag;
        CUmemGenericAllocationHandle ph;
        CU(cuMemCreate(&ph, sz, &ap, 0));
        CU(cuMulticastBindMem(mc, 0, ph, 0, gran, 0));
        CUmemAccessDesc acc = {};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = d;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CUdeviceptr va = 0, mva = 0;
        CU(cuMemAddressReserve(&va, sz, 0, 0, 0));
        CU(cuMemMap(va, sz, 0, ph, 0));
        CU(cuMemSetAccess(va, sz, &acc, 1));
        CU(cuMemAddressReserve(&mva, gran, 0, 0, 0));
        CU(cuMemMap(mva, gran, 0, mc, 0));
        CU(cuMemSetAccess(mva, gran, &acc, 1));
        uc[d] = reinterpret_cast<uint64_t *>(va);
        mcp[d] = reinterpret_cast<uint64_t *>(mva);
        CK(cudaMemset(uc[d], 0, 64));
        CK(cudaDeviceSynchronize());
    }
    const float mc_ms = time_all([&](int d) {
        multicast_rounds<<<1, 32>>>(mcp[d], uc[d], n, rounds);
        CK(cudaGetLastError());
    });
    std::printf("{\"probe\": \"multicast_barrier\", \"n\": %d, \"rounds\": %d, \"us_per_round\": %.3f, "
                "\"granularity\": %zu}\n", n, rounds, mc_ms * 1e3 / rounds, gran);
    // check the final counters: rounds * n on every rank
    for (int d = 0; d < n; ++d) {
        uint64_t h = 0;
        CK(cudaSetDevice(d));
        CK(cudaMemcpy(&h, uc[d], 8, cudaMemcpyDeviceToHost));
        if (h != static_cast<uint64_t>(rounds) * n)
            std::printf("{\"error\": \"rank %d counter %llu != %llu\"}\n", d,
                        (unsigned long long)h, (unsigned long long)rounds * n);
    }
    // can the multicast handle be exported as a POSIX fd (cross-process sharing)?
    int fd = -1;
    CUresult r = cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    std::printf("{\"probe\": \"multicast_export_fd\", \"ok\": %d}\n", r == CUDA_SUCCESS && fd >= 0);
    return 0;
}
