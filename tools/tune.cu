// tune.cu -- launch-shape sweep of the GDRAA kernels on 1..4 B200s of one box, single
// process: rank d's kernel runs on device d and reaches its peers through
// cudaDeviceEnablePeerAccess pointers (same kernel code as the library; the IPC and job
// server plumbing is not involved).  Prints one JSON line per (kernel, shape, config),
// with a per-phase breakdown from %globaltimer stamps (kernels built with GDRAA_TRACE).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -o tools/tune tools/tune.cu -lcuda
//   ./tools/tune <world> <L> <f32|bf16> <sgd|mp|mean> [iters] [lib|lsu|tma|tail|ctas|solo]
//     lib : the library's launch shapes (LSU and TMA kernels)
//     lsu : sweep of the LSU kernel's (U, threads, CTAs/SM)
//     tma : sweep of the TMA kernel's (consumer warps, stages)
//     tail: end-game variants of the TMA kernel (small-chunk size, in-flight depth)
//     ctas: both kernels at grid caps 16/32/64/all (how many SMs the collective needs)
//     mc  : the TMA kernel with NVLS multicast all-gather and / or barriers (needs -lcuda)
//     solo: the library shapes with rank 0 alone (barriers pre-satisfied): one rank's
//           NVLink traffic in one direction pair, and a kernel ncu can replay
#define GDRAA_TRACE 1
#define GDRAA_EXPERIMENTAL 1   // the measured-and-rejected variants (multicast, dist exit)
#include "../paper_1802_02326_b200/csrc/gdraa_kernels.cu"

#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace gdraa;

#define CU(x)                                                                            \
    do {                                                                                 \
        CUresult r_ = (x);                                                               \
        if (r_ != CUDA_SUCCESS) {                                                        \
            const char *s_ = nullptr;                                                    \
            cuGetErrorString(r_, &s_);                                                   \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?"); \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)
#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x,               \
                         cudaGetErrorString(e));                                         \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)

struct Bufs {
    void *g[3];
    float *w[3], *v[3];
    void *model[3];   // bf16 model copy (mode mp: the all-gathered buffer; w is the master)
    Pad *pad;
    void *mc_dst[3];  // mc mode: multicast VA of this set's broadcast buffer (w or model)
    uint64_t *mc_bar, *bar_local;   // mc mode: multicast / local VA of {entry, exit} counters
};

static int W, NDEV;
static size_t L;
static int DT, MODE_;
static int ITERS = 50;
static std::string WHAT = "lsu";
static std::vector<Bufs> B;
static ErrBlock *err_d;
static std::vector<uint64_t *> TR;   // per-device trace ring (64 calls x 8 vr x 8 stamps)
// solo: only device 0 (rank 0) runs; its pad's entry/exit slots are pre-set past every
// epoch, so both barriers pass at once and the kernel moves rank 0's NVLink traffic alone
// (no kernel waits on another GPU: ncu kernel replay works on it).
static bool SOLO = false;
static uint32_t FLAGS = kFlagCtaFence;
// mc: NVLS multicast A/B: the broadcast buffers are VMM allocations
// bound to one multicast object per set (all N devices); MC_AG sends w' with one
// multimem.st per vector instead of N-1 unicast stores, MC_BAR runs both barriers as one
// multimem.red per rank.
static bool MC = false, MC_AG = false, MC_BAR = false;

// Time `fn` (grid gx x threads, dynamic smem) on all W devices; print one line.
template <typename TG, int WORLD, int MODE>
void run(void (*fn)(KParams), int threads, int smem, int gx, const char *kernel,
         const std::string &shape) {
    const uint64_t c = (L + WORLD - 1) / WORLD;
    const uint64_t blk = (c + kQuantum - 1) / kQuantum * kQuantum;
    std::vector<cudaStream_t> st(WORLD);
    std::vector<cudaEvent_t> e0(WORLD), e1(WORLD);
    for (int d = 0; d < WORLD; ++d) {
        CK(cudaSetDevice(d));
        if (smem > 48 * 1024)
            CK(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        CK(cudaStreamCreate(&st[d]));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
    }
    const int active = SOLO ? 1 : WORLD;
    auto launch = [&](int set) {
        for (int d = 0; d < active; ++d) {
            KParams p;
            std::memset(&p, 0, sizeof p);
            p.world = WORLD;
            p.rank0 = d;
            p.n = L;
            p.blk = blk;
            p.lr = 0.1f;
            p.mom = 0.9f;
            p.timeout_ns = 10ull * 1000000000ull;
            for (int q = 0; q < WORLD; ++q) {
                p.src[0][q] = B[q].g[set];
                p.dst[0][q] = MODE == kSgd   ? (void *)B[q].w[set]
                              : MODE == kSgdMp ? B[q].model[set]
                                               : B[q].g[set];
                p.pad[0][q] = B[q].pad;
            }
            p.v[0] = B[d].v[set];
            p.wm[0] = MODE == kSgdMp ? B[d].w[set] : nullptr;
            p.mc_dst[0] = MC_AG ? B[d].mc_dst[set] : nullptr;
            p.mc_bar[0] = MC_BAR ? B[d].mc_bar : nullptr;
            p.bar_local[0] = MC_BAR ? B[d].bar_local : nullptr;
            p.wd = MODE == kSgdMp ? 0.001f : 0.0f;
            p.flags = FLAGS;
            p.err = err_d;
            p.trace = TR[d];
            CK(cudaSetDevice(d));
            fn<<<dim3(gx, 1), threads, smem, st[d]>>>(p);
            CK(cudaGetLastError());
        }
    };
    for (int i = 0; i < 5; ++i) launch(i % 3);
    for (int d = 0; d < WORLD; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    for (int d = 0; d < active; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
    for (int i = 0; i < ITERS; ++i) launch(i % 3);
    float worst = 0;
    for (int d = 0; d < active; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e1[d], st[d]));
        CK(cudaEventSynchronize(e1[d]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
        worst = std::max(worst, ms);
    }
    if (err_d->code) {
        std::fprintf(stderr, "timeout reported\n");
        std::exit(2);
    }
    // stamps: 0 start, 1 entry passed, 5 first CTA data done, 6 last CTA data done,
    // 3 last CTA arrived (after its fence), 4 exit barrier passed
    double acc[6] = {0, 0, 0, 0, 0, 0};
    int cnt = 0;
    for (int d = 0; d < active; ++d) {
        std::vector<uint64_t> h(64 * kMaxWorld * 8);
        CK(cudaSetDevice(d));
        CK(cudaMemcpy(h.data(), TR[d], h.size() * 8, cudaMemcpyDeviceToHost));
        for (int e = 0; e < 64; ++e) {
            const uint64_t *a = &h[(e * kMaxWorld) * 8];
            const uint64_t *b = &h[(((e + 1) % 64) * kMaxWorld) * 8];
            if (!a[0] || !a[4] || !b[0] || b[0] < a[4] || b[0] - a[4] > 1000000) continue;
            if (a[5] == ~0ull || a[6] < a[5] || a[5] < a[1]) continue;
            acc[0] += a[1] - a[0];
            acc[1] += a[5] - a[1];
            acc[2] += a[6] - a[5];
            acc[3] += a[3] - a[6];
            acc[4] += a[4] - a[3];
            acc[5] += b[0] - a[4];
            ++cnt;
        }
    }
    const double t = worst / ITERS * 1e-3;
    const int sg = sizeof(TG);
    const double sw = MODE == kSgd ? 4 : (MODE == kSgdMp ? 2 : sg);
    const double bytes = WORLD == 1 ? (MODE == kMean ? 2.0 * sg * L
                                                     : (sg + 16.0 + (MODE == kSgdMp ? 2 : 0)) * L)
                                    : (WORLD - 1.0) / WORLD * L * (sg + sw);
    auto ph = [&](int k) { return cnt ? acc[k] / cnt / 1e3 : 0.0; };
    std::printf("{\"world\": %d, \"L\": %zu, \"dtype\": \"%s\", \"mode\": \"%s\", \"kernel\": "
                "\"%s\", \"shape\": \"%s\", \"threads\": %d, \"smem\": %d, \"grid\": %d, "
                "\"us\": %.2f, \"gbs_per_rank\": %.1f, \"phase_us\": {\"entry\": %.2f, "
                "\"data_first_cta\": %.2f, \"cta_spread\": %.2f, \"drain\": %.2f, "
                "\"exit\": %.2f, \"gap_to_next\": %.2f}}\n",
                WORLD, L, sg == 4 ? "f32" : "bf16",
                MODE == kSgd ? "sgd" : (MODE == kSgdMp ? "mp" : "mean"),
                (std::string(kernel) + (SOLO ? "_solo" : "") + (MC_AG ? "_mcag" : "") +
                 (MC_BAR ? "_mcbar" : "")).c_str(),
                shape.c_str(), threads, smem, gx, t * 1e6, bytes / t / 1e9, ph(0), ph(1), ph(2),
                ph(3), ph(4), ph(5));
    std::fflush(stdout);
    for (int d = 0; d < WORLD; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaStreamDestroy(st[d]));
    }
}

static int sm_count() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    return sms;
}

template <typename TG, int WORLD, int MODE, int U, int THREADS, int MINB>
void lsu(int cap = 0) {
    auto fn = gdraa_kernel<TG, WORLD, MODE, U, THREADS, MINB>;
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, THREADS, 0));
    const uint64_t c = (L + WORLD - 1) / WORLD;
    const uint64_t nvec = ((c + kQuantum - 1) / kQuantum * kQuantum + 3) / 4;
    uint64_t gx = std::min<uint64_t>((nvec + THREADS * U - 1) / (THREADS * U),
                                     (uint64_t)sm_count() * per);
    if (cap > 0) gx = std::min<uint64_t>(gx, cap);
    char shape[64];
    std::snprintf(shape, sizeof shape, "U%d_T%d_minb%d_per%d", U, THREADS, MINB, per);
    run<TG, WORLD, MODE>(fn, THREADS, 0, (int)std::max<uint64_t>(gx, 1), "lsu", shape);
}

template <typename TG, int WORLD, int MODE, int CW, int ST, int TD = 4, int TDEP = ST, int ROT = 0,
          int VE = 0, int SKB = 40>
void tma(int cap = 0) {
    using C = TmaCfg<TG, WORLD, MODE, CW, ST, TD, TDEP, ROT, SKB>;
    auto fn = gdraa_tma_kernel<TG, WORLD, MODE, CW, ST, TD, TDEP, ROT, VE, SKB>;
    CK(cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                            cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, C::THREADS, C::SMEM));
    const uint64_t c = (L + WORLD - 1) / WORLD;
    const uint64_t blk = (c + kQuantum - 1) / kQuantum * kQuantum;
    uint64_t gx = std::min<uint64_t>(((blk & ~7ull) + C::CH - 1) / C::CH,
                                     (uint64_t)sm_count() * per);
    if (cap > 0) gx = std::min<uint64_t>(gx, cap);
    char shape[64];
    std::snprintf(shape, sizeof shape, "CW%d_ST%d_CH%d_TD%d_TDEP%d_ROT%d_VE%d_SKB%d_per%d", CW,
                  ST, C::CH, TD, C::TDEPTH, ROT, VE, SKB, per);
    run<TG, WORLD, MODE>(fn, C::THREADS, C::SMEM, (int)std::max<uint64_t>(gx, 1), "tma", shape);
}

template <typename TG, int WORLD, int MODE>
void sweep() {
    using S = Shape<TG, WORLD, MODE>;
    if (WHAT == "lib") {
        lsu<TG, WORLD, MODE, S::U, S::THREADS, S::MINB>();
        tma<TG, WORLD, MODE, 16, 4>();
    } else if (WHAT == "lsu") {
        lsu<TG, WORLD, MODE, 1, 512, 2>();
        lsu<TG, WORLD, MODE, 1, 512, 3>();
        lsu<TG, WORLD, MODE, 1, 512, 4>();
        lsu<TG, WORLD, MODE, 2, 512, 2>();
        lsu<TG, WORLD, MODE, 2, 1024, 1>();
        lsu<TG, WORLD, MODE, 4, 512, 1>();
        lsu<TG, WORLD, MODE, 1, 1024, 1>();
        lsu<TG, WORLD, MODE, 4, 256, 1>();
    } else if (WHAT == "tma") {
        tma<TG, WORLD, MODE, 4, 4>();
        tma<TG, WORLD, MODE, 8, 2>();
        tma<TG, WORLD, MODE, 8, 3>();
        tma<TG, WORLD, MODE, 8, 4>();
        tma<TG, WORLD, MODE, 8, 5>();
        tma<TG, WORLD, MODE, 16, 4>();
    } else if (WHAT == "tail") {
        // end-game variants of the library's TMA shape (16 consumer warps, 4 stages)
        for (int rep = 0; rep < 2; ++rep) {
            tma<TG, WORLD, MODE, 16, 4, 4, 4>();
            tma<TG, WORLD, MODE, 16, 4, 8, 4>();
            tma<TG, WORLD, MODE, 16, 4, 16, 4>();
            tma<TG, WORLD, MODE, 16, 4, 4, 2>();
            tma<TG, WORLD, MODE, 16, 4, 8, 2>();
            tma<TG, WORLD, MODE, 16, 4, 16, 2>();
            tma<TG, WORLD, MODE, 16, 4, 8, 1>();
            tma<TG, WORLD, MODE, 16, 4, 4, 4, 1>();
            tma<TG, WORLD, MODE, 16, 4, 8, 2, 1>();
        }
    } else if (WHAT == "ve") {
        // bf16 broadcasts: 4 vs 8 elements per consumer thread and step (8-byte vs 16-byte
        // stores per destination), twice, interleaved
        if constexpr (MODE == kSgdMp || (MODE == kMean && !std::is_same<TG, float>::value))
            for (int rep = 0; rep < 2; ++rep) {
                tma<TG, WORLD, MODE, 16, 4, 4, 4, 0, 4>();
                tma<TG, WORLD, MODE, 16, 4, 4, 4, 0, 8>();
            }
    } else if (WHAT == "stage") {
        // chunk size (stage bytes) x ring depth, twice interleaved; the library: 40 KB x 4
        for (int rep = 0; rep < 2; ++rep) {
            tma<TG, WORLD, MODE, 16, 4, 4, 4, 0, 0, 40>();
            tma<TG, WORLD, MODE, 16, 5, 4, 5, 0, 0, 40>();
            tma<TG, WORLD, MODE, 16, 3, 4, 3, 0, 0, 64>();
            tma<TG, WORLD, MODE, 16, 2, 4, 2, 0, 0, 100>();
            tma<TG, WORLD, MODE, 16, 6, 4, 6, 0, 0, 28>();
        }
    } else if (WHAT == "mc") {
        // the library's TMA shape: unicast, multicast all-gather, multicast barriers, both;
        // twice, interleaved
        for (int rep = 0; rep < 2; ++rep)
            for (int v = 0; v < 4; ++v) {
                MC_AG = (v & 1) != 0;
                MC_BAR = (v & 2) != 0;
                tma<TG, WORLD, MODE, 16, 4>();
            }
        MC_AG = MC_BAR = false;
    } else if (WHAT == "ctas") {
        for (int cap : {16, 32, 64, 0}) {
            lsu<TG, WORLD, MODE, S::U, S::THREADS, S::MINB>(cap);
            tma<TG, WORLD, MODE, 8, 4>(cap);
            tma<TG, WORLD, MODE, 16, 4>(cap);
        }
    }
}

template <typename TG, int MODE>
void dispatch_world() {
    switch (W) {
        case 1: sweep<TG, 1, MODE>(); break;
        case 2: sweep<TG, 2, MODE>(); break;
        case 4: sweep<TG, 4, MODE>(); break;
        default: std::fprintf(stderr, "world must be 1, 2 or 4\n"); std::exit(1);
    }
}

// One multicast object over W devices; each device binds `bytes` of its own VMM memory
// (readable / writable by every device, so unicast peer stores keep working) and maps
// the object.  Returns per device the local and the multicast VA.
static void make_multicast(size_t bytes, std::vector<void *> &local, std::vector<void *> &mcva) {
    CUmulticastObjectProp prop = {};
    prop.numDevices = W;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    prop.size = bytes;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t sz = (bytes + gran - 1) / gran * gran;
    prop.size = sz;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &prop));
    for (int d = 0; d < W; ++d) {
        CUdevice dev;
        CU(cuDeviceGet(&dev, d));
        CU(cuMulticastAddDevice(mc, dev));
    }
    std::vector<CUmemAccessDesc> acc(W);
    for (int q = 0; q < W; ++q) {
        acc[q] = {};
        acc[q].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc[q].location.id = q;
        acc[q].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    local.resize(W);
    mcva.resize(W);
    for (int d = 0; d < W; ++d) {
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
        CU(cuMemSetAccess(va, sz, acc.data(), W));
        CU(cuMemAddressReserve(&mva, sz, 0, 0, 0));
        CU(cuMemMap(mva, sz, 0, mc, 0));
        CU(cuMemSetAccess(mva, sz, &acc[d], 1));
        CK(cudaMemset(reinterpret_cast<void *>(va), 0, sz));
        CK(cudaDeviceSynchronize());
        local[d] = reinterpret_cast<void *>(va);
        mcva[d] = reinterpret_cast<void *>(mva);
    }
}

static void setup_multicast() {
    const bool mp = MODE_ == kSgdMp;
    const size_t bytes = L * (MODE_ == kSgd ? 4 : (mp ? 2 : (DT == GDRAA_BF16 ? 2 : 4)));
    for (int s = 0; s < 3; ++s) {
        std::vector<void *> local, mcva;
        make_multicast(bytes, local, mcva);
        for (int d = 0; d < W; ++d) {
            if (MODE_ == kSgd) B[d].w[s] = static_cast<float *>(local[d]);
            else if (mp) B[d].model[s] = local[d];
            else B[d].g[s] = local[d];
            B[d].mc_dst[s] = mcva[d];
        }
    }
    std::vector<void *> local, mcva;
    make_multicast(64, local, mcva);
    for (int d = 0; d < W; ++d) {
        B[d].bar_local = static_cast<uint64_t *>(local[d]);
        B[d].mc_bar = static_cast<uint64_t *>(mcva[d]);
    }
}

int main(int argc, char **argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: tune <world> <L> <f32|bf16> <sgd|mp|mean> [iters] [lib|lsu|tma|tail|ctas|solo|mc|ve|stage]\n");
        return 1;
    }
    W = std::atoi(argv[1]);
    L = std::strtoull(argv[2], nullptr, 10);
    DT = std::string(argv[3]) == "bf16" ? GDRAA_BF16 : GDRAA_F32;
    MODE_ = std::string(argv[4]) == "mean" ? kMean : (std::string(argv[4]) == "mp" ? kSgdMp : kSgd);
    if (const char *f = std::getenv("GDRAA_EXIT_FENCE"))
        FLAGS = std::strcmp(f, "thread") == 0 ? 0u : kFlagCtaFence;
    if (const char *f = std::getenv("GDRAA_DIST_EXIT"))
        if (f[0] == '1') FLAGS |= kFlagDistExit;
    if (argc > 5) ITERS = std::atoi(argv[5]);
    if (argc > 6) WHAT = argv[6];
    if (WHAT == "solo") {
        SOLO = true;
        WHAT = "lib";
    }
    MC = WHAT == "mc";
    if (MC) CU(cuInit(0));
    CK(cudaGetDeviceCount(&NDEV));
    if (NDEV < W) {
        std::fprintf(stderr, "need %d GPUs, have %d\n", W, NDEV);
        return 1;
    }
    const size_t gb = L * (DT == GDRAA_BF16 ? 2 : 4);
    B.resize(W);
    for (int d = 0; d < W; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < W; ++q)
            if (q != d) CK(cudaDeviceEnablePeerAccess(q, 0));
        for (int s = 0; s < 3; ++s) {
            CK(cudaMalloc(&B[d].g[s], gb));
            CK(cudaMalloc(&B[d].w[s], L * 4));
            CK(cudaMalloc(&B[d].v[s], L * 4));
            CK(cudaMalloc(&B[d].model[s], L * 2));
            CK(cudaMemset(B[d].model[s], 0, L * 2));
            CK(cudaMemset(B[d].g[s], 0, gb));
            CK(cudaMemset(B[d].w[s], 0, L * 4));
            CK(cudaMemset(B[d].v[s], 0, L * 4));
        }
        CK(cudaMalloc(&B[d].pad, sizeof(Pad)));
        CK(cudaMemset(B[d].pad, 0, sizeof(Pad)));
        if (SOLO && d == 0) {   // every peer "has arrived" at every epoch
            Pad h;
            std::memset(&h, 0, sizeof h);
            for (int q = 0; q < kMaxWorld; ++q)
                h.entry[q] = h.exit[q] = h.recv_done[q] = 1ull << 60;
            CK(cudaMemcpy(B[d].pad, &h, sizeof h, cudaMemcpyHostToDevice));
        }
        uint64_t *tr;
        CK(cudaMalloc(&tr, 64 * kMaxWorld * 8 * 8));
        CK(cudaMemset(tr, 0, 64 * kMaxWorld * 8 * 8));
        TR.push_back(tr);
    }
    if (MC) setup_multicast();
    void *eh;
    CK(cudaHostAlloc(&eh, sizeof(ErrBlock), cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(eh, 0, sizeof(ErrBlock));
    err_d = (ErrBlock *)eh;   // UVA: the host pointer is valid on the device
    if (DT == GDRAA_F32) {
        if (MODE_ == kSgd) dispatch_world<float, kSgd>();
        else if (MODE_ == kSgdMp) dispatch_world<float, kSgdMp>();
        else dispatch_world<float, kMean>();
    } else {
        if (MODE_ == kSgd) dispatch_world<__nv_bfloat16, kSgd>();
        else if (MODE_ == kSgdMp) dispatch_world<__nv_bfloat16, kSgdMp>();
        else dispatch_world<__nv_bfloat16, kMean>();
    }
    return 0;
}
