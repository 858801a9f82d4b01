// ll128_probe.cu -- does a 128-byte line written by 8 lanes of one warp store instruction
// arrive over NVLink as a unit, so that a flag in the line's last 8 bytes implies the other
// 120 bytes are there too?  That is the premise of an "LL128" small-message protocol
// (15/16 payload per line instead of the LL path's 1/2, DESIGN.md §6 latency path), which
// the library serves only experimentally (GDRAA_LL128, off by default); this probe
// measures the premise the experimental kernels rest on.
//
// Two devices, one process.  The sender (GPU 0) writes, for epochs e = 1..E, a buffer of
// LINES 128-byte lines into GPU 1's memory: lane j of each 8-lane group stores 16 bytes
// (st.volatile.global.v2.u64), words 0..14 = tag(e, line, word), word 15 = flag e.
// The receiver (GPU 1) polls every line until its flag reads e (ld.volatile.v2.u64, the
// flag lane's result shuffled to the group), then checks the 15 payload words of the same
// read against tag(e, ...).  A flag seen with any stale payload word is a torn line.
// Sender and receiver run concurrently; the receiver acknowledges epoch e back to the
// sender before e + 1 is written (so lines are only ever overwritten by the next epoch).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ll128_probe \
//        tools/ll128_probe.cu
//   tools/ll128_probe [lines_per_epoch=262144] [epochs=200] [control=0] [same=0]
// same = 1: sender and receiver on GPU 0 (half the SMs each), the buffer in GPU 0's own
// memory -- the virtual-rank case, where no NVLink is involved.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            std::printf("{\"error\": \"%s:%d %s\"}\n", __FILE__, __LINE__,               \
                        cudaGetErrorString(e_));                                         \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)

__device__ __forceinline__ uint64_t tag(uint64_t e, uint64_t line, int w) {
    return (e << 40) ^ (line << 4) ^ static_cast<uint64_t>(w) ^ 0x5bd1e995ull;
}

__device__ __forceinline__ void st_v2(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b)
                 : "memory");
}
__device__ __forceinline__ void ld_v2(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p)
                 : "memory");
}
__device__ __forceinline__ uint64_t ld_acq(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
constexpr uint64_t kGiveUpNs = 10ull * 1000 * 1000 * 1000;   // every spin gives up after 10 s

__device__ __forceinline__ void st_rel(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Persistent sender: every thread owns 16 bytes of a line per step; a grid-wide epoch
// loop waits for the receiver's ack of e - 1 (one poller per CTA) before writing epoch e.
// control = 1 (negative control, validates the detector): the flag lane stores its flag
// word first, in its own instruction, and the line's payload afterwards -- a reader can
// then see the new flag with old payload, and torn_lines must come out > 0.
__global__ void sender(uint64_t *remote, uint64_t lines, int epochs, const uint64_t *ack,
                       unsigned *gave_up, int control) {
    const uint64_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthr = gridDim.x * blockDim.x;
    const int j = threadIdx.x & 7;   // lane within the 8-lane line group
    for (uint64_t e = 1; e <= static_cast<uint64_t>(epochs); ++e) {
        if (threadIdx.x == 0) {
            const uint64_t t0 = gtimer();
            while (ld_acq(ack) < e - 1)
                if (gtimer() - t0 > kGiveUpNs) {
                    atomicExch(gave_up, 1u);
                    break;
                }
        }
        __syncthreads();
        if (*reinterpret_cast<volatile unsigned *>(gave_up)) return;
        for (uint64_t t = tid; t < lines * 8; t += nthr) {
            const uint64_t line = t >> 3;
            const uint64_t a = tag(e, line, 2 * j);
            const uint64_t b = j == 7 ? e : tag(e, line, 2 * j + 1);
            if (control) {
                if (j == 7) {
                    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(remote + line * 16 + 15),
                                 "l"(e)
                                 : "memory");
                    __nanosleep(200);
                }
                __syncwarp();
                if (j == 7)
                    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(remote + line * 16 + 14),
                                 "l"(a)
                                 : "memory");
                else
                    st_v2(remote + line * 16 + 2 * j, a, b);
            } else {
                st_v2(remote + line * 16 + 2 * j, a, b);
            }
        }
    }
}

// Receiver: polls its lines for epoch e, checks the payload of the read that showed the
// flag, counts torn lines; then acknowledges e to the sender (release, after a grid
// barrier made of an atomic counter).
__global__ void receiver(const uint64_t *buf, uint64_t lines, int epochs, uint64_t *ack_remote,
                         unsigned *arrive, unsigned long long *torn,
                         unsigned long long *polls, unsigned *gave_up) {
    const uint64_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthr = gridDim.x * blockDim.x;
    const int j = threadIdx.x & 7;
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);   // this lane's 8-lane group
    unsigned long long my_torn = 0, my_polls = 0;
    for (uint64_t e = 1; e <= static_cast<uint64_t>(epochs); ++e) {
        // every warp iterates the same trip count (lines * 8 is a multiple of 32)
        for (uint64_t t = tid; t < lines * 8; t += nthr) {
            const uint64_t line = t >> 3;
            uint64_t a, b;
            bool done = false;
            const uint64_t t0 = gtimer();
            while (!done) {
                ld_v2(buf + line * 16 + 2 * j, a, b);
                ++my_polls;
                const uint64_t flag = __shfl_sync(gmask, b, 7, 8);
                done = flag == e;   // the same decision in all 8 lanes of the group
                const bool late = __shfl_sync(gmask, gtimer() - t0 > kGiveUpNs, 0, 8);
                if (late) {
                    atomicExch(gave_up, 1u);
                    break;
                }
            }
            if (!done) break;
            bool ok = a == tag(e, line, 2 * j) && (j == 7 || b == tag(e, line, 2 * j + 1));
            const unsigned bad = __ballot_sync(gmask, !ok) & gmask;
            if (bad && j == 7) ++my_torn;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned prev = atomicAdd(arrive, 1u);
            if (prev == gridDim.x * e - 1) st_rel(ack_remote, e);   // last CTA of epoch e
            const uint64_t t0 = gtimer();
            while (*reinterpret_cast<volatile unsigned *>(arrive) < gridDim.x * e)
                if (gtimer() - t0 > kGiveUpNs) {
                    atomicExch(gave_up, 1u);
                    break;
                }
        }
        __syncthreads();
        if (*reinterpret_cast<volatile unsigned *>(gave_up)) break;
    }
    atomicAdd(torn, my_torn);
    atomicAdd(polls, my_polls);
}

int main(int argc, char **argv) {
    const uint64_t lines = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 262144;
    const int epochs = argc > 2 ? std::atoi(argv[2]) : 200;
    const int control = argc > 3 ? std::atoi(argv[3]) : 0;
    const int same = argc > 4 ? std::atoi(argv[4]) : 0;
    const int dr = same ? 0 : 1;   // the receiver's (and the buffer's) device
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2 && !same) {
        std::printf("{\"error\": \"needs 2 GPUs\"}\n");
        return 1;
    }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = same ? sms / 2 : sms;
    uint64_t *buf = nullptr, *ack = nullptr;
    unsigned *arrive = nullptr, *gave_up_s = nullptr, *gave_up_r = nullptr;
    unsigned long long *torn = nullptr, *polls = nullptr;
    CK(cudaSetDevice(dr));
    if (!same) CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaMalloc(&buf, lines * 128));
    CK(cudaMemset(buf, 0, lines * 128));
    CK(cudaMalloc(&arrive, 2 * sizeof(unsigned)));
    CK(cudaMemset(arrive, 0, 2 * sizeof(unsigned)));
    gave_up_r = arrive + 1;
    CK(cudaMalloc(&torn, 2 * sizeof(unsigned long long)));
    CK(cudaMemset(torn, 0, 2 * sizeof(unsigned long long)));
    polls = torn + 1;
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(0));
    if (!same) CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaMalloc(&ack, 2 * sizeof(uint64_t)));
    CK(cudaMemset(ack, 0, 2 * sizeof(uint64_t)));
    gave_up_s = reinterpret_cast<unsigned *>(ack + 1);
    CK(cudaDeviceSynchronize());

    // load both kernels now: under lazy module loading the first launch of a kernel waits
    // for the device to idle, which on one device deadlocks the second grid behind the first
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, sender));
    CK(cudaFuncGetAttributes(&fa, receiver));
    // both grids must be fully resident (they wait on each other): one CTA per SM
    cudaEvent_t t0, t1;
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    cudaStream_t rs;   // same device: the two grids need separate streams to run together
    CK(cudaSetDevice(dr));
    CK(cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking));
    receiver<<<grid, 256, 0, rs>>>(buf, lines, epochs, ack, arrive, torn, polls, gave_up_r);
    CK(cudaGetLastError());
    CK(cudaSetDevice(0));
    cudaStream_t ss;
    CK(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
    CK(cudaEventRecord(t0, ss));
    sender<<<grid, 256, 0, ss>>>(buf, lines, epochs, ack, gave_up_s, control);
    CK(cudaGetLastError());
    CK(cudaEventRecord(t1, ss));
    CK(cudaDeviceSynchronize());
    CK(cudaSetDevice(dr));
    CK(cudaDeviceSynchronize());
    unsigned long long h[2];
    CK(cudaMemcpy(h, torn, sizeof h, cudaMemcpyDeviceToHost));
    unsigned gu[2] = {0, 0};
    CK(cudaMemcpy(&gu[1], gave_up_r, sizeof(unsigned), cudaMemcpyDeviceToHost));
    CK(cudaSetDevice(0));
    CK(cudaMemcpy(&gu[0], gave_up_s, sizeof(unsigned), cudaMemcpyDeviceToHost));
    uint64_t acked = 0;
    CK(cudaMemcpy(&acked, ack, sizeof acked, cudaMemcpyDeviceToHost));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, t0, t1));
    const double bytes = static_cast<double>(lines) * 128 * epochs;
    std::printf("{\"probe\": \"ll128_line_atomicity\", \"same_device\": %d, \"control\": %d, \"lines_per_epoch\": %llu, \"epochs\": %d, "
                "\"lines_checked\": %.0f, \"torn_lines\": %llu, \"polls\": %llu, "
                "\"sender_ms\": %.3f, \"gbs_one_way_incl_acks\": %.1f, \"gave_up\": [%u, %u], \"acked_epochs\": %llu}\n",
                same, control, static_cast<unsigned long long>(lines), epochs,
                static_cast<double>(lines) * epochs, h[0], h[1], ms, bytes / (ms * 1e-3) / 1e9, gu[0],
                gu[1], static_cast<unsigned long long>(acked));
    return 0;
}
