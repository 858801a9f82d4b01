// jobserver_proto.h -- control-plane protocol between gdraa ranks and the job server.
//
// The job server is the paper's MiMatrix central node: it "only
// receives and sends messages" and "undertakes ... controlling, scheduling and
// monitoring ... without weight data transfer".  Here it carries exactly:
//   HELLO / HELLO_OK   rank joins; gets the name of the shared go/done page   (S:95 WorkerReady)
//   REG / REG_OK|ERR   64-byte CUDA IPC handles + offsets, shape check      (P:123 ibv_reg_mr)
//   BYE / BYE_OK       collective shutdown                                  (S:95 Shutdown)
// and a POSIX shared-memory page with per-rank go/done counters (S:95 IterStart /
// IterDone) that the kernels' last CTA writes through a host mapping.  No message type
// carries tensor data; `data_bytes` in the page counts the payload of any message outside
// this vocabulary (its sender is dropped), so it reads 0 unless something tried.
// Plain C structs; both sides are the same binary architecture (one node).
#pragma once

#include <cstdint>

namespace gdraa {
namespace proto {

constexpr uint32_t kMagic = 0x41524447u;   // "GDRA"
constexpr int kMaxRanks = 8;

enum Kind : uint16_t {
    HELLO = 1,
    HELLO_OK = 2,
    REG = 3,
    REG_OK = 4,
    REG_ERR = 5,
    BYE = 6,
    BYE_OK = 7,
    FAIL = 8,
};

struct Hdr {
    uint32_t magic;
    uint16_t kind;
    uint16_t rank;
    uint32_t len;     // payload bytes following the header
    uint32_t seq;     // registration sequence number (REG*), 0 otherwise
};

struct Hello {
    int32_t world;
    int32_t pid;
    uint8_t uuid[16];   // CUDA device UUID of the rank's GPU (informational)
};

struct HelloOk {
    char shm_name[64];
    int32_t world;
    int32_t gated;
    uint64_t job_id;
};

// One rank's registration record.  `handle` is a cudaIpcMemHandle_t (opaque bytes to
// the job server, which never opens it).
struct Reg {
    uint64_t n;        // elements (or bytes for the signal pad)
    int32_t dtype;     // gdraa_dtype_t, or -1 for the signal pad
    int32_t what;      // 0 = signal pad, 1 = data buffer
    uint64_t offset;   // byte offset of the registered pointer in its allocation
    uint8_t handle[64];
};

struct RegOk {
    int32_t world;
    int32_t _pad;
    Reg regs[kMaxRanks];
};

struct Fail {
    int32_t code;      // gdraa_err_t
    char msg[188];
};

// Shared go/done page (one per job).  Ranks map it with cudaHostRegister so the kernel
// can write done[] directly; the job server polls it.
struct alignas(64) ShmPage {
    uint64_t magic;
    int32_t world;
    int32_t gated;
    volatile uint64_t go[kMaxRanks];        // rank r may launch call e once go[r] >= e
    volatile uint64_t done[kMaxRanks];      // written by rank r's kernel: calls completed
    volatile int32_t abort;                 // set by the job server if a rank vanished
    volatile int32_t dead_rank;
    volatile uint64_t control_bytes;        // bytes of control messages handled
    volatile uint64_t data_bytes;           // payload bytes of non-control messages (dropped)
    volatile uint64_t registrations;
};

}  // namespace proto
}  // namespace gdraa
