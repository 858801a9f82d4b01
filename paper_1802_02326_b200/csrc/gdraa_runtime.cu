// gdraa_runtime.cu -- host runtime behind include/gdraa.h.
//
// Owns: the job-server connection (control plane), CUDA IPC registration of the
// caller's buffers (the analogue of P:123's ibv_reg_mr), the signal pads that carry the
// two synchronisations, the host-mapped go/done and failure pages, sticky errors and
// counters.  Each collective call validates on the host, then enqueues exactly one
// kernel (gdraa_kernels.cu) on the caller's stream: no host synchronisation.
#include <cuda.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "gdraa_internal.h"
#include "jobserver_proto.h"

namespace gdraa {
namespace {

thread_local std::string t_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            return fail(GDRAA_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));    \
    } while (0)

uint64_t now_ns() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return static_cast<uint64_t>(ts.tv_sec) * 1000000000ull + ts.tv_nsec;
}

uint64_t env_u64(const char *name, uint64_t dflt) {
    const char *v = std::getenv(name);
    if (v == nullptr || *v == 0) return dflt;
    return std::strtoull(v, nullptr, 10);
}

size_t elem_size(int dtype) { return dtype == GDRAA_F32 ? 4 : 2; }

// Q-aligned ceil partition (AMB-8).
void partition(uint64_t n, int world, int rank, uint64_t *blk, uint64_t *off, uint64_t *len) {
    const uint64_t c = (n + world - 1) / world;
    const uint64_t b = (c + kQuantum - 1) / kQuantum * kQuantum;
    uint64_t o = static_cast<uint64_t>(rank) * b;
    if (o > n) o = n;
    *blk = b;
    *off = o;
    *len = b < n - o ? b : n - o;
}

// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda needed).
using GetRangeFn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
GetRangeFn get_range_fn() {
    static GetRangeFn fn = nullptr;
    if (fn == nullptr) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<GetRangeFn>(p);
    }
    return fn;
}

// ---------------------------------------------------------------------------------
// Job-server client
// ---------------------------------------------------------------------------------
bool io_all(int fd, void *buf, size_t n, bool rd, uint64_t deadline_ns) {
    char *p = static_cast<char *>(buf);
    while (n > 0) {
        if (rd) {
            timeval tv{};
            uint64_t left = deadline_ns > now_ns() ? deadline_ns - now_ns() : 0;
            if (left == 0) return false;
            tv.tv_sec = left / 1000000000ull;
            tv.tv_usec = (left % 1000000000ull) / 1000;
            setsockopt(fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
        }
        ssize_t k = rd ? ::recv(fd, p, n, 0) : ::send(fd, p, n, MSG_NOSIGNAL);
        if (k == 0) return false;
        if (k < 0) {
            if (errno == EINTR) continue;
            return false;
        }
        p += k;
        n -= static_cast<size_t>(k);
    }
    return true;
}

// ---------------------------------------------------------------------------------
// State
// ---------------------------------------------------------------------------------
struct Registration {
    void *local = nullptr;
    size_t n = 0;
    int dtype = 0;
    void *peer[kMaxWorld] = {};
};

// Calls share their pad (epoch, arrival and work counters) and LL slots, so a call issued
// on another stream than the previous one first waits for everything issued so far on the
// previous call's stream (an event recorded there at that moment; calls on one stream pay
// nothing, and programmatic dependent launch between them is kept).  Not while either
// stream is capturing: a graph's own edges order the calls captured into it.
struct StreamOrder {
    cudaStream_t last = nullptr;
    cudaEvent_t ev = nullptr;
    bool have = false;
};

// A bucket set (gdraa_bucket_set_begin / _end): the calls inside it skip their exit
// barrier, so their results are complete only at _end; they must therefore write disjoint
// destination ranges.  spans = the [lo, hi) byte ranges written so far in the open set.
// A streamed set (gdraa_bucket_set_begin_streamed) is served by one persistent kernel on
// the library's own stream, launched at the set's first call; every call then only
// describes its bucket with stream memory operations on the caller's stream (SetDesc).
struct Streamed {
    bool on = false;                 // the open set is streamed
    bool launched = false;           // its kernel has been launched (at the first call)
    int ctas = 0;                    // CTAs per rank of that kernel
    uint32_t gen = 0;                // set generation (tags in SetDesc)
    uint32_t nb = 0;                 // buckets described so far
    int mode = -1, dtype = -1;       // what the kernel was launched for
    const void *key[4] = {};         // base pointers it was launched with: g, dst, v, wm
    float lr = 0.f, mom = 0.f, wd = 0.f;
    cudaStream_t last = nullptr;     // stream of the last described bucket
    SetDesc *desc = nullptr;         // device memory
    uint32_t *next = nullptr;        // device memory, kSetMax chunk counters per (v)rank
    cudaStream_t ps = nullptr;       // the kernel's stream (non-blocking)
    cudaEvent_t done = nullptr;      // recorded on ps after the kernel
    cudaEvent_t start = nullptr;     // the first call's stream, when it reaches that call
};

struct BucketSet {
    bool open = false;
    std::vector<std::pair<uintptr_t, uintptr_t>> spans;
    Streamed st;
};

// cuStreamWriteValue64 through the runtime's driver entry point (no -lcuda needed).
using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WriteValue64Fn write_value64_fn() {
    static WriteValue64Fn fn = nullptr;
    if (fn == nullptr) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WriteValue64Fn>(p);
    }
    return fn;
}

int write_value(cudaStream_t s, const uint64_t *addr, uint64_t v) {
    WriteValue64Fn wv = write_value64_fn();
    if (wv == nullptr) return fail(GDRAA_ECUDA, "cuStreamWriteValue64 unavailable");
    if (wv(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v, 0) != CUDA_SUCCESS)
        return fail(GDRAA_ECUDA, "cuStreamWriteValue64 failed");
    return GDRAA_OK;
}

// Open a streamed set: device state allocated on first use (rows = virtual ranks).
int streamed_open(Streamed &st, int rows, int ctas) {
    if (st.desc == nullptr) {
        void *d = nullptr, *n = nullptr;
        CUDA_TRY(cudaMalloc(&d, sizeof(SetDesc)));
        CUDA_TRY(cudaMemset(d, 0, sizeof(SetDesc)));
        CUDA_TRY(cudaMalloc(&n, sizeof(uint32_t) * kSetMax * rows));
        CUDA_TRY(cudaMemset(n, 0, sizeof(uint32_t) * kSetMax * rows));
        CUDA_TRY(cudaStreamCreateWithFlags(&st.ps, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&st.start, cudaEventDisableTiming));
        CUDA_TRY(cudaDeviceSynchronize());
        st.desc = static_cast<SetDesc *>(d);
        st.next = static_cast<uint32_t *>(n);
    }
    st.on = true;
    st.launched = false;
    st.ctas = ctas;
    st.gen += 1;
    st.nb = 0;
    st.last = nullptr;
    return GDRAA_OK;
}

void streamed_free(Streamed &st) {
    if (st.desc) cudaFree(st.desc);
    if (st.next) cudaFree(st.next);
    if (st.ps) cudaStreamDestroy(st.ps);
    if (st.done) cudaEventDestroy(st.done);
    if (st.start) cudaEventDestroy(st.start);
    st = Streamed{};
}

int set_check(const BucketSet &b, const void *dst, size_t bytes) {
    if (!b.open) return GDRAA_OK;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(dst), hi = lo + bytes;
    for (const auto &sp : b.spans)
        if (lo < sp.second && sp.first < hi)
            return fail(GDRAA_EINVAL, "bucket set: destination range %p + %zu bytes overlaps "
                        "a range written earlier in the set (results are complete only at "
                        "gdraa_bucket_set_end)", dst, bytes);
    return GDRAA_OK;
}

void set_note(BucketSet &b, const void *dst, size_t bytes) {
    if (!b.open) return;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(dst);
    b.spans.emplace_back(lo, lo + bytes);
}

struct State {
    bool inited = false;
    int world = 0, rank = 0, device = 0;
    int sock = -1;
    proto::ShmPage *page = nullptr;     // shared go/done page (host)
    bool page_registered = false;
    bool page_owned = false;            // world == 1 without a job server: our own page
    Pad *pad = nullptr;
    Pad *peer_pad[kMaxWorld] = {};
    uint4 *ll = nullptr;                // small-message receive slots (world > 1)
    uint4 *peer_ll[kMaxWorld] = {};
    uint64_t ll_pairs = 0;
    uint64_t ll_sgd_limit = 0;          // small-message SGD threshold (bytes), fixed at init
    ErrBlock *err_h = nullptr, *err_d = nullptr;
    volatile uint64_t *done_d = nullptr;
    const volatile int32_t *abort_d = nullptr;   // device alias of the page's abort flag
    std::vector<Registration> regs;
    std::map<std::pair<int, std::string>, void *> opened;   // (peer, handle) -> base
    uint32_t reg_seq = 0;
    uint64_t timeout_ns = 30000000000ull;
    bool gated = false;
    uint64_t issued = 0;
    // Cross-stream ordering (see StreamOrder): every call shares this rank's pad and LL slots.
    StreamOrder order;
    BucketSet set;                      // open bucket set (deferred exit barriers)
    bool fatal = false;
    int fatal_code = 0;
    std::string fatal_msg;
    gdraa_stats_t host{};
};

State g;
std::mutex g_mu;

int send_msg(uint16_t kind, uint32_t seq, const void *payload, uint32_t len) {
    proto::Hdr h{proto::kMagic, kind, static_cast<uint16_t>(g.rank), len, seq};
    const uint64_t dl = now_ns() + 10000000000ull;
    if (!io_all(g.sock, &h, sizeof h, false, dl) ||
        (len && !io_all(g.sock, const_cast<void *>(payload), len, false, dl)))
        return fail(GDRAA_EJOBSERVER, "job server: send failed: %s", std::strerror(errno));
    return GDRAA_OK;
}

// Receive one message; FAIL from the server becomes an error with its message.
int recv_msg(uint16_t want, uint32_t seq, void *payload, uint32_t len, uint64_t timeout_ns,
             uint16_t *got_kind = nullptr) {
    proto::Hdr h;
    const uint64_t dl = now_ns() + timeout_ns;
    if (!io_all(g.sock, &h, sizeof h, true, dl))
        return fail(GDRAA_EJOBSERVER, "job server: no reply (waiting for kind %u): %s", want,
                    errno ? std::strerror(errno) : "closed");
    std::vector<char> body(h.len);
    if (h.len && !io_all(g.sock, body.data(), h.len, true, dl))
        return fail(GDRAA_EJOBSERVER, "job server: truncated reply");
    if (got_kind) *got_kind = h.kind;
    if (h.magic != proto::kMagic) return fail(GDRAA_EJOBSERVER, "job server: bad magic");
    if (h.kind == proto::FAIL || h.kind == proto::REG_ERR) {
        proto::Fail f{};
        std::memcpy(&f, body.data(), std::min(sizeof f, body.size()));
        f.msg[sizeof f.msg - 1] = 0;
        return fail(f.code ? f.code : GDRAA_EJOBSERVER, "job server: %s", f.msg);
    }
    if (h.kind != want || h.seq != seq || h.len != len)
        return fail(GDRAA_EJOBSERVER, "job server: unexpected reply kind %u seq %u len %u",
                    h.kind, h.seq, h.len);
    if (len) std::memcpy(payload, body.data(), len);
    return GDRAA_OK;
}

int connect_jobserver(const char *path, uint64_t timeout_ns) {
    const uint64_t dl = now_ns() + timeout_ns;
    sockaddr_un addr{};
    addr.sun_family = AF_UNIX;
    if (std::strlen(path) >= sizeof addr.sun_path)
        return fail(GDRAA_EINVAL, "GDRAA_JOBSERVER path too long");
    std::snprintf(addr.sun_path, sizeof addr.sun_path, "%s", path);
    while (true) {
        int fd = ::socket(AF_UNIX, SOCK_STREAM, 0);
        if (fd < 0) return fail(GDRAA_EJOBSERVER, "socket: %s", std::strerror(errno));
        if (::connect(fd, reinterpret_cast<sockaddr *>(&addr), sizeof addr) == 0) {
            g.sock = fd;
            return GDRAA_OK;
        }
        ::close(fd);
        if (now_ns() > dl)
            return fail(GDRAA_EJOBSERVER, "cannot connect to job server at %s: %s", path,
                        std::strerror(errno));
        usleep(20000);
    }
}

// Exchange one registration record with every rank through the job server.
int exchange(const proto::Reg &mine, proto::RegOk *all) {
    const uint32_t seq = ++g.reg_seq;
    int rc = send_msg(proto::REG, seq, &mine, sizeof mine);
    if (rc) return rc;
    return recv_msg(proto::REG_OK, seq, all, sizeof *all,
                    env_u64("GDRAA_CONNECT_TIMEOUT_MS", 120000) * 1000000ull);
}

// Export the allocation holding [ptr, ptr+bytes) and map every peer's counterpart.
int ipc_exchange(void *ptr, size_t bytes, uint64_t n, int dtype, int what,
                 void *out_peer[kMaxWorld]) {
    GetRangeFn range = get_range_fn();
    if (range == nullptr) return fail(GDRAA_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return fail(GDRAA_EINVAL, "pointer %p is not device memory of this context", ptr);
    const uint64_t offset = reinterpret_cast<uint64_t>(ptr) - base;
    if (offset + bytes > size)
        return fail(GDRAA_EINVAL, "buffer [%p, +%zu) exceeds its allocation (%zu bytes)", ptr,
                    bytes, size);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess)
        return fail(GDRAA_ECUDA,
                    "cudaIpcGetMemHandle: %s (buffers must come from cudaMalloc; with PyTorch "
                    "keep PYTORCH_CUDA_ALLOC_CONF expandable_segments off)",
                    cudaGetErrorString(e));
    proto::Reg mine{};
    mine.n = n;
    mine.dtype = dtype;
    mine.what = what;
    mine.offset = offset;
    static_assert(sizeof(h) == sizeof(mine.handle), "IPC handle size");
    std::memcpy(mine.handle, &h, sizeof h);
    proto::RegOk all{};
    int rc = exchange(mine, &all);
    if (rc) return rc;
    for (int p = 0; p < g.world; ++p) {
        if (p == g.rank) {
            out_peer[p] = ptr;
            continue;
        }
        std::string key(reinterpret_cast<const char *>(all.regs[p].handle), 64);
        auto it = g.opened.find({p, key});
        void *pbase = nullptr;
        if (it != g.opened.end()) {
            pbase = it->second;
        } else {
            cudaIpcMemHandle_t ph;
            std::memcpy(&ph, all.regs[p].handle, sizeof ph);
            e = cudaIpcOpenMemHandle(&pbase, ph, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess)
                return fail(GDRAA_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", p,
                            cudaGetErrorString(e));
            g.opened[{p, key}] = pbase;
        }
        out_peer[p] = static_cast<char *>(pbase) + all.regs[p].offset;
    }
    return GDRAA_OK;
}

int check_sticky() {
    if (!g.inited) return fail(GDRAA_ESTATE, "gdraa_init has not been called");
    if (g.fatal) return fail(g.fatal_code, "%s", g.fatal_msg.c_str());
    // a rank the job server saw die explains a device-side give-up: report it first
    if (g.page != nullptr && !g.page_owned && g.page->abort) {
        g.fatal = true;
        g.fatal_code = GDRAA_EJOBSERVER;
        g.fatal_msg = "job server reports rank " + std::to_string(g.page->dead_rank) + " died";
        return fail(GDRAA_EJOBSERVER, "%s", g.fatal_msg.c_str());
    }
    if (g.err_h != nullptr && g.err_h->code != 0) {
        std::string miss;
        for (int p = 0; p < kMaxWorld; ++p)
            if (g.err_h->missing[p]) miss += (miss.empty() ? "" : ",") + std::to_string(p);
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "peer timeout in the %s synchronisation after %llu ms: missing rank(s) %s",
                      g.err_h->phase == 1 ? "entry (paper 2nd)" : "exit (paper 1st)",
                      (unsigned long long)(g.timeout_ns / 1000000ull), miss.c_str());
        g.fatal = true;
        g.fatal_code = GDRAA_ETIMEOUT;
        g.fatal_msg = buf;
        return fail(GDRAA_ETIMEOUT, "%s", buf);
    }
    return GDRAA_OK;
}

const Registration *find_reg(const void *ptr) {
    for (const auto &r : g.regs)
        if (r.local == ptr) return &r;
    return nullptr;
}

int wait_go() {
    if (!g.gated || g.page == nullptr) return GDRAA_OK;
    const uint64_t want = g.issued + 1;
    const uint64_t dl = now_ns() + g.timeout_ns;
    while (g.page->go[g.rank] < want) {
        if (g.page->abort) return check_sticky();
        if (now_ns() > dl) return fail(GDRAA_ETIMEOUT, "gated: no go(%llu) from job server",
                                       (unsigned long long)want);
        usleep(5);
    }
    return GDRAA_OK;
}

void fill_common(KParams &p, uint64_t n) {
    std::memset(&p, 0, sizeof p);
    p.world = g.world;
    p.rank0 = g.rank;
    p.n = n;
    uint64_t off, len;
    partition(n, g.world, g.rank, &p.blk, &off, &len);
    p.timeout_ns = g.timeout_ns;
    for (int q = 0; q < g.world; ++q) {
        p.pad[0][q] = g.peer_pad[q];
        p.ll[0][q] = g.peer_ll[q];
    }
    p.ll_pairs = g.ll_pairs;
    p.ll_sleep_ns = static_cast<uint32_t>(env_u64("GDRAA_LL_SLEEP_NS", 256));
    p.flags = env_kernel_flags() | (g.set.open ? kFlagDeferExit : 0u);
    p.err = g.err_d;
    // IterDone: the last CTA's store into the host-mapped page costs nothing measurable
    // (profiles/r69_alpha.json: two-shot sgd sweep with and without it within 0.2 us)
    p.done[0] = g.done_d;
    p.abort = g.abort_d;
}

// Lemma 1/2 accounting of one call (s_w: bytes per broadcast element; 0 = same as g).
void account(uint64_t n, int dtype_g, uint64_t s_w, bool launched = true) {
    uint64_t blk, off, len;
    partition(n, g.world, g.rank, &blk, &off, &len);
    const uint64_t sg = elem_size(dtype_g), sw = s_w ? s_w : sg, n1 = g.world - 1;
    g.host.rs_bytes_in += sg * n1 * len;
    g.host.rs_bytes_out += sg * (n - len);
    g.host.ag_bytes_out += sw * n1 * len;
    g.host.ag_bytes_in += sw * (n - len);
    g.host.adds += n1 * len;
    g.host.divides += len;
    if (launched) g.host.launches += 1;
}

bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}

// Before a launch on s: order it after the previous call if that was on another stream.
int order_after_previous(StreamOrder &o, cudaStream_t s) {
    if (!o.have || s == o.last || capturing(s) || capturing(o.last)) return GDRAA_OK;
    if (o.ev == nullptr) CUDA_TRY(cudaEventCreateWithFlags(&o.ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(o.ev, o.last));
    CUDA_TRY(cudaStreamWaitEvent(s, o.ev, 0));
    return GDRAA_OK;
}

// After a launch on s: remember the stream.
int note_launch(StreamOrder &o, cudaStream_t s) {
    o.last = s;
    o.have = true;
    return GDRAA_OK;
}

// One call of an open streamed set.  p describes the call as for the per-call kernels
// (pointers offset to the range's start); they are rebased to the buffers' starts, which
// the persistent kernel indexes with each bucket's `first`.  The first call launches the
// kernel on the set's own stream (ordered after the previous collective); every call then
// describes its bucket on the caller's stream cs.
int streamed_call(BucketSet &set, StreamOrder &order, KParams p, int rows, bool coop,
                  int dtype, int mode, cudaStream_t cs, uint64_t first, uint64_t count) {
    Streamed &st = set.st;
    if (capturing(cs))
        return fail(GDRAA_EINVAL, "streamed bucket sets cannot be captured into a CUDA graph");
    if (st.nb >= static_cast<uint32_t>(kSetMax) - 1)
        return fail(GDRAA_EINVAL, "streamed bucket set: at most %d buckets", kSetMax - 1);
    const size_t eg = elem_size(dtype), ed = mode == kSgd ? 4 : (mode == kSgdMp ? 2 : eg);
    auto back = [&](const void *ptr, size_t es) -> void * {
        return ptr == nullptr ? nullptr
                              : const_cast<char *>(static_cast<const char *>(ptr)) - first * es;
    };
    for (int r = 0; r < rows; ++r) {
        for (int q = 0; q < p.world; ++q) {
            p.src[r][q] = back(p.src[r][q], eg);
            p.dst[r][q] = back(p.dst[r][q], ed);
        }
        p.v[r] = static_cast<float *>(back(p.v[r], 4));
        p.wm[r] = static_cast<float *>(back(p.wm[r], 4));
    }
    const void *key[4] = {p.src[0][p.rank0], p.dst[0][p.rank0], p.v[0], p.wm[0]};
    if (!st.launched) {
        p.sdesc = st.desc;
        for (int r = 0; r < rows; ++r) p.snext[r] = st.next + static_cast<size_t>(r) * kSetMax;
        p.sgen = st.gen;
        int rc = order_after_previous(order, st.ps);
        if (rc) return rc;
        // the kernel becomes resident (and holds its SMs) only once the first bucket is
        // final, i.e. when the caller's stream reaches this call
        CUDA_TRY(cudaEventRecord(st.start, cs));
        CUDA_TRY(cudaStreamWaitEvent(st.ps, st.start, 0));
        cudaError_t e = launch_gdraa_tma_set(p, dtype, mode, rows, coop, st.ps, st.ctas);
        if (e != cudaSuccess)
            return fail(GDRAA_ECUDA, "bucket-set kernel launch: %s", cudaGetErrorString(e));
        CUDA_TRY(cudaEventRecord(st.done, st.ps));
        note_launch(order, st.ps);
        st.launched = true;
        st.mode = mode;
        st.dtype = dtype;
        std::memcpy(st.key, key, sizeof key);
        st.lr = p.lr;
        st.mom = p.mom;
        st.wd = p.wd;
    } else if (mode != st.mode || dtype != st.dtype || std::memcmp(key, st.key, sizeof key) != 0 ||
               p.lr != st.lr || p.mom != st.mom || p.wd != st.wd) {
        return fail(GDRAA_EINVAL, "streamed bucket set: every call must use the buffers, mode, "
                    "dtype and lr/mom/wd of the set's first call");
    }
    const uint32_t k = st.nb;
    int rc = write_value(cs, &st.desc->first[k], first);
    if (!rc) rc = write_value(cs, &st.desc->count[k], count);
    if (!rc) rc = write_value(cs, &st.desc->ready[k], set_tag(st.gen, k));
    if (rc) return rc;
    st.nb += 1;
    st.last = cs;
    return GDRAA_OK;
}

// Close an open streamed set on s: the close marker, then s waits for the kernel.
int streamed_close(BucketSet &set, StreamOrder &order, cudaStream_t s) {
    Streamed &st = set.st;
    st.on = false;
    if (!st.launched) return GDRAA_OK;
    st.launched = false;
    int rc = write_value(s, &st.desc->ready[st.nb], set_close(st.gen));
    if (rc) return rc;
    CUDA_TRY(cudaStreamWaitEvent(s, st.done, 0));
    return note_launch(order, s);
}

int launch(const KParams &p, int dtype, int mode, cudaStream_t s) {
    int gx = 0;
    cudaError_t e = use_tma_kernel(dtype, mode, p.world)
                        ? launch_gdraa_tma(p, dtype, mode, 1, false, s, &gx)
                                     : launch_gdraa(p, dtype, mode, 1, false, s, &gx);
    if (e != cudaSuccess) return fail(GDRAA_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
    g.issued += 1;
    return GDRAA_OK;
}

// ---------------------------------------------------------------------------------
// Virtual ranks on one GPU: pads per (device, world), one failure page per device.
// ---------------------------------------------------------------------------------
struct VrDevice {
    Pad *pads[kMaxWorld + 1] = {};      // pads[world] -> `world` consecutive Pads
    uint4 *ll[kMaxWorld + 1] = {};      // ll[world] -> `world` LL receive areas
    uint64_t ll_pairs[kMaxWorld + 1] = {};
    ErrBlock *err_h = nullptr, *err_d = nullptr;
    StreamOrder order;                  // virtual-rank calls share these pads too
    BucketSet set[kMaxWorld + 1];       // open bucket set per world (gdraa_vr_bucket_set_*)
};

}  // namespace

// Kernel variant switches.  Exit fence: one fence.acq_rel.sys per CTA after
// __syncthreads() (default) -- measured 6-7 us faster per call than one per thread at
// R50 (N = 2: 166.5 -> 160.0 us, N = 4: 244.1 -> 237.3 us; profiles/r62_fence_ab.json);
// GDRAA_EXIT_FENCE=thread restores the per-thread fence for A/B runs.
uint32_t env_kernel_flags() {
    static const uint32_t v = [] {
        const char *e = std::getenv("GDRAA_EXIT_FENCE");
        return (e != nullptr && std::strcmp(e, "thread") == 0) ? 0u : kFlagCtaFence;
    }();
    return v;
}

uint64_t ll_limit_bytes(int world) {
    if (world < 2) return 0;
    const uint64_t dflt = kLLBaseBytes / static_cast<uint64_t>(world - 1);
    return env_u64("GDRAA_LL_MAX_BYTES", dflt) / 8 * 8;
}

uint64_t ll_sgd_limit_bytes(int world) {
    if (world < 2) return 0;
    const uint64_t dflt = kLLSgdBaseBytes / static_cast<uint64_t>(world - 1);
    return env_u64("GDRAA_LL_SGD_MAX_BYTES", dflt);
}

namespace {

// One rank's LL receive area: [2 parities][world senders][pairs] x 16 bytes.
size_t ll_area_bytes(int world, uint64_t pairs) { return 2ull * world * pairs * sizeof(uint4); }
std::map<int, VrDevice> g_vr;

int vr_prepare(int world, VrDevice **out) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    VrDevice &d = g_vr[dev];
    if (d.err_h == nullptr) {
        void *h = nullptr;
        CUDA_TRY(cudaHostAlloc(&h, sizeof(ErrBlock), cudaHostAllocMapped | cudaHostAllocPortable));
        std::memset(h, 0, sizeof(ErrBlock));
        d.err_h = static_cast<ErrBlock *>(h);
        void *dp = nullptr;
        CUDA_TRY(cudaHostGetDevicePointer(&dp, h, 0));
        d.err_d = static_cast<ErrBlock *>(dp);
    }
    if (d.err_h->code != 0) {
        std::string miss;
        for (int p = 0; p < kMaxWorld; ++p)
            if (d.err_h->missing[p]) miss += (miss.empty() ? "" : ",") + std::to_string(p);
        return fail(GDRAA_ETIMEOUT, "virtual-rank peer timeout (phase %d, vrank %d): missing %s",
                    d.err_h->phase, d.err_h->vrank, miss.c_str());
    }
    if (d.pads[world] == nullptr) {
        void *pp = nullptr;
        CUDA_TRY(cudaMalloc(&pp, sizeof(Pad) * world));
        CUDA_TRY(cudaMemset(pp, 0, sizeof(Pad) * world));
        d.pads[world] = static_cast<Pad *>(pp);
    }
    const uint64_t pairs = ll_limit_bytes(world) / 8;
    if (world > 1 && pairs > 0 && d.ll[world] == nullptr) {
        void *lp = nullptr;
        CUDA_TRY(cudaMalloc(&lp, ll_area_bytes(world, pairs) * world));
        CUDA_TRY(cudaMemset(lp, 0, ll_area_bytes(world, pairs) * world));
        d.ll[world] = static_cast<uint4 *>(lp);
        d.ll_pairs[world] = pairs;
    }
    *out = &d;
    return GDRAA_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// One virtual-rank call: src = g (or buf), dst = w / buf / bf16 model copy, v and wm
// (master, kSgdMp only) rank-local.
struct VrArgs {
    int world;
    const void *const *src;
    void *const *dst;
    float *const *v;
    float *const *wm;
    size_t n;
    int dtype;
    float lr, mom, wd;
    int mode;
    size_t first = 0;    // element offset already applied to the pointers (range calls)
};

int vr_run(const VrArgs &a, cudaStream_t s) {
    const int world = a.world, mode = a.mode;
    const bool upd = mode != kMean;
    if (world < 1 || world > kMaxWorld) return fail(GDRAA_EINVAL, "world %d out of [1,%d]", world, kMaxWorld);
    if (a.n == 0) return fail(GDRAA_EINVAL, "n must be >= 1");
    if (a.dtype != GDRAA_F32 && a.dtype != GDRAA_BF16) return fail(GDRAA_EINVAL, "bad dtype %d", a.dtype);
    if (a.src == nullptr || a.dst == nullptr || (upd && a.v == nullptr) ||
        (mode == kSgdMp && a.wm == nullptr))
        return fail(GDRAA_EINVAL, "null pointer array");
    if (upd && !(std::isfinite(a.lr) && std::isfinite(a.mom) && std::isfinite(a.wd)))
        return fail(GDRAA_EINVAL, "lr, mom and wd must be finite");
    for (int q = 0; q < world; ++q) {
        if (a.src[q] == nullptr || a.dst[q] == nullptr || !aligned16(a.src[q]) ||
            !aligned16(a.dst[q]) || (upd && (a.v[q] == nullptr || !aligned16(a.v[q]))) ||
            (mode == kSgdMp && (a.wm[q] == nullptr || !aligned16(a.wm[q]))))
            return fail(GDRAA_EINVAL, "rank %d: null or non-16-byte-aligned buffer", q);
    }
    const int dtype = a.dtype;
    const size_t n = a.n;
    const void *const *src = a.src;
    void *const *dst = a.dst;
    VrDevice *d = nullptr;
    int rc = vr_prepare(world, &d);
    if (rc) return rc;
    KParams p;
    std::memset(&p, 0, sizeof p);
    p.world = world;
    p.rank0 = 0;
    p.n = n;
    uint64_t off, len;
    partition(n, world, 0, &p.blk, &off, &len);
    p.lr = a.lr;
    p.mom = a.mom;
    p.wd = a.wd;
    p.timeout_ns = env_u64("GDRAA_TIMEOUT_MS", 30000) * 1000000ull;
    for (int r = 0; r < world; ++r) {
        for (int q = 0; q < world; ++q) {
            p.src[r][q] = src[q];
            p.dst[r][q] = dst[q];
            p.pad[r][q] = d->pads[world] + q;
            if (d->ll[world] != nullptr)
                p.ll[r][q] = d->ll[world] +
                             q * (ll_area_bytes(world, d->ll_pairs[world]) / sizeof(uint4));
        }
        p.v[r] = upd ? a.v[r] : nullptr;
        p.wm[r] = mode == kSgdMp ? a.wm[r] : nullptr;
    }
    p.err = d->err_d;
    p.ll_pairs = d->ll[world] != nullptr ? d->ll_pairs[world] : 0;
    p.ll_sleep_ns = static_cast<uint32_t>(env_u64("GDRAA_LL_SLEEP_NS", 256));
    BucketSet &set = d->set[world];
    p.flags = env_kernel_flags() | (set.open ? kFlagDeferExit : 0u);
    const size_t es = dtype == GDRAA_F32 ? 4 : 2;
    const size_t ed = mode == kSgd ? 4 : (mode == kSgdMp ? 2 : es);
    for (int q = 0; q < world; ++q) {
        rc = set_check(set, dst[q], n * ed);
        if (rc) return rc;
    }
    if (set.open && set.st.on && world > 1) {          // streamed bucket set
        rc = streamed_call(set, d->order, p, world, true, dtype, mode, s, a.first, n);
        if (rc) return rc;
        for (int q = 0; q < world; ++q) set_note(set, dst[q], n * ed);
        return GDRAA_OK;
    }
    rc = order_after_previous(d->order, s);
    if (rc) return rc;
    cudaError_t e;
    const char *what;
    if (mode == kMean && world > 1 && n * es <= 8 * p.ll_pairs) {   // latency path
        e = launch_gdraa_ll(p, dtype, world, true, s);
        what = "vr LL launch";
    } else if (upd && world > 1 && n * es <= ll_sgd_limit_bytes(world) &&
               ll_sgd_fits(p.blk, dtype, mode, p.ll_pairs)) {   // small-message SGD step
        e = launch_gdraa_ll_sgd(p, dtype, mode, world, true, s);
        what = "vr LL SGD launch";
    } else {
        int gx = 0;
        e = use_tma_kernel(dtype, mode, world)
                ? launch_gdraa_tma(p, dtype, mode, world, true, s, &gx)
                : launch_gdraa(p, dtype, mode, world, true, s, &gx);
        what = "vr kernel launch";
    }
    if (e != cudaSuccess) return fail(GDRAA_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    for (int q = 0; q < world; ++q) set_note(set, dst[q], n * ed);
    return note_launch(d->order, s);
}

}  // namespace
}  // namespace gdraa

using namespace gdraa;

extern "C" {

const char *gdraa_last_error(void) { return t_err.c_str(); }

const char *gdraa_version(void) { return "gdraa 0.1.0 (sm_100a)"; }

size_t gdraa_small_message_bytes(int world) {
    if (world < 1 || world > kMaxWorld) return 0;
    return static_cast<size_t>(ll_limit_bytes(world));
}

size_t gdraa_small_step_bytes(int world, int dtype, int mixed) {
    if (world < 2 || world > kMaxWorld || (dtype != GDRAA_F32 && dtype != GDRAA_BF16)) return 0;
    const uint64_t lim = ll_sgd_limit_bytes(world), pairs = ll_limit_bytes(world) / 8;
    const uint64_t es = elem_size(dtype);
    // largest n <= lim / es whose shard fits one sender's LL slot (blk grows with n)
    const int mode = mixed ? kSgdMp : kSgd;
    uint64_t lo = 0, hi = lim / es;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo + 1) / 2;
        uint64_t blk, off, len;
        partition(mid, world, 0, &blk, &off, &len);
        if (ll_sgd_fits(blk, dtype, mode, pairs)) lo = mid; else hi = mid - 1;
    }
    const uint64_t n = lo;
    return static_cast<size_t>(n * es);
}

int gdraa_shard(int world, int rank, size_t n, size_t *off, size_t *len) {
    if (off == nullptr || len == nullptr) return fail(GDRAA_EINVAL, "null output pointer");
    if (n == 0) return fail(GDRAA_EINVAL, "n must be >= 1");
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        return fail(GDRAA_EINVAL, "world %d / rank %d out of range", world, rank);
    uint64_t b, o, l;
    partition(n, world, rank, &b, &o, &l);
    *off = o;
    *len = l;
    return GDRAA_OK;
}

// Frees everything gdraa_init acquired (socket, peer mappings, pads, pages) and resets
// the state; used by gdraa_finalize and when gdraa_init fails part-way.
static void release_resources() {
    if (g.sock >= 0) ::close(g.sock);
    for (auto &kv : g.opened) cudaIpcCloseMemHandle(kv.second);
    if (g.pad) cudaFree(g.pad);
    if (g.ll) cudaFree(g.ll);
    if (g.page_registered) cudaHostUnregister(g.page);
    if (g.page) munmap(g.page, 4096);
    if (g.err_h) cudaFreeHost(g.err_h);
    if (g.order.ev) cudaEventDestroy(g.order.ev);
    streamed_free(g.set.st);
    State s;
    g = s;
}

static int init_impl(int world, int rank);

int gdraa_init(int world, int rank) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g.inited) return fail(GDRAA_ESTATE, "already initialised (world %d, rank %d)", g.world, g.rank);
    const int rc = init_impl(world, rank);
    if (rc != GDRAA_OK) {   // leave nothing half-built behind (a retry starts clean)
        const std::string keep = t_err;
        release_resources();
        t_err = keep;
    }
    return rc;
}

static int init_impl(int world, int rank) {
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        return fail(GDRAA_EINVAL, "world %d / rank %d out of range [1,%d]", world, rank, kMaxWorld);
    State s;
    g = s;
    g.world = world;
    g.rank = rank;
    g.timeout_ns = env_u64("GDRAA_TIMEOUT_MS", 30000) * 1000000ull;
    CUDA_TRY(cudaGetDevice(&g.device));
    int cc_major = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, g.device));
    if (cc_major != 10) return fail(GDRAA_ECUDA, "device %d is not sm_100 (compute %d.x)", g.device, cc_major);

    auto cleanup_fail = [&](int rc) {
        if (g.sock >= 0) ::close(g.sock);
        g.sock = -1;
        return rc;
    };

    // Signal pad and failure page.
    void *pp = nullptr;
    CUDA_TRY(cudaMalloc(&pp, sizeof(Pad)));
    CUDA_TRY(cudaMemset(pp, 0, sizeof(Pad)));
    CUDA_TRY(cudaDeviceSynchronize());
    g.pad = static_cast<Pad *>(pp);
    void *eh = nullptr;
    CUDA_TRY(cudaHostAlloc(&eh, sizeof(ErrBlock), cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(eh, 0, sizeof(ErrBlock));
    g.err_h = static_cast<ErrBlock *>(eh);
    void *ed = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(&ed, eh, 0));
    g.err_d = static_cast<ErrBlock *>(ed);

    const char *js = std::getenv("GDRAA_JOBSERVER");
    if (world > 1 && (js == nullptr || *js == 0))
        return fail(GDRAA_EJOBSERVER, "world > 1 needs GDRAA_JOBSERVER=<socket path> "
                                      "(start paper_1802_02326_b200.jobserver)");
    if (js != nullptr && *js != 0) {
        int rc = connect_jobserver(js, env_u64("GDRAA_CONNECT_TIMEOUT_MS", 120000) * 1000000ull);
        if (rc) return rc;
        proto::Hello hello{};
        hello.world = world;
        hello.pid = static_cast<int32_t>(getpid());
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, g.device) == cudaSuccess)
            std::memcpy(hello.uuid, &prop.uuid, sizeof hello.uuid);
        rc = send_msg(proto::HELLO, 0, &hello, sizeof hello);
        if (rc) return cleanup_fail(rc);
        proto::HelloOk ok{};
        rc = recv_msg(proto::HELLO_OK, 0, &ok, sizeof ok,
                      env_u64("GDRAA_CONNECT_TIMEOUT_MS", 120000) * 1000000ull);
        if (rc) return cleanup_fail(rc);
        g.gated = ok.gated != 0;
        int fd = shm_open(ok.shm_name, O_RDWR, 0);
        if (fd < 0) return cleanup_fail(fail(GDRAA_EJOBSERVER, "shm_open(%s): %s", ok.shm_name, std::strerror(errno)));
        void *mem = mmap(nullptr, 4096, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        ::close(fd);
        if (mem == MAP_FAILED) return cleanup_fail(fail(GDRAA_EJOBSERVER, "mmap shm: %s", std::strerror(errno)));
        g.page = static_cast<proto::ShmPage *>(mem);
    } else {
        void *mem = mmap(nullptr, 4096, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
        if (mem == MAP_FAILED) return fail(GDRAA_ECUDA, "mmap: %s", std::strerror(errno));
        std::memset(mem, 0, 4096);
        g.page = static_cast<proto::ShmPage *>(mem);
        g.page_owned = true;
    }
    // Kernels write done[rank] ("IterDone") straight into the shared page.
    cudaError_t e = cudaHostRegister(g.page, 4096, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) return cleanup_fail(fail(GDRAA_ECUDA, "cudaHostRegister(go/done page): %s", cudaGetErrorString(e)));
    g.page_registered = true;
    void *pd = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(&pd, g.page, 0));
    g.done_d = &static_cast<proto::ShmPage *>(pd)->done[rank];
    g.abort_d = &static_cast<proto::ShmPage *>(pd)->abort;

    // Exchange signal pads (registration sequence 1).
    void *peers[kMaxWorld] = {};
    if (world > 1) {
        int rc = ipc_exchange(g.pad, sizeof(Pad), sizeof(Pad), -1, 0, peers);
        if (rc) return cleanup_fail(rc);
    } else {
        peers[0] = g.pad;
    }
    for (int p = 0; p < world; ++p) g.peer_pad[p] = static_cast<Pad *>(peers[p]);

    // Small-message receive slots (registration sequence 2): [2][world][pairs] x 16 B.
    const uint64_t ll_bytes = ll_limit_bytes(world);
    if (world > 1 && ll_bytes > 0) {
        g.ll_pairs = ll_bytes / 8;
        const size_t sz = ll_area_bytes(world, g.ll_pairs);
        void *lp = nullptr;
        CUDA_TRY(cudaMalloc(&lp, sz));
        CUDA_TRY(cudaMemset(lp, 0, sz));
        CUDA_TRY(cudaDeviceSynchronize());
        g.ll = static_cast<uint4 *>(lp);
        void *lpeers[kMaxWorld] = {};
        int rc = ipc_exchange(g.ll, sz, sz, -2, 2, lpeers);
        if (rc) return cleanup_fail(rc);
        for (int p = 0; p < world; ++p) g.peer_ll[p] = static_cast<uint4 *>(lpeers[p]);
    }
    // Path selection must agree on every rank (a rank on the LL path and a peer on the
    // two-shot path would wait for each other until the timeout): the thresholds are fixed
    // here and checked across ranks through the job server (registration sequence 3).
    g.ll_sgd_limit = g.ll_pairs ? ll_sgd_limit_bytes(world) : 0;
    if (world > 1) {
        proto::Reg cfg{};
        cfg.what = 3;
        cfg.n = g.ll_sgd_limit;
        cfg.dtype = static_cast<int32_t>(std::min<uint64_t>(g.ll_pairs, INT32_MAX));
        proto::RegOk all{};
        int rc = exchange(cfg, &all);
        if (rc == GDRAA_ESHAPE)
            rc = fail(GDRAA_ESHAPE, "ranks disagree on the small-message thresholds "
                      "(GDRAA_LL_MAX_BYTES / GDRAA_LL_SGD_MAX_BYTES must match on every "
                      "rank): %s",
                      t_err.c_str());
        if (rc) return cleanup_fail(rc);
    }
    g.inited = true;
    return GDRAA_OK;
}

int gdraa_register(void *buf, size_t n, int dtype) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_sticky();
    if (rc) return rc;
    if (buf == nullptr || n == 0) return fail(GDRAA_EINVAL, "null buffer or n == 0");
    if (dtype != GDRAA_F32 && dtype != GDRAA_BF16) return fail(GDRAA_EINVAL, "bad dtype %d", dtype);
    if (!aligned16(buf)) return fail(GDRAA_EINVAL, "buffer %p is not 16-byte aligned", buf);
    if (find_reg(buf) != nullptr) return fail(GDRAA_EINVAL, "buffer %p already registered", buf);
    Registration r;
    r.local = buf;
    r.n = n;
    r.dtype = dtype;
    if (g.world > 1) {
        rc = ipc_exchange(buf, n * elem_size(dtype), n, dtype, 1, r.peer);
        if (rc) return rc;
    } else {
        cudaPointerAttributes a;
        CUDA_TRY(cudaPointerGetAttributes(&a, buf));
        if (a.type != cudaMemoryTypeDevice) return fail(GDRAA_EINVAL, "buffer %p is not device memory", buf);
        r.peer[0] = buf;
    }
    g.regs.push_back(r);
    return GDRAA_OK;
}

int gdraa_deregister(void *buf) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited) return fail(GDRAA_ESTATE, "gdraa_init has not been called");
    for (auto it = g.regs.begin(); it != g.regs.end(); ++it) {
        if (it->local == buf) {
            g.regs.erase(it);
            return GDRAA_OK;
        }
    }
    return fail(GDRAA_ENOTREG, "buffer %p is not registered", buf);
}

// Resolve the element range [first, first + count) of a registration (count == SIZE_MAX:
// the whole buffer).  Ranges start on an 8-element boundary so every vector access and
// every 1-D bulk copy (16-byte aligned, also for bf16) stays aligned.
static int resolve_range(const Registration *r, size_t first, size_t *count) {
    if (*count == SIZE_MAX) {
        if (first != 0) return fail(GDRAA_EINVAL, "whole-buffer call with first != 0");
        *count = r->n;
        return GDRAA_OK;
    }
    if (*count == 0) return fail(GDRAA_EINVAL, "count must be >= 1");
    if (first % 8 != 0) return fail(GDRAA_EINVAL, "first (%zu) must be a multiple of 8", first);
    if (first > r->n || *count > r->n - first)
        return fail(GDRAA_EINVAL, "range [%zu, %zu) exceeds the registered %zu elements", first,
                    first + *count, r->n);
    return GDRAA_OK;
}

static void *offset_ptr(void *p, size_t elems, size_t es) {
    return p == nullptr ? nullptr : static_cast<char *>(p) + elems * es;
}

static int mean_common(void *buf, size_t first, size_t count, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_sticky();
    if (rc) return rc;
    const Registration *r = find_reg(buf);
    if (r == nullptr) return fail(GDRAA_ENOTREG, "buffer %p is not registered", buf);
    rc = resolve_range(r, first, &count);
    if (rc) return rc;
    rc = wait_go();
    if (rc) return rc;
    const size_t es = elem_size(r->dtype);
    rc = set_check(g.set, offset_ptr(r->local, first, es), count * es);
    if (rc) return rc;
    KParams p;
    fill_common(p, count);
    for (int q = 0; q < g.world; ++q) {
        p.src[0][q] = offset_ptr(r->peer[q], first, es);
        p.dst[0][q] = offset_ptr(r->peer[q], first, es);
    }
    const cudaStream_t cs = reinterpret_cast<cudaStream_t>(s);
    if (g.set.open && g.set.st.on && g.world > 1) {    // streamed bucket set
        const bool first_call = !g.set.st.launched;
        rc = streamed_call(g.set, g.order, p, 1, false, r->dtype, kMean, cs, first, count);
        if (rc) return rc;
        account(count, r->dtype, 0, first_call);
        set_note(g.set, offset_ptr(r->local, first, es), count * es);
        return GDRAA_OK;
    }
    rc = order_after_previous(g.order, cs);
    if (rc) return rc;
    if (g.ll != nullptr && count * es <= 8 * g.ll_pairs) {
        // small message: the latency path (same result, bit for bit)
        cudaError_t e = launch_gdraa_ll(p, r->dtype, 1, false, cs);
        if (e != cudaSuccess) return fail(GDRAA_ECUDA, "LL kernel launch: %s", cudaGetErrorString(e));
        g.issued += 1;
    } else {
        rc = launch(p, r->dtype, kMean, cs);
        if (rc) return rc;
    }
    account(count, r->dtype, 0);
    set_note(g.set, offset_ptr(r->local, first, es), count * es);
    return note_launch(g.order, cs);
}

int gdraa_allreduce_mean(void *buf, gdraa_stream_t s) { return mean_common(buf, 0, SIZE_MAX, s); }

int gdraa_allreduce_mean_range(void *buf, size_t first, size_t count, gdraa_stream_t s) {
    if (count == SIZE_MAX) return fail(GDRAA_EINVAL, "count out of range");
    return mean_common(buf, first, count, s);
}

// Shared body of gdraa_sgd_step / _ex / _range (mode kSgd: dst = replicated fp32 w) and
// gdraa_sgd_step_mp / _mp_range (mode kSgdMp: dst = replicated bf16 model copy, wm =
// local master), on the element range [first, first + count) (SIZE_MAX: everything).
static int sgd_common(int mode, float *wm, void *dst, const void *gr, float *v, size_t first,
                      size_t count, float lr, float mom, float wd, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = check_sticky();
    if (rc) return rc;
    if (!(std::isfinite(lr) && std::isfinite(mom) && std::isfinite(wd)))
        return fail(GDRAA_EINVAL, "lr, mom and wd must be finite");
    const char *dname = mode == kSgd ? "w" : "w_model";
    const Registration *rw = find_reg(dst);
    const Registration *rg = find_reg(gr);
    if (rw == nullptr) return fail(GDRAA_ENOTREG, "%s %p is not registered", dname, dst);
    if (rg == nullptr) return fail(GDRAA_ENOTREG, "g %p is not registered", gr);
    const int want = mode == kSgd ? GDRAA_F32 : GDRAA_BF16;
    if (rw->dtype != want)
        return fail(GDRAA_EINVAL, "%s must be registered as %s", dname,
                    want == GDRAA_F32 ? "GDRAA_F32" : "GDRAA_BF16");
    if (rw->n != rg->n)
        return fail(GDRAA_EINVAL, "%s (n=%zu) and g (n=%zu) differ in length", dname, rw->n, rg->n);
    if (rw == rg) return fail(GDRAA_EINVAL, "%s and g must be distinct buffers", dname);
    if (v == nullptr || !aligned16(v)) return fail(GDRAA_EINVAL, "v is null or not 16-byte aligned");
    if (mode == kSgdMp && (wm == nullptr || !aligned16(wm)))
        return fail(GDRAA_EINVAL, "w_master is null or not 16-byte aligned");
    rc = resolve_range(rw, first, &count);
    if (rc) return rc;
    rc = wait_go();
    if (rc) return rc;
    const size_t eg = elem_size(rg->dtype), ew = elem_size(rw->dtype);
    rc = set_check(g.set, offset_ptr(rw->local, first, ew), count * ew);
    if (rc) return rc;
    KParams p;
    fill_common(p, count);
    p.lr = lr;
    p.mom = mom;
    p.wd = wd;
    for (int q = 0; q < g.world; ++q) {
        p.src[0][q] = offset_ptr(rg->peer[q], first, eg);
        p.dst[0][q] = offset_ptr(rw->peer[q], first, ew);
    }
    p.v[0] = static_cast<float *>(offset_ptr(v, first, 4));
    p.wm[0] = mode == kSgdMp ? static_cast<float *>(offset_ptr(wm, first, 4)) : nullptr;
    const cudaStream_t cs = reinterpret_cast<cudaStream_t>(s);
    if (g.set.open && g.set.st.on && g.world > 1) {    // streamed bucket set
        const bool first_call = !g.set.st.launched;
        rc = streamed_call(g.set, g.order, p, 1, false, rg->dtype, mode, cs, first, count);
        if (rc) return rc;
        account(count, rg->dtype, mode == kSgd ? 4 : 2, first_call);
        set_note(g.set, offset_ptr(rw->local, first, ew), count * ew);
        return GDRAA_OK;
    }
    rc = order_after_previous(g.order, cs);
    if (rc) return rc;
    if (g.ll != nullptr && count * eg <= g.ll_sgd_limit &&
        ll_sgd_fits(p.blk, rg->dtype, mode, g.ll_pairs)) {
        // small message: the data carries both synchronisations (same result, bit for bit)
        cudaError_t e = launch_gdraa_ll_sgd(p, rg->dtype, mode, 1, false, cs);
        if (e != cudaSuccess) return fail(GDRAA_ECUDA, "LL SGD kernel launch: %s", cudaGetErrorString(e));
        g.issued += 1;
    } else {
        rc = launch(p, rg->dtype, mode, cs);
        if (rc) return rc;
    }
    account(count, rg->dtype, mode == kSgd ? 4 : 2);
    set_note(g.set, offset_ptr(rw->local, first, ew), count * ew);
    return note_launch(g.order, cs);
}

int gdraa_sgd_step(float *w, const void *gr, float *v, float lr, float mom, gdraa_stream_t s) {
    return sgd_common(kSgd, nullptr, w, gr, v, 0, SIZE_MAX, lr, mom, 0.0f, s);
}

int gdraa_sgd_step_ex(float *w, const void *gr, float *v, float lr, float mom, float wd,
                      gdraa_stream_t s) {
    return sgd_common(kSgd, nullptr, w, gr, v, 0, SIZE_MAX, lr, mom, wd, s);
}

int gdraa_sgd_step_mp(float *w_master, void *w_model, const void *gr, float *v, float lr,
                      float mom, float wd, gdraa_stream_t s) {
    return sgd_common(kSgdMp, w_master, w_model, gr, v, 0, SIZE_MAX, lr, mom, wd, s);
}

int gdraa_sgd_step_range(float *w, const void *gr, float *v, size_t first, size_t count,
                         float lr, float mom, float wd, gdraa_stream_t s) {
    if (count == SIZE_MAX) return fail(GDRAA_EINVAL, "count out of range");
    return sgd_common(kSgd, nullptr, w, gr, v, first, count, lr, mom, wd, s);
}

int gdraa_sgd_step_mp_range(float *w_master, void *w_model, const void *gr, float *v,
                            size_t first, size_t count, float lr, float mom, float wd,
                            gdraa_stream_t s) {
    if (count == SIZE_MAX) return fail(GDRAA_EINVAL, "count out of range");
    return sgd_common(kSgdMp, w_master, w_model, gr, v, first, count, lr, mom, wd, s);
}

int gdraa_bucket_set_begin(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited) return fail(GDRAA_ESTATE, "gdraa_init has not been called");
    if (g.set.open) return fail(GDRAA_ESTATE, "a bucket set is already open");
    g.set.open = true;
    g.set.spans.clear();
    return GDRAA_OK;
}

int gdraa_bucket_set_begin_streamed(int ctas) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited) return fail(GDRAA_ESTATE, "gdraa_init has not been called");
    if (g.set.open) return fail(GDRAA_ESTATE, "a bucket set is already open");
    if (ctas < 1) return fail(GDRAA_EINVAL, "ctas must be >= 1");
    if (g.gated)
        return fail(GDRAA_ESTATE, "streamed bucket sets need ungated mode (IterDone is "
                    "written once per set)");
    int rc = check_sticky();
    if (rc) return rc;
    if (g.world > 1) {
        rc = streamed_open(g.set.st, 1, ctas);
        if (rc) return rc;
    }
    g.set.open = true;
    g.set.spans.clear();
    return GDRAA_OK;
}

int gdraa_bucket_set_end(gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited) return fail(GDRAA_ESTATE, "gdraa_init has not been called");
    if (!g.set.open) return fail(GDRAA_ESTATE, "no bucket set is open");
    g.set.open = false;
    g.set.spans.clear();
    const cudaStream_t cs0 = reinterpret_cast<cudaStream_t>(s);
    if (g.set.st.on) {                     // streamed: the kernel does the exit barrier
        int rc = streamed_close(g.set, g.order, cs0);
        if (rc) return rc;
        return check_sticky();
    }
    int rc = check_sticky();
    if (rc) return rc;
    if (g.world == 1) return GDRAA_OK;     // no barrier to defer
    KParams p;
    fill_common(p, 1);
    const cudaStream_t cs = reinterpret_cast<cudaStream_t>(s);
    rc = order_after_previous(g.order, cs);
    if (rc) return rc;
    cudaError_t e = launch_gdraa_exit(p, 1, false, cs);
    if (e != cudaSuccess) return fail(GDRAA_ECUDA, "exit kernel launch: %s", cudaGetErrorString(e));
    g.host.launches += 1;
    return note_launch(g.order, cs);
}

float gdraa_poly_lr(float lr0, uint64_t iter, uint64_t max_iter, float power) {
    if (max_iter == 0) return -1.0f;
    if (iter >= max_iter) return 0.0f;
    const double frac = 1.0 - static_cast<double>(iter) / static_cast<double>(max_iter);
    return static_cast<float>(static_cast<double>(lr0) * std::pow(frac, static_cast<double>(power)));
}

int gdraa_get_stats(gdraa_stats_t *out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (out == nullptr) return fail(GDRAA_EINVAL, "null output");
    if (!g.inited) return fail(GDRAA_ESTATE, "gdraa_init has not been called");
    if (g.set.st.launched)
        return fail(GDRAA_ESTATE, "a streamed bucket set is open (its kernel waits for "
                    "gdraa_bucket_set_end; synchronising now would wait for ever)");
    CUDA_TRY(cudaDeviceSynchronize());
    Pad host;
    CUDA_TRY(cudaMemcpy(&host, g.pad, sizeof host, cudaMemcpyDeviceToHost));
    *out = g.host;
    out->calls = host.calls;
    out->sync_waits = host.sync_waits;
    out->ll_calls = host.ll_calls;
    out->iter_done = g.page ? g.page->done[g.rank] : 0;
    out->iter_start = g.page ? g.page->go[g.rank] : 0;
    return GDRAA_OK;
}

int gdraa_finalize(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g.inited) return fail(GDRAA_ESTATE, "gdraa_init has not been called");
    int rc = GDRAA_OK;
    if (g.set.open && g.set.st.launched && !g.fatal) {
        // a streamed set left open: close it where its last bucket was described
        const int crc = streamed_close(g.set, g.order, g.set.st.last);
        if (crc) rc = crc;
        g.set.open = false;
    }
    if (g.set.open && g.world > 1 && !g.fatal) {
        // a bucket set left open: run its deferred exit barrier so that the peers'
        // gdraa_bucket_set_end (which waits for ours) completes
        KParams p;
        fill_common(p, 1);
        if (cudaDeviceSynchronize() != cudaSuccess ||
            launch_gdraa_exit(p, 1, false, nullptr) != cudaSuccess)
            rc = fail(GDRAA_ECUDA, "exit kernel launch at finalize");
    }
    g.set.open = false;
    cudaError_t se = cudaDeviceSynchronize();
    {
        int st = check_sticky();
        if (st) rc = st;
    }
    if (se != cudaSuccess && rc == GDRAA_OK) rc = fail(GDRAA_ECUDA, "cudaDeviceSynchronize: %s", cudaGetErrorString(se));
    std::string keep = t_err;
    if (g.sock >= 0) {
        if (send_msg(proto::BYE, 0, nullptr, 0) == GDRAA_OK && !g.fatal) {
            int brc = recv_msg(proto::BYE_OK, 0, nullptr, 0, 60000000000ull);
            if (brc && rc == GDRAA_OK) {
                rc = brc;
                keep = t_err;
            }
        }
    }
    release_resources();
    t_err = keep;
    return rc;
}

int gdraa_vr_allreduce_mean(int world, void *const *bufs, size_t n, int dtype, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    VrArgs a{world, reinterpret_cast<const void *const *>(bufs), bufs, nullptr, nullptr, n, dtype,
             0.f, 0.f, 0.f, kMean};
    return vr_run(a, reinterpret_cast<cudaStream_t>(s));
}

int gdraa_vr_sgd_step(int world, float *const *w, const void *const *g_, float *const *v, size_t n,
                      int dtype, float lr, float mom, gdraa_stream_t s) {
    return gdraa_vr_sgd_step_ex(world, w, g_, v, n, dtype, lr, mom, 0.0f, s);
}

int gdraa_vr_sgd_step_ex(int world, float *const *w, const void *const *g_, float *const *v,
                         size_t n, int dtype, float lr, float mom, float wd, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    VrArgs a{world, g_, reinterpret_cast<void *const *>(w), v, nullptr, n, dtype, lr, mom, wd, kSgd};
    return vr_run(a, reinterpret_cast<cudaStream_t>(s));
}

int gdraa_vr_sgd_step_mp(int world, float *const *w_master, void *const *w_model,
                         const void *const *g_, float *const *v, size_t n, int dtype, float lr,
                         float mom, float wd, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    VrArgs a{world, g_, w_model, v, w_master, n, dtype, lr, mom, wd, kSgdMp};
    return vr_run(a, reinterpret_cast<cudaStream_t>(s));
}

// Bucketed virtual-rank calls: the same kernels on [first, first + count) of every rank's
// buffers (the owner rule of gdraa_sgd_step_range applies to the range).
static int vr_range(VrArgs a, size_t first, size_t count, cudaStream_t s) {
    if (a.world < 1 || a.world > kMaxWorld) return fail(GDRAA_EINVAL, "world %d out of [1,%d]", a.world, kMaxWorld);
    if (count == 0) return fail(GDRAA_EINVAL, "count must be >= 1");
    if (first % 8 != 0) return fail(GDRAA_EINVAL, "first (%zu) must be a multiple of 8", first);
    if (first > a.n || count > a.n - first)
        return fail(GDRAA_EINVAL, "range [%zu, %zu) exceeds the %zu elements", first,
                    first + count, a.n);
    if (a.src == nullptr || a.dst == nullptr || (a.mode != kMean && a.v == nullptr) ||
        (a.mode == kSgdMp && a.wm == nullptr))
        return fail(GDRAA_EINVAL, "null pointer array");
    const size_t eg = a.dtype == GDRAA_F32 ? 4 : 2;
    const size_t ed = a.mode == kSgd ? 4 : (a.mode == kSgdMp ? 2 : eg);
    const void *src[kMaxWorld];
    void *dst[kMaxWorld];
    float *v[kMaxWorld], *wm[kMaxWorld];
    for (int q = 0; q < a.world; ++q) {
        src[q] = offset_ptr(const_cast<void *>(a.src[q]), first, eg);
        dst[q] = offset_ptr(a.dst[q], first, ed);
        v[q] = a.v ? static_cast<float *>(offset_ptr(a.v[q], first, 4)) : nullptr;
        wm[q] = a.wm ? static_cast<float *>(offset_ptr(a.wm[q], first, 4)) : nullptr;
    }
    a.src = src;
    a.dst = dst;
    a.v = a.v ? v : nullptr;
    a.wm = a.wm ? wm : nullptr;
    a.n = count;
    a.first = first;
    return vr_run(a, s);
}

int gdraa_vr_allreduce_mean_range(int world, void *const *bufs, size_t n, int dtype,
                                  size_t first, size_t count, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    VrArgs a{world, reinterpret_cast<const void *const *>(bufs), bufs, nullptr, nullptr, n, dtype,
             0.f, 0.f, 0.f, kMean};
    return vr_range(a, first, count, reinterpret_cast<cudaStream_t>(s));
}

int gdraa_vr_sgd_step_range(int world, float *const *w, const void *const *g_, float *const *v,
                            size_t n, int dtype, size_t first, size_t count, float lr, float mom,
                            float wd, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    VrArgs a{world, g_, reinterpret_cast<void *const *>(w), v, nullptr, n, dtype, lr, mom, wd, kSgd};
    return vr_range(a, first, count, reinterpret_cast<cudaStream_t>(s));
}

int gdraa_vr_sgd_step_mp_range(int world, float *const *w_master, void *const *w_model,
                               const void *const *g_, float *const *v, size_t n, int dtype,
                               size_t first, size_t count, float lr, float mom, float wd,
                               gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    VrArgs a{world, g_, w_model, v, w_master, n, dtype, lr, mom, wd, kSgdMp};
    return vr_range(a, first, count, reinterpret_cast<cudaStream_t>(s));
}

int gdraa_vr_bucket_set_begin(int world) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (world < 1 || world > kMaxWorld) return fail(GDRAA_EINVAL, "world %d out of [1,%d]", world, kMaxWorld);
    VrDevice *d = nullptr;
    int rc = vr_prepare(world, &d);
    if (rc) return rc;
    if (d->set[world].open) return fail(GDRAA_ESTATE, "a bucket set is already open (world %d)", world);
    d->set[world].open = true;
    d->set[world].spans.clear();
    return GDRAA_OK;
}

int gdraa_vr_bucket_set_begin_streamed(int world, int ctas) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (world < 1 || world > kMaxWorld) return fail(GDRAA_EINVAL, "world %d out of [1,%d]", world, kMaxWorld);
    if (ctas < 1) return fail(GDRAA_EINVAL, "ctas must be >= 1");
    VrDevice *d = nullptr;
    int rc = vr_prepare(world, &d);
    if (rc) return rc;
    if (d->set[world].open) return fail(GDRAA_ESTATE, "a bucket set is already open (world %d)", world);
    if (world > 1) {
        rc = streamed_open(d->set[world].st, world, ctas);
        if (rc) return rc;
    }
    d->set[world].open = true;
    d->set[world].spans.clear();
    return GDRAA_OK;
}

int gdraa_vr_bucket_set_end(int world, gdraa_stream_t s) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (world < 1 || world > kMaxWorld) return fail(GDRAA_EINVAL, "world %d out of [1,%d]", world, kMaxWorld);
    VrDevice *d = nullptr;
    int rc = vr_prepare(world, &d);
    if (rc) return rc;
    if (!d->set[world].open) return fail(GDRAA_ESTATE, "no bucket set is open (world %d)", world);
    d->set[world].open = false;
    d->set[world].spans.clear();
    if (d->set[world].st.on)
        return streamed_close(d->set[world], d->order, reinterpret_cast<cudaStream_t>(s));
    if (world == 1) return GDRAA_OK;
    KParams p;
    std::memset(&p, 0, sizeof p);
    p.world = world;
    p.rank0 = 0;
    p.timeout_ns = env_u64("GDRAA_TIMEOUT_MS", 30000) * 1000000ull;
    for (int r = 0; r < world; ++r)
        for (int q = 0; q < world; ++q) p.pad[r][q] = d->pads[world] + q;
    p.err = d->err_d;
    const cudaStream_t cs = reinterpret_cast<cudaStream_t>(s);
    rc = order_after_previous(d->order, cs);
    if (rc) return rc;
    cudaError_t e = launch_gdraa_exit(p, world, true, cs);
    if (e != cudaSuccess) return fail(GDRAA_ECUDA, "vr exit kernel launch: %s", cudaGetErrorString(e));
    return note_launch(d->order, cs);
}

}  // extern "C"
