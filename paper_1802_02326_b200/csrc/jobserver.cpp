// gdraa_jobserver -- the MiMatrix "job server" control plane.
//
//   gdraa_jobserver --socket PATH --world N [--gated] [--timeout-ms T] [--stats FILE]
//
// Message-driven: it accepts N rank connections on a Unix socket, rendezvouses
// HELLO, relays CUDA IPC handles for every registration after checking that n / dtype
// agree (S:177 shape-mismatch), owns the shared go/done page the kernels write their
// per-iteration completion into, and ends with a collective BYE.  It never opens an IPC
// handle and links no CUDA library, so it cannot touch weight data (structural evidence:
// tests/test_jobserver.py::test_jobserver_links_no_cuda).  Its data_bytes counter counts
// the payload of any message outside the control vocabulary (the sender is dropped) and
// is reported at exit.
#include <fcntl.h>
#include <poll.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <sys/stat.h>
#include <sys/un.h>
#include <time.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "jobserver_proto.h"

using namespace gdraa::proto;

namespace {

constexpr int kEINVAL = -1, kESHAPE = -3, kEJOBSERVER = -7;

struct Client {
    int fd = -1;
    int rank = -1;
    bool hello = false;
    bool bye = false;
    bool gone = false;
};

uint64_t now_ms() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return static_cast<uint64_t>(ts.tv_sec) * 1000u + ts.tv_nsec / 1000000u;
}

bool read_all(int fd, void *buf, size_t n) {
    char *p = static_cast<char *>(buf);
    while (n > 0) {
        ssize_t k = ::recv(fd, p, n, 0);
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

bool write_all(int fd, const void *buf, size_t n) {
    const char *p = static_cast<const char *>(buf);
    while (n > 0) {
        ssize_t k = ::send(fd, p, n, MSG_NOSIGNAL);
        if (k < 0) {
            if (errno == EINTR) continue;
            return false;
        }
        p += k;
        n -= static_cast<size_t>(k);
    }
    return true;
}

struct Server {
    int world = 0;
    bool gated = false;
    uint64_t timeout_ms = 120000;
    std::string sock_path, stats_path, shm_name;
    int lfd = -1;
    ShmPage *page = nullptr;
    std::vector<Client> clients;
    std::map<uint32_t, std::map<int, Reg>> pending;   // seq -> rank -> record
    int hellos = 0, byes = 0;
    bool failed = false;
    std::string fail_msg;

    bool send_msg(Client &c, uint16_t kind, uint32_t seq, const void *payload, uint32_t len) {
        Hdr h{kMagic, kind, static_cast<uint16_t>(c.rank < 0 ? 0 : c.rank), len, seq};
        page->control_bytes = page->control_bytes + sizeof h + len;
        return write_all(c.fd, &h, sizeof h) && (len == 0 || write_all(c.fd, payload, len));
    }

    void broadcast_fail(int code, const std::string &msg) {
        Fail f{};
        f.code = code;
        std::snprintf(f.msg, sizeof f.msg, "%s", msg.c_str());
        for (auto &c : clients)
            if (!c.gone) send_msg(c, FAIL, 0, &f, sizeof f);
    }

    void drop(Client &c, const char *why) {
        if (c.gone) return;
        c.gone = true;
        ::close(c.fd);
        // A connection that never completed HELLO is not a rank of this job (a readiness
        // probe, a stale rank of an earlier job): close it without failing the job.
        if (!c.hello) return;
        if (!c.bye && !failed) {   // the first failure is the one reported
            failed = true;
            fail_msg = "rank " + std::to_string(c.rank) + " disconnected (" + why + ")";
            page->dead_rank = c.rank;
            page->abort = 1;
            broadcast_fail(kEJOBSERVER, fail_msg);
        }
    }

    void on_message(Client &c, const Hdr &h, const std::vector<char> &body) {
        page->control_bytes = page->control_bytes + sizeof h + body.size();
        switch (h.kind) {
            case HELLO: {
                if (body.size() != sizeof(Hello) || c.hello) return drop(c, "bad HELLO");
                Hello m;
                std::memcpy(&m, body.data(), sizeof m);
                if (m.world != world || h.rank >= world) {
                    Fail f{};
                    f.code = kEINVAL;
                    std::snprintf(f.msg, sizeof f.msg, "world %d / rank %d do not match job world %d",
                                  m.world, h.rank, world);
                    c.rank = h.rank;
                    send_msg(c, FAIL, 0, &f, sizeof f);
                    return drop(c, "world mismatch");
                }
                for (auto &o : clients)
                    if (&o != &c && o.hello && o.rank == h.rank) return drop(c, "duplicate rank");
                c.rank = h.rank;
                c.hello = true;
                if (++hellos == world) {
                    HelloOk ok{};
                    std::snprintf(ok.shm_name, sizeof ok.shm_name, "%s", shm_name.c_str());
                    ok.world = world;
                    ok.gated = gated ? 1 : 0;
                    ok.job_id = static_cast<uint64_t>(getpid());
                    for (auto &o : clients)
                        if (!o.gone) send_msg(o, HELLO_OK, 0, &ok, sizeof ok);
                }
                return;
            }
            case REG: {
                if (!c.hello || body.size() != sizeof(Reg)) return drop(c, "bad REG");
                Reg r;
                std::memcpy(&r, body.data(), sizeof r);
                auto &slot = pending[h.seq];
                if (slot.count(c.rank)) return drop(c, "duplicate REG");
                slot[c.rank] = r;
                if (static_cast<int>(slot.size()) < world) return;
                // all ranks registered sequence h.seq: check shapes agree
                const Reg &r0 = slot.begin()->second;
                bool same = true;
                for (auto &kv : slot)
                    same = same && kv.second.what == r0.what && kv.second.n == r0.n &&
                           kv.second.dtype == r0.dtype;
                if (!same) {
                    Fail f{};
                    f.code = kESHAPE;
                    int k = std::snprintf(f.msg, sizeof f.msg, "registration %u: shape mismatch:",
                                          h.seq);
                    for (auto &kv : slot)
                        if (k < static_cast<int>(sizeof f.msg))
                            k += std::snprintf(f.msg + k, sizeof f.msg - k, " r%d(n=%llu,dt=%d)",
                                               kv.first, (unsigned long long)kv.second.n,
                                               kv.second.dtype);
                    for (auto &o : clients)
                        if (!o.gone) send_msg(o, REG_ERR, h.seq, &f, sizeof f);
                } else {
                    RegOk ok{};
                    ok.world = world;
                    for (auto &kv : slot) ok.regs[kv.first] = kv.second;
                    for (auto &o : clients)
                        if (!o.gone) send_msg(o, REG_OK, h.seq, &ok, sizeof ok);
                    page->registrations = page->registrations + 1;
                }
                pending.erase(h.seq);
                return;
            }
            case BYE: {
                if (c.bye) return;
                c.bye = true;
                if (++byes == world) {
                    for (auto &o : clients)
                        if (!o.gone) send_msg(o, BYE_OK, 0, nullptr, 0);
                }
                return;
            }
            default:
                // Not a control message.  None of the protocol's kinds carries tensor
                // data, so the payload of anything else is counted as data and its sender
                // dropped: data_bytes is a guard that reads 0 only if no rank ever tried
                // to move data through the job server.
                page->data_bytes = page->data_bytes + body.size();
                page->control_bytes = page->control_bytes - sizeof h - body.size();
                return drop(c, "unknown message");
        }
    }

    void gate() {
        // go[r] = (min over ranks of done) + 1: nobody starts call e+1 before every rank
        // finished call e (IterStart after all IterDone).
        uint64_t lo = ~0ull;
        for (int r = 0; r < world; ++r) lo = page->done[r] < lo ? page->done[r] : lo;
        for (int r = 0; r < world; ++r)
            if (page->go[r] < lo + 1) page->go[r] = lo + 1;
    }

    int run() {
        char name[64];
        std::snprintf(name, sizeof name, "/gdraa_js_%d_%llu", static_cast<int>(getpid()),
                      static_cast<unsigned long long>(now_ms() & 0xFFFFFF));
        shm_name = name;
        int sfd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
        if (sfd < 0) return perror_ret("shm_open");
        if (ftruncate(sfd, 4096) != 0) return perror_ret("ftruncate");
        void *mem = mmap(nullptr, 4096, PROT_READ | PROT_WRITE, MAP_SHARED, sfd, 0);
        ::close(sfd);
        if (mem == MAP_FAILED) return perror_ret("mmap");
        std::memset(mem, 0, 4096);
        page = static_cast<ShmPage *>(mem);
        page->magic = kMagic;
        page->world = world;
        page->gated = gated ? 1 : 0;
        for (int r = 0; r < kMaxRanks; ++r) page->go[r] = 1;

        lfd = ::socket(AF_UNIX, SOCK_STREAM, 0);
        if (lfd < 0) return perror_ret("socket");
        sockaddr_un addr{};
        addr.sun_family = AF_UNIX;
        if (sock_path.size() >= sizeof addr.sun_path) return fail_ret("socket path too long");
        std::snprintf(addr.sun_path, sizeof addr.sun_path, "%s", sock_path.c_str());
        ::unlink(sock_path.c_str());
        if (::bind(lfd, reinterpret_cast<sockaddr *>(&addr), sizeof addr) != 0)
            return perror_ret("bind");
        if (::listen(lfd, 64) != 0) return perror_ret("listen");

        const uint64_t t0 = now_ms();
        while (true) {
            std::vector<pollfd> fds;
            fds.push_back({lfd, POLLIN, 0});
            for (auto &c : clients) fds.push_back({c.gone ? -1 : c.fd, POLLIN, 0});
            int k = ::poll(fds.data(), fds.size(), gated ? 1 : 50);
            if (k < 0 && errno != EINTR) return perror_ret("poll");
            if (gated && hellos == world) gate();
            if (hellos < world && now_ms() - t0 > timeout_ms) {
                failed = true;
                fail_msg = "timeout: only " + std::to_string(hellos) + " of " +
                           std::to_string(world) + " ranks joined";
                broadcast_fail(kEJOBSERVER, fail_msg);
                break;
            }
            if (k <= 0) continue;
            if (fds[0].revents & POLLIN) {
                int cfd = ::accept(lfd, nullptr, nullptr);
                if (cfd >= 0) {
                    Client c;
                    c.fd = cfd;
                    clients.push_back(c);
                }
            }
            for (size_t i = 1; i < fds.size(); ++i) {
                Client &c = clients[i - 1];
                if (c.gone || !(fds[i].revents & (POLLIN | POLLHUP | POLLERR))) continue;
                Hdr h;
                if (!read_all(c.fd, &h, sizeof h)) {
                    drop(c, "EOF");
                    continue;
                }
                if (h.magic != kMagic || h.len > 4096) {
                    drop(c, "bad header");
                    continue;
                }
                std::vector<char> body(h.len);
                if (h.len && !read_all(c.fd, body.data(), h.len)) {
                    drop(c, "EOF in body");
                    continue;
                }
                on_message(c, h, body);
            }
            bool all_gone = !clients.empty();
            for (auto &c : clients) all_gone = all_gone && (c.gone || c.bye);
            if (byes == world || (all_gone && hellos > 0 && failed)) break;
        }
        finish();
        return failed ? 1 : 0;
    }

    void finish() {
        for (auto &c : clients)
            if (!c.gone) ::close(c.fd);
        if (lfd >= 0) ::close(lfd);
        ::unlink(sock_path.c_str());
        char line[512];
        std::snprintf(line, sizeof line,
                      "{\"jobserver\": {\"world\": %d, \"ranks_joined\": %d, \"registrations\": %llu, "
                      "\"control_bytes\": %llu, \"data_bytes\": %llu, \"done\": [",
                      world, hellos, (unsigned long long)page->registrations,
                      (unsigned long long)page->control_bytes,
                      (unsigned long long)page->data_bytes);
        std::string s = line;
        for (int r = 0; r < world; ++r) {
            s += std::to_string(page->done[r]);
            if (r + 1 < world) s += ", ";
        }
        s += "], \"ok\": ";
        s += failed ? "false" : "true";
        s += ", \"error\": \"" + fail_msg + "\"}}";
        std::printf("%s\n", s.c_str());
        std::fflush(stdout);
        if (!stats_path.empty()) {
            FILE *f = std::fopen(stats_path.c_str(), "w");
            if (f) {
                std::fprintf(f, "%s\n", s.c_str());
                std::fclose(f);
            }
        }
        shm_unlink(shm_name.c_str());
    }

    int perror_ret(const char *what) {
        std::fprintf(stderr, "gdraa_jobserver: %s: %s\n", what, std::strerror(errno));
        return 2;
    }
    int fail_ret(const char *what) {
        std::fprintf(stderr, "gdraa_jobserver: %s\n", what);
        return 2;
    }
};

}  // namespace

int main(int argc, char **argv) {
    Server s;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto next = [&](const char *what) -> std::string {
            if (i + 1 >= argc) {
                std::fprintf(stderr, "gdraa_jobserver: %s needs a value\n", what);
                std::exit(2);
            }
            return argv[++i];
        };
        if (a == "--socket") s.sock_path = next("--socket");
        else if (a == "--world") s.world = std::atoi(next("--world").c_str());
        else if (a == "--gated") s.gated = true;
        else if (a == "--timeout-ms") s.timeout_ms = std::strtoull(next("--timeout-ms").c_str(), nullptr, 10);
        else if (a == "--stats") s.stats_path = next("--stats");
        else {
            std::fprintf(stderr, "usage: gdraa_jobserver --socket PATH --world N [--gated] "
                                 "[--timeout-ms T] [--stats FILE]\n");
            return 2;
        }
    }
    if (s.sock_path.empty() || s.world < 1 || s.world > kMaxRanks) {
        std::fprintf(stderr, "gdraa_jobserver: need --socket and --world in [1,%d]\n", kMaxRanks);
        return 2;
    }
    return s.run();
}
