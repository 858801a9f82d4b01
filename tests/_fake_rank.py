"""A Python speaker of the job-server protocol (csrc/jobserver_proto.h) used to test the
control plane on a CPU-only host with fake 64-byte IPC handles."""
import mmap
import os
import socket
import struct
import time

MAGIC = 0x41524447
HELLO, HELLO_OK, REG, REG_OK, REG_ERR, BYE, BYE_OK, FAIL = range(1, 9)
HDR = struct.Struct("<IHHII")
HELLO_S = struct.Struct("<ii16s")
HELLO_OK_S = struct.Struct("<64siiQ")
REG_S = struct.Struct("<QiiQ64s")
FAIL_S = struct.Struct("<i188s")


class FakeRank:
    def __init__(self, path, rank, world, timeout=20.0):
        self.rank, self.world = rank, world
        deadline = time.time() + timeout
        while True:
            try:
                self.sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
                self.sock.connect(path)
                break
            except OSError:
                self.sock.close()
                if time.time() > deadline:
                    raise
                time.sleep(0.02)
        self.sock.settimeout(timeout)

    def send(self, kind, payload=b"", seq=0):
        self.sock.sendall(HDR.pack(MAGIC, kind, self.rank, len(payload), seq) + payload)

    def _recv_exact(self, n):
        buf = b""
        while len(buf) < n:
            chunk = self.sock.recv(n - len(buf))
            if not chunk:
                raise ConnectionError("job server closed the connection")
            buf += chunk
        return buf

    def recv(self):
        magic, kind, rank, ln, seq = HDR.unpack(self._recv_exact(HDR.size))
        assert magic == MAGIC
        return kind, seq, self._recv_exact(ln) if ln else b""

    def hello(self, world=None):
        self.send(HELLO, HELLO_S.pack(self.world if world is None else world, os.getpid(),
                                      bytes(16)))

    def expect_hello_ok(self):
        kind, _, body = self.recv()
        assert kind == HELLO_OK, (kind, body)
        name, world, gated, job = HELLO_OK_S.unpack(body)
        return name.rstrip(b"\0").decode(), world, gated

    def register(self, seq, n, dtype, handle, offset=0, what=1):
        self.send(REG, REG_S.pack(n, dtype, what, offset, handle), seq=seq)

    def recv_reg(self):
        kind, seq, body = self.recv()
        if kind == REG_OK:
            world, _ = struct.unpack_from("<ii", body, 0)
            regs = [REG_S.unpack_from(body, 8 + REG_S.size * i) for i in range(world)]
            return "ok", seq, regs
        code, msg = FAIL_S.unpack(body)
        return ("err" if kind == REG_ERR else "fail"), code, msg.rstrip(b"\0").decode()

    def bye(self):
        self.send(BYE)
        kind, _, _ = self.recv()
        assert kind == BYE_OK
        self.sock.close()


def read_page(shm_name):
    """Fields of proto::ShmPage."""
    with open("/dev/shm/" + shm_name.lstrip("/"), "rb") as f:
        m = mmap.mmap(f.fileno(), 4096, access=mmap.ACCESS_READ)
        magic, world, gated = struct.unpack_from("<Qii", m, 0)
        go = struct.unpack_from("<8Q", m, 16)
        done = struct.unpack_from("<8Q", m, 80)
        abort, dead = struct.unpack_from("<ii", m, 144)
        ctrl, data, regs = struct.unpack_from("<QQQ", m, 152)
        m.close()
    return dict(magic=magic, world=world, gated=gated, go=go, done=done, abort=abort,
                dead_rank=dead, control_bytes=ctrl, data_bytes=data, registrations=regs)
