"""Job-server control plane on the CPU-only host with fake handles:
rendezvous, handle relay, shape-mismatch detection, dead-rank detection, the
go/done page, and the zero-data invariant."""
import json
import os
import subprocess
import threading

import pytest

from paper_1802_02326_b200 import jobserver
from tests._fake_rank import FAIL, FakeRank, read_page


@pytest.fixture
def sock(tmp_path):
    return str(tmp_path / "js.sock")


def _finish(proc):
    out, err = proc.communicate(timeout=30)
    return json.loads(out.strip().splitlines()[-1])["jobserver"], proc.returncode


def _run_ranks(world, sock, body):
    """Run body(rank_client) for every rank concurrently; re-raise the first failure."""
    errs = []

    def run(r):
        try:
            body(FakeRank(sock, r, world))
        except BaseException as e:   # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    if errs:
        raise errs[0]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rendezvous_and_handle_relay(sock, world):
    proc = jobserver.start(world, sock)
    pages = {}

    def body(c):
        c.hello()
        name, w, gated = c.expect_hello_ok()
        assert w == world and gated == 0
        pages[c.rank] = name
        for seq in (1, 2, 3):
            handle = bytes([c.rank, seq]) * 32
            c.register(seq, 1000 * seq, seq % 2, handle, offset=256 * c.rank)
            st, got_seq, regs = c.recv_reg()
            assert st == "ok" and got_seq == seq
            for p, (n, dt, what, off, h) in enumerate(regs):
                assert (n, dt, off, h) == (1000 * seq, seq % 2, 256 * p, bytes([p, seq]) * 32)
        c.bye()

    _run_ranks(world, sock, body)
    stats, rc = _finish(proc)
    assert rc == 0 and stats["ok"]
    assert stats["ranks_joined"] == world and stats["registrations"] == 3
    assert stats["data_bytes"] == 0 and stats["control_bytes"] > 0
    assert len(set(pages.values())) == 1


def test_shape_mismatch_reported_to_every_rank(sock):
    world = 3
    proc = jobserver.start(world, sock)
    seen = {}

    def body(c):
        c.hello()
        c.expect_hello_ok()
        n = 1000 if c.rank != 2 else 999           # rank 2 disagrees on L
        c.register(1, n, 0, bytes(64))
        seen[c.rank] = c.recv_reg()
        c.bye()

    _run_ranks(world, sock, body)
    _finish(proc)
    for r in range(world):
        st, code, msg = seen[r]
        assert st == "err" and code == -3 and "shape mismatch" in msg, seen[r]
        assert "r2(n=999" in msg


def test_world_mismatch_rejected(sock):
    proc = jobserver.start(2, sock, timeout_ms=3000)
    c = FakeRank(sock, 0, 2)
    c.hello(world=4)
    kind, _, body = c.recv()
    assert kind == FAIL
    stats, rc = _finish(proc)
    assert rc != 0 and not stats["ok"]


def test_dead_rank_detected(sock):
    world = 2
    proc = jobserver.start(world, sock)
    a, b = FakeRank(sock, 0, world), FakeRank(sock, 1, world)
    a.hello()
    b.hello()
    name, _, _ = a.expect_hello_ok()
    b.expect_hello_ok()
    b.sock.close()                                  # rank 1 dies before registering
    a.register(1, 10, 0, bytes(64))
    st, code, msg = a.recv_reg()
    assert st == "fail" and code == -7 and "rank 1" in msg
    a.sock.close()
    stats, rc = _finish(proc)
    assert rc != 0 and "rank 1" in stats["error"]


def test_pre_hello_connection_does_not_abort(sock):
    """A connection that closes before HELLO (readiness probe, stale rank of an earlier
    job) is not a rank: the job goes on and ends cleanly."""
    import socket as s
    world = 2
    proc = jobserver.start(world, sock)
    a = FakeRank(sock, 0, world)                   # waits until the server is up
    probe = s.socket(s.AF_UNIX, s.SOCK_STREAM)
    probe.connect(sock)
    probe.close()                                   # connect + close, no HELLO
    b = FakeRank(sock, 1, world)
    a.hello()
    b.hello()
    name, _, _ = a.expect_hello_ok()
    b.expect_hello_ok()
    a.register(1, 10, 0, bytes(64))
    b.register(1, 10, 0, bytes(64))
    assert a.recv_reg()[0] == "ok" and b.recv_reg()[0] == "ok"
    assert read_page(name)["abort"] == 0
    a.send(6)
    b.send(6)
    assert a.recv()[0] == 7 and b.recv()[0] == 7
    stats, rc = _finish(proc)
    assert rc == 0 and stats["ok"] and stats["data_bytes"] == 0


def test_data_bytes_counts_non_control_payload(sock):
    """data_bytes is a guard, not a constant: a message outside the control vocabulary
    (here a would-be 4 KiB tensor payload) is counted and its sender dropped, which
    fails the job for every rank (the job server moves no weight data)."""
    world = 2
    proc = jobserver.start(world, sock)
    a, b = FakeRank(sock, 0, world), FakeRank(sock, 1, world)
    a.hello()
    b.hello()
    name, _, _ = a.expect_hello_ok()
    b.expect_hello_ok()
    b.send(42, bytes(4096))                         # not a control message
    kind, _, _ = a.recv()
    assert kind == FAIL
    page = read_page(name)
    assert page["data_bytes"] == 4096 and page["abort"] == 1 and page["dead_rank"] == 1
    a.sock.close()
    b.sock.close()
    stats, rc = _finish(proc)
    assert rc != 0 and stats["data_bytes"] == 4096


def test_go_done_page(sock):
    """The shared page the kernels write done[r] into (S:95 IterDone); in gated mode
    the job server raises go[r] = min(done) + 1 (IterStart)."""
    world = 2
    proc = jobserver.start(world, sock, gated=True)
    a, b = FakeRank(sock, 0, world), FakeRank(sock, 1, world)
    a.hello()
    b.hello()
    name, _, gated = a.expect_hello_ok()
    b.expect_hello_ok()
    assert gated == 1
    page = read_page(name)
    assert page["world"] == world and page["go"][:2] == (1, 1) and page["data_bytes"] == 0
    # emulate the kernels' last CTA writing done[r] through the host mapping
    import mmap
    import struct
    import time
    with open("/dev/shm/" + name.lstrip("/"), "r+b") as f:
        m = mmap.mmap(f.fileno(), 4096)
        struct.pack_into("<Q", m, 80, 1)            # done[0] = 1
        time.sleep(0.05)
        assert read_page(name)["go"][:2] == (1, 1)  # rank 1 not done yet
        struct.pack_into("<Q", m, 88, 1)            # done[1] = 1
        deadline = time.time() + 5
        while read_page(name)["go"][:2] != (2, 2) and time.time() < deadline:
            time.sleep(0.01)
        assert read_page(name)["go"][:2] == (2, 2)
        m.close()
    a.send(6)
    b.send(6)
    assert a.recv()[0] == 7 and b.recv()[0] == 7
    stats, rc = _finish(proc)
    assert rc == 0 and stats["done"] == [1, 1] and stats["data_bytes"] == 0


def test_jobserver_links_no_cuda():
    """It cannot touch weight data: no CUDA runtime or driver library is linked."""
    out = subprocess.run(["ldd", jobserver.BINARY], capture_output=True, text=True).stdout
    assert "libcuda" not in out and "libcudart" not in out, out
    syms = subprocess.run(["nm", "-D", jobserver.BINARY], capture_output=True, text=True).stdout
    assert "cudaIpcOpenMemHandle" not in syms and "cuIpc" not in syms


def _gloo_rank(rank, world, sock, port, n, out):
    import torch.distributed as dist
    from paper_1802_02326_b200 import gdraa
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    c = FakeRank(sock, rank, world)
    c.hello()
    c.expect_hello_ok()
    c.register(1, n, 0, bytes([rank + 1]) * 64, offset=rank * 16)
    st, _, regs = c.recv_reg()
    assert st == "ok"
    shard = gdraa.gdraa_shard(world, rank, n)
    table = [None] * world
    dist.all_gather_object(table, {"regs": [(r[0], r[3], r[4]) for r in regs], "shard": shard})
    c.bye()
    dist.destroy_process_group()
    if rank == 0:
        with open(out, "w") as f:
            json.dump([{"regs": [(a, b, h.hex()) for a, b, h in t["regs"]], "shard": t["shard"]}
                       for t in table], f)


def test_two_process_gloo_host_path(sock, tmp_path):
    """world_size-2 multi-process host path on CPU (gloo): both ranks see the same
    relayed handle table, and their gdraa_shard() blocks tile [0, n)."""
    import socket as s
    import torch.multiprocessing as mp
    world, n = 2, 1_000_003
    with s.socket() as t:
        t.bind(("127.0.0.1", 0))
        port = t.getsockname()[1]
    proc = jobserver.start(world, sock)
    out = str(tmp_path / "table.json")
    mp.start_processes(_gloo_rank, args=(world, sock, port, n, out), nprocs=world, join=True,
                       start_method="spawn")
    stats, rc = _finish(proc)
    assert rc == 0 and stats["data_bytes"] == 0
    table = json.load(open(out))
    assert table[0]["regs"] == table[1]["regs"]
    assert [r[2] for r in table[0]["regs"]] == [bytes([p + 1]).hex() * 64 for p in range(world)]
    shards = sorted(tuple(t["shard"]) for t in table)
    assert shards[0][0] == 0 and shards[0][0] + shards[0][1] == shards[1][0]
    assert shards[1][0] + shards[1][1] == n
    assert os.path.exists(jobserver.BINARY)
