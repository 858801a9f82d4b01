"""Failure handling over real processes (one per GPU; on a one-GPU box both ranks share
it, time-sliced -- tests.conftest.mp_world): a peer that never arrives makes the
kernel give up after GDRAA_TIMEOUT_MS and every later call report GDRAA_ETIMEOUT naming
the missing rank ("peer-timeout ... names the missing ranks"); a peer process that
dies is seen by the job server (socket EOF), whose abort flag -- mapped into the
kernel's spin loops -- ends the wait long before the timeout (GDRAA_EJOBSERVER)."""
import json
import os
import time

import pytest
import torch
import torch.multiprocessing as mp

from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a GPU")]


def _setup(rank, world, sock, timeout_ms, n):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["GDRAA_JOBSERVER"] = sock
    os.environ["GDRAA_TIMEOUT_MS"] = str(timeout_ms)
    from tests.conftest import rank_device
    dev = rank_device(rank)
    from paper_1802_02326_b200 import gdraa
    gdraa.gdraa_init(world, rank)
    w = torch.zeros(n, device=dev)
    g = torch.ones(n, device=dev)
    v = torch.zeros(n, device=dev)
    gdraa.gdraa_register(w)
    gdraa.gdraa_register(g)
    return gdraa, w, g, v


def _timeout_worker(rank, world, sock, out, mode, n):
    # rank 0 gives up after 1.5 s when the peer just skips the call; when the peer dies
    # it keeps a 60 s timeout, so only the job server's abort flag can end its wait early
    gdraa, w, g, v = _setup(rank, world, sock,
                            1500 if rank == 0 and mode in ("skip", "streamed") else 60000, n)
    res = {"rank": rank}
    if rank == 0:
        t0 = time.time()
        if mode == "streamed":
            # one bucket of a streamed set: the persistent kernel's entry wait gives up
            gdraa.gdraa_bucket_set_begin_streamed(8)
            gdraa.gdraa_sgd_step_range(w, g, v, 0, n, 0.1, 0.9)
            gdraa.gdraa_bucket_set_end()
        else:
            gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9)    # the peer never arrives
        torch.cuda.synchronize()                         # kernel gives up after 1.5 s
        res["kernel_s"] = time.time() - t0
        try:
            gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9)
            res["second"] = "ok"
        except gdraa.GdraaError as e:
            res["second"] = e.name
            res["msg"] = str(e)
        try:
            gdraa.gdraa_finalize()
            res["finalize"] = "ok"
        except gdraa.GdraaError as e:
            res["finalize"] = e.name
    else:
        if mode == "die":
            time.sleep(1.0)
            os._exit(3)                                  # dies without finalize
        time.sleep(4.0)                                  # alive, but skips the call
        gdraa.gdraa_finalize()
        res["finalize"] = "ok"
    with open(os.path.join(out, f"r{rank}.json"), "w") as f:
        json.dump(res, f)


def _run(tmp_path, mode, n):
    from paper_1802_02326_b200 import jobserver
    world = 2
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_timeout_worker, args=(r, world, sock, str(tmp_path), mode, n))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    out, err = js.communicate(timeout=60)
    return [p.exitcode for p in procs], json.load(open(tmp_path / "r0.json")), out


# 2^18 fp32 elements take the small-message SGD kernel (data-carried synchronisation),
# 2^21 the two-shot kernel (device barriers): both must time out and abort the same way
SIZES = [1 << 18, 1 << 21]


@pytest.mark.parametrize("n", SIZES)
def test_peer_timeout_names_missing_rank(tmp_path, n):
    codes, r0, _ = _run(tmp_path, "skip", n)
    assert codes == [0, 0], codes
    assert 1.0 < r0["kernel_s"] < 20, r0
    assert r0["second"] == "GDRAA_ETIMEOUT" and "missing rank(s) 1" in r0["msg"], r0
    assert r0["finalize"] == "GDRAA_ETIMEOUT", r0


def test_streamed_set_peer_timeout(tmp_path):
    """The persistent bucket-set kernel gives up like the per-call kernels: the set ends,
    the next call reports GDRAA_ETIMEOUT naming the missing rank."""
    codes, r0, _ = _run(tmp_path, "streamed", 1 << 21)
    assert codes == [0, 0], codes
    assert 1.0 < r0["kernel_s"] < 20, r0
    assert r0["second"] == "GDRAA_ETIMEOUT" and "missing rank(s) 1" in r0["msg"], r0
    assert r0["finalize"] == "GDRAA_ETIMEOUT", r0


@pytest.mark.parametrize("n", SIZES)
def test_dead_rank_aborts_the_wait(tmp_path, n):
    # rank 0's kernel would wait 60 s; the job server's abort flag ends it in seconds
    codes, r0, js_out = _run(tmp_path, "die", n)
    assert codes[1] == 3 and codes[0] == 0, codes
    assert r0["kernel_s"] < 15, r0
    assert r0["second"] == "GDRAA_EJOBSERVER" and "rank 1" in r0["msg"], r0
    assert "disconnected" in js_out


def _mismatch_worker(rank, world, sock, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["GDRAA_JOBSERVER"] = sock
    # rank 1 would serve small steps with the two-shot kernel, rank 0 with the LL kernel
    os.environ["GDRAA_LL_SGD_MAX_BYTES"] = "0" if rank == 1 else str(1 << 20)
    from tests.conftest import rank_device
    rank_device(rank)
    from paper_1802_02326_b200 import gdraa
    res = {"rank": rank}
    try:
        gdraa.gdraa_init(world, rank)
        res["init"] = "ok"
        gdraa.gdraa_finalize()
    except gdraa.GdraaError as e:
        res["init"] = e.name
        res["msg"] = str(e)
    with open(os.path.join(out, f"m{rank}.json"), "w") as f:
        json.dump(res, f)


def test_threshold_mismatch_rejected_at_init(tmp_path):
    """Ranks that would pick different kernels for the same call are refused at
    gdraa_init (GDRAA_ESHAPE on every rank) instead of timing out mid-training."""
    from paper_1802_02326_b200 import jobserver
    world = 2
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_mismatch_worker, args=(r, world, sock, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    js.communicate(timeout=60)
    for r in range(world):
        res = json.load(open(tmp_path / f"m{r}.json"))
        assert res["init"] == "GDRAA_ESHAPE", res
        assert "GDRAA_LL_SGD_MAX_BYTES" in res["msg"], res
