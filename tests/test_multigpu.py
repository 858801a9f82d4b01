"""Multi-process parity over NVLink: one process per GPU, job server control plane,
CUDA-IPC peer mappings, the fused kernel pulling/pushing peer memory.  Runs with
world = number of visible GPUs (2 or 4 under `gpurun --gpus N`) over NVLink; on a one-GPU
box (the driver's round-end configuration) with world 2, both ranks on the one GPU as
separate processes and CUDA contexts, time-sliced (tests.conftest.mp_world): no NVLink,
but every other part of the multi-process path -- job server, IPC mappings of
caching-allocator blocks, cross-process release/acquire flags, bulk copies from
IPC-mapped addresses, IterDone/IterStart -- runs as it does across GPUs."""
import json
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from tests.conftest import has_cuda, mp_world

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a GPU")]


def _worker(rank, world, sock, L_list, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1802_02326_b200 import gdraa
    from tests._parity import compare
    from tests.test_gpu_parity import from_dev, make_grads, to_dev

    from tests.conftest import rank_device
    dev = rank_device(rank)
    os.environ["GDRAA_JOBSERVER"] = sock
    gdraa.gdraa_init(world, rank)
    report = {"rank": rank, "cases": 0}
    calls = 0
    for L in L_list:
        for dt in ("f32", "bf16"):
            bf16 = dt == "bf16"
            for family in ("int", "like"):
                gs = make_grads(family, 31 + L % 97, world, L, bf16)
                # allreduce_mean (in place, registered buffer)
                buf = to_dev(gs[rank], bf16, dev)
                gdraa.gdraa_register(buf)
                gdraa.gdraa_allreduce_mean(buf)
                calls += 1
                torch.cuda.synchronize()
                compare(from_dev(buf), oracle.allreduce_mean(gs), dt,
                        what=f"mean L={L} {dt} {family} rank {rank}")
                # fused sgd_step, 3 chained iterations
                if family == "int":
                    w0, v0, lr, mom = (synth.w_integer(5, L), synth.v_integer(5, L),
                                       synth.INT_LR, synth.INT_MOM)
                else:
                    w0, v0, lr, mom = (synth.w_like(5, L), np.zeros(L, np.float32),
                                       synth.PAPER_LR, synth.PAPER_MOM)
                g = to_dev(gs[rank], bf16, dev)
                w, v = to_dev(w0, dev=dev), to_dev(v0, dev=dev)
                gdraa.gdraa_register(w)
                gdraa.gdraa_register(g)
                off, ln = gdraa.gdraa_shard(world, rank, L)
                for it in range(3 if family == "like" else 1):
                    w0, v0 = oracle.sgd_step(gs, w0, v0, lr, mom)
                    gdraa.gdraa_sgd_step(w, g, v, lr, mom)
                    calls += 1
                    torch.cuda.synchronize()
                    compare(from_dev(w), w0, "f32", what=f"w it{it} L={L} {dt} {family} r{rank}")
                    compare(from_dev(v)[off:off + ln], v0[off:off + ln], "f32",
                            what=f"v it{it} L={L} {dt} {family} r{rank}")
                assert np.array_equal(from_dev(g), gs[rank])     # g read-only (AMB-18)
                # NEXT-1: weight decay and the mixed-precision all-gather (bf16 model copy)
                w0, v0 = synth.w_like(6, L), synth.w_like(7, L)
                we, ve, me = oracle.sgd_step_wd(gs, w0, v0, lr, mom, 0.001,
                                                model_dtype=oracle.BF16)
                wm, vm = to_dev(w0, dev=dev), to_dev(v0, dev=dev)
                model = torch.zeros(L, dtype=torch.bfloat16, device=dev)
                gdraa.gdraa_register(model)
                gdraa.gdraa_sgd_step_mp(wm, model, g, vm, lr, mom, 0.001)
                calls += 1
                torch.cuda.synchronize()
                compare(from_dev(model), me, "bf16", what=f"mp model L={L} {dt} {family} r{rank}")
                compare(from_dev(wm)[off:off + ln], we[off:off + ln], "f32", what="mp master")
                compare(from_dev(vm)[off:off + ln], ve[off:off + ln], "f32", what="mp v")
                w2, v2 = to_dev(w0, dev=dev), to_dev(v0, dev=dev)
                gdraa.gdraa_register(w2)
                gdraa.gdraa_sgd_step_ex(w2, g, v2, lr, mom, 0.001)
                calls += 1
                torch.cuda.synchronize()
                compare(from_dev(w2), we, "f32", what=f"ex w L={L} {dt} {family} r{rank}")
                compare(from_dev(v2)[off:off + ln], ve[off:off + ln], "f32", what="ex v")
                for t in (model, w2):
                    gdraa.gdraa_deregister(t)
                for t in (buf, w, g):
                    gdraa.gdraa_deregister(t)
                report["cases"] += 1
    st = gdraa.gdraa_get_stats()
    assert st["calls"] == calls, (st, calls)
    # exactly two device synchronisations per call; small calls take the latency
    # paths, whose synchronisation travels with the data (NEXT-2)
    lim = gdraa.gdraa_small_message_bytes(world)
    small = 0
    for L in L_list:
        for es, code in ((4, gdraa.GDRAA_F32), (2, gdraa.GDRAA_BF16)):
            step = L * es <= gdraa.gdraa_small_step_bytes(world, code)
            step_mp = L * es <= gdraa.gdraa_small_step_bytes(world, code, mixed=True)
            small += 2 * (L * es <= lim)                       # mean, both families
            small += (1 + 3) * step                            # sgd: int 1 + like 3 steps
            small += 2 * step_mp + 2 * step                    # mp and ex, both families
    assert st["ll_calls"] == small, (st, small)
    assert st["sync_waits"] == 2 * (calls - st["ll_calls"]), st
    # a0: the kernel's last CTA wrote IterDone = calls completed into the job server's page
    assert st["iter_done"] == calls, (st, calls)
    report["stats"] = st
    report["calls"] = calls
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(report, f)


def test_multiprocess_parity(tmp_path):
    from paper_1802_02326_b200 import jobserver
    world = mp_world()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    L_list = [1, 1000, 70_001, 1 << 20]
    try:
        mp.start_processes(_worker, args=(world, sock, L_list, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        out, err = js.communicate(timeout=120)
    line = json.loads(out.strip().splitlines()[-1])["jobserver"]
    assert line["ok"] and line["data_bytes"] == 0, line
    assert line["ranks_joined"] == world
    reps = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    for rep in reps:
        assert rep["cases"] == len(L_list) * 4
    # the job server saw every rank's IterDone reach the number of calls
    assert line["done"] == [reps[0]["calls"]] * world, line


def _gated_worker(rank, world, sock, out_dir):
    """Gated mode (IterStart): every call waits on the host until the job server
    raised go[rank] to its call number, i.e. until every rank finished the previous call.
    Mixed small (LL) and two-shot steps, chained; bit-exact against the oracle."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1802_02326_b200 import gdraa
    from tests._parity import compare
    from tests.test_gpu_parity import from_dev, make_grads, to_dev

    from tests.conftest import rank_device
    dev = rank_device(rank)
    os.environ["GDRAA_JOBSERVER"] = sock
    gdraa.gdraa_init(world, rank)
    calls = 0
    for L in (1000, 1 << 20, 3_000_017):
        gs = make_grads("like", 71, world, L, False)
        w0, v0 = synth.w_like(71, L), np.zeros(L, np.float32)
        g = to_dev(gs[rank], dev=dev)
        w, v = to_dev(w0, dev=dev), to_dev(v0, dev=dev)
        gdraa.gdraa_register(w)
        gdraa.gdraa_register(g)
        off, ln = gdraa.gdraa_shard(world, rank, L)
        for it in range(4):
            w0, v0 = oracle.sgd_step(gs, w0, v0, 0.1, 0.9)
            gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9)
            calls += 1
            st = gdraa.gdraa_get_stats()           # synchronises: IterDone of this call
            assert st["iter_done"] == calls and st["iter_start"] >= calls, (st, calls)
        compare(from_dev(w), w0, "f32", what=f"gated w L={L} r{rank}")
        compare(from_dev(v)[off:off + ln], v0[off:off + ln], "f32", what=f"gated v r{rank}")
        gdraa.gdraa_deregister(w)
        gdraa.gdraa_deregister(g)
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"gated{rank}.json"), "w") as f:
        json.dump({"calls": calls}, f)


def test_multiprocess_gated(tmp_path):
    from paper_1802_02326_b200 import jobserver
    world = mp_world()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock, gated=True)
    try:
        mp.start_processes(_gated_worker, args=(world, sock, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        out, err = js.communicate(timeout=120)
    line = json.loads(out.strip().splitlines()[-1])["jobserver"]
    calls = [json.load(open(tmp_path / f"gated{r}.json"))["calls"] for r in range(world)]
    assert line["ok"] and line["data_bytes"] == 0 and line["done"] == calls, line


BUCKETS = [(600_000, 400_000), (0, 600_000), (1_000_000, 48_576)]   # backward order


def _bucket_worker(rank, world, sock, out_dir):
    """NEXT-3: the gradient buffer reduced and applied bucket by bucket (last layers
    first, as a backward pass produces them) on a side stream; w must equal the
    whole-buffer oracle step and v the oracle on every rank's per-bucket shards."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1802_02326_b200 import gdraa
    from tests._parity import compare
    from tests.test_gpu_parity import from_dev, make_grads, to_dev

    from tests.conftest import rank_device
    dev = rank_device(rank)
    os.environ["GDRAA_JOBSERVER"] = sock
    gdraa.gdraa_init(world, rank)
    L = 1_048_576
    side = torch.cuda.Stream()
    for dt in ("f32", "bf16"):
        bf16 = dt == "bf16"
        gs = make_grads("like", 61, world, L, bf16)
        w0, v0 = synth.w_like(61, L), synth.w_like(62, L)
        w_exp, v_exp = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
        g = to_dev(gs[rank], bf16, dev)
        w, v = to_dev(w0, dev=dev), to_dev(v0, dev=dev)
        gdraa.gdraa_register(w)
        gdraa.gdraa_register(g)
        done = torch.cuda.Event()
        for first, count in BUCKETS:
            done.record(torch.cuda.current_stream())     # "the bucket's gradient is ready"
            side.wait_event(done)
            gdraa.gdraa_sgd_step_range(w, g, v, first, count, 0.1, 0.9, 0.001, stream=side)
        side.synchronize()
        compare(from_dev(w), w_exp, "f32", what=f"bucketed w {dt} r{rank}")
        vh = from_dev(v)
        for first, count in BUCKETS:
            off, ln = gdraa.gdraa_shard(world, rank, count)
            a, b = first + off, first + off + ln
            compare(vh[a:b], v_exp[a:b], "f32", what=f"bucketed v {dt} r{rank}")
        # allreduce_mean on the same buckets (both the LL and the two-shot sizes)
        buf = to_dev(gs[rank], bf16, dev)
        gdraa.gdraa_register(buf)
        for first, count in BUCKETS:
            gdraa.gdraa_allreduce_mean_range(buf, first, count, stream=side)
        side.synchronize()
        compare(from_dev(buf), oracle.allreduce_mean(gs), dt, what=f"bucketed mean {dt}")
        for t in (w, g, buf):
            gdraa.gdraa_deregister(t)
    # a bucket set (NEXT-3, "two syncs per bucket-set"): the two-shot buckets skip their
    # exit barrier, gdraa_bucket_set_end runs one for the set; two chained iterations
    L2 = 6_048_576
    set_buckets = [(3_000_000, 3_000_000), (6_000_000, 48_576), (0, 3_000_000)]
    for dt in ("f32", "bf16"):
        bf16 = dt == "bf16"
        es = 2 if bf16 else 4
        gs = make_grads("like", 63, world, L2, bf16)
        w0, v0 = synth.w_like(63, L2), synth.w_like(64, L2)
        w1, v1 = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
        w2, v2 = oracle.sgd_step_wd(gs, w1, v1, 0.1, 0.9, 0.001)
        g = to_dev(gs[rank], bf16, dev)
        w, v = to_dev(w0, dev=dev), to_dev(v0, dev=dev)
        gdraa.gdraa_register(w)
        gdraa.gdraa_register(g)
        lim = gdraa.gdraa_small_step_bytes(world, gdraa.GDRAA_BF16 if bf16 else gdraa.GDRAA_F32)
        two_shot = sum(c * es > lim for _, c in set_buckets)
        assert 0 < two_shot < len(set_buckets)
        st0 = gdraa.gdraa_get_stats()
        for it in range(2):
            gdraa.gdraa_bucket_set_begin()
            for first, count in set_buckets:
                done = torch.cuda.Event()
                done.record(torch.cuda.current_stream())
                side.wait_event(done)
                gdraa.gdraa_sgd_step_range(w, g, v, first, count, 0.1, 0.9, 0.001, stream=side)
            gdraa.gdraa_bucket_set_end(stream=side)
            torch.cuda.current_stream().wait_stream(side)
            if it == 0:
                torch.cuda.synchronize()
                compare(from_dev(w), w1, "f32", what=f"set w it0 {dt} r{rank}")
        torch.cuda.synchronize()
        compare(from_dev(w), w2, "f32", what=f"set w it1 {dt} r{rank}")
        vh = from_dev(v)
        for first, count in set_buckets:
            off, ln = gdraa.gdraa_shard(world, rank, count)
            a, b = first + off, first + off + ln
            compare(vh[a:b], v2[a:b], "f32", what=f"set v {dt} r{rank}")
        st1 = gdraa.gdraa_get_stats()
        # per set: one entry barrier per two-shot bucket + the set's single exit barrier
        assert st1["sync_waits"] - st0["sync_waits"] == 2 * (two_shot + 1), (st0, st1)
        # the same two iterations as streamed sets (one persistent kernel per set)
        w.copy_(torch.from_numpy(w0).to(dev))
        v.copy_(torch.from_numpy(v0).to(dev))
        for it in range(2):
            gdraa.gdraa_bucket_set_begin_streamed(16)
            for first, count in set_buckets:
                done = torch.cuda.Event()
                done.record(torch.cuda.current_stream())
                side.wait_event(done)
                gdraa.gdraa_sgd_step_range(w, g, v, first, count, 0.1, 0.9, 0.001, stream=side)
            gdraa.gdraa_bucket_set_end(stream=side)
            torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        compare(from_dev(w), w2, "f32", what=f"streamed set w {dt} r{rank}")
        vh = from_dev(v)
        for first, count in set_buckets:
            off, ln = gdraa.gdraa_shard(world, rank, count)
            a, b = first + off, first + off + ln
            compare(vh[a:b], v2[a:b], "f32", what=f"streamed set v {dt} r{rank}")
        st2 = gdraa.gdraa_get_stats()
        n_b = len(set_buckets)
        assert st2["calls"] - st1["calls"] == 2 * n_b, (st1, st2)
        assert st2["sync_waits"] - st1["sync_waits"] == 2 * (n_b + 1), (st1, st2)
        assert st2["launches"] - st1["launches"] == 2, (st1, st2)     # one kernel per set
        assert st2["iter_done"] == st2["calls"], st2
        for t in (w, g):
            gdraa.gdraa_deregister(t)
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"bucket{rank}.ok"), "w") as f:
        f.write("ok")


def test_multiprocess_bucketed_ranges(tmp_path):
    from paper_1802_02326_b200 import jobserver
    world = mp_world()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    try:
        mp.start_processes(_bucket_worker, args=(world, sock, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        js.communicate(timeout=120)
    assert all((tmp_path / f"bucket{r}.ok").exists() for r in range(world))


def _open_set_worker(rank, world, sock, out_dir):
    """Rank 0 closes its bucket set; every other rank calls gdraa_finalize with the set
    still open, which must run the deferred exit barrier so that rank 0's completes."""
    import sys
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1802_02326_b200 import gdraa
    from tests.conftest import rank_device

    dev = rank_device(rank)
    os.environ["GDRAA_JOBSERVER"] = sock
    os.environ["GDRAA_TIMEOUT_MS"] = "20000"
    gdraa.gdraa_init(world, rank)
    L = 4_000_000                                      # two-shot at every world size
    w = torch.zeros(L, device=dev)
    g = torch.ones(L, device=dev)
    v = torch.zeros(L, device=dev)
    gdraa.gdraa_register(w)
    gdraa.gdraa_register(g)
    gdraa.gdraa_bucket_set_begin()
    gdraa.gdraa_sgd_step_range(w, g, v, 0, L, 0.5, 0.0)
    t0 = time.time()
    if rank == 0:
        gdraa.gdraa_bucket_set_end()
        torch.cuda.synchronize()
        assert bool((w == -0.5).all())
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"open{rank}.json"), "w") as f:
        json.dump({"s": time.time() - t0}, f)


def test_finalize_closes_an_open_bucket_set(tmp_path):
    from paper_1802_02326_b200 import jobserver
    world = mp_world()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    try:
        mp.start_processes(_open_set_worker, args=(world, sock, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        out, _ = js.communicate(timeout=120)
    line = json.loads(out.strip().splitlines()[-1])["jobserver"]
    assert line["ok"], line
    for r in range(world):
        assert json.load(open(tmp_path / f"open{r}.json"))["s"] < 15


def _ls_worker(rank, world, sock, out_dir):
    """NEXT-4 over real processes: each rank computes its own b-sample least-squares
    gradient and steps through gdraa_sgd_step; rank 0 checks the serial trajectory."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1802_02326_b200 import gdraa
    from synth.least_squares import Problem
    from tests.test_gpu_training import serial_trajectory

    from tests.conftest import rank_device
    dev = rank_device(rank)
    os.environ["GDRAA_JOBSERVER"] = sock
    gdraa.gdraa_init(world, rank)
    P = Problem(seed=5)
    b, lr, mom, iters = 8, 0.05, 0.9, 100
    ref = serial_trajectory(P, iters, world, b, lr, mom)
    w = torch.zeros(P.d, device=dev)
    g = torch.zeros(P.d, device=dev)
    v = torch.zeros(P.d, device=dev)
    gdraa.gdraa_register(w)
    gdraa.gdraa_register(g)
    gap = 0.0
    for it in range(iters):
        X, y = P.batch(it, world, b, rank=rank)
        Xt = torch.from_numpy(X.astype(np.float32)).to(dev)
        yt = torch.from_numpy(y.astype(np.float32)).to(dev)
        g.copy_(Xt.T @ (Xt @ w - yt) / b)
        gdraa.gdraa_sgd_step(w, g, v, lr, mom)
        gap = max(gap, float(np.max(np.abs(w.cpu().numpy() - ref[it]))))
    final = w.cpu().numpy()
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"ls{rank}.json"), "w") as f:
        json.dump({"gap": gap, "w": final.view(np.uint32).tolist()}, f)


def test_multiprocess_least_squares_ssgd(tmp_path):
    from paper_1802_02326_b200 import jobserver
    world = mp_world()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    try:
        mp.start_processes(_ls_worker, args=(world, sock, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        js.communicate(timeout=120)
    reps = [json.load(open(tmp_path / f"ls{r}.json")) for r in range(world)]
    assert all(r["gap"] < 1e-5 for r in reps), [r["gap"] for r in reps]
    assert all(r["w"] == reps[0]["w"] for r in reps)      # bitwise identical replicas


# ---------------------------------------------------------------------------------------
# Full BASELINE sizes in bench.py's launch configuration (one process per GPU, the public
# calls, the two-shot kernel), compared with the oracle on sampled windows: the oracle is
# elementwise, so a window of every rank's gradient (regenerated from synth's
# counter-based streams) and of w/v reproduces the exact expected bits there.
# ---------------------------------------------------------------------------------------
FULL = [("r50", "f32", False), ("r101", "f32", False), ("r50", "bf16", False),
        ("r50", "bf16", True)]
WIN = 4096


def _windows(L, world, seed):
    import synth
    from paper_1802_02326_b200 import gdraa
    starts = {0, L - WIN, synth.neg_zero_segment(seed, L) * synth.SEGMENT}
    for r in range(1, world):                      # every shard boundary
        off, _ = gdraa.gdraa_shard(world, r, L)
        starts.add(max(0, off - WIN // 2))
    rng = np.random.default_rng(seed)
    starts.update(int(x) for x in rng.integers(0, L - WIN, 8))
    return sorted(min(max(0, s), L - WIN) for s in starts)


def _window_grads(seed, world, a, L, bf16):
    import synth
    k = synth.neg_zero_segment(seed, L) * synth.SEGMENT
    out = []
    for p in range(world):
        g = synth.grad_like(seed, p, WIN, start=a)
        lo, hi = max(a, k), min(a + WIN, k + synth.SEGMENT)   # the all-ranks -0.0 segment
        if lo < hi:
            g[lo - a:hi - a] = np.float32(-0.0)
        out.append(synth.to_bf16_bits_trunc(g) if bf16 else g)
    return out


def _full_worker(rank, world, sock, out_dir, configs=None):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1802_02326_b200 import gdraa
    from tests._parity import compare
    from tests.test_gpu_parity import from_dev, to_dev

    from tests.conftest import rank_device
    dev = rank_device(rank)
    os.environ["GDRAA_JOBSERVER"] = sock
    gdraa.gdraa_init(world, rank)
    lr, mom, wd = synth.PAPER_LR, synth.PAPER_MOM, 0.001
    checked = 0
    for name, dt, mp_ in (configs or FULL):
        L = synth.L_R50 if name == "r50" else synth.L_R101
        bf16 = dt == "bf16"
        assert L * (2 if bf16 else 4) > gdraa.gdraa_small_step_bytes(world)   # two-shot
        off, ln = gdraa.gdraa_shard(world, rank, L)
        w0 = synth.w_like(3, L)
        w = to_dev(w0, dev=dev)
        v = torch.zeros(L, device=dev)
        model = torch.zeros(L, dtype=torch.bfloat16, device=dev) if mp_ else None
        gdraa.gdraa_register(model if mp_ else w)
        wins = _windows(L, world, 40)
        state = {a: (w0[a:a + WIN].copy(), np.zeros(WIN, np.float32)) for a in wins}
        for it in range(2):                                # two chained steps
            seed = 40 + it
            gh = synth.grad_like_full(seed, rank, L)
            g = to_dev(synth.to_bf16_bits_trunc(gh) if bf16 else gh, bf16, dev)
            del gh
            gdraa.gdraa_register(g)
            if mp_:
                gdraa.gdraa_sgd_step_mp(w, model, g, v, lr, mom, wd)
            else:
                gdraa.gdraa_sgd_step(w, g, v, lr, mom)
            torch.cuda.synchronize()
            wh, vh = from_dev(w), from_dev(v)
            mh = from_dev(model) if mp_ else None
            for a in wins:
                gs = _window_grads(seed, world, a, L, bf16)
                if mp_:
                    we, ve, me = oracle.sgd_step_wd(gs, *state[a], lr, mom, wd,
                                                    model_dtype=oracle.BF16)
                    compare(mh[a:a + WIN], me, "bf16", what=f"{name} mp model it{it} @{a} r{rank}")
                else:
                    we, ve = oracle.sgd_step(gs, *state[a], lr, mom)
                    compare(wh[a:a + WIN], we, "f32", what=f"{name} {dt} w it{it} @{a} r{rank}")
                # owner-sharded state (v, and the fp32 master for _mp): owned indices only
                lo, hi = max(a, off), min(a + WIN, off + ln)
                if lo < hi:
                    compare(vh[lo:hi], ve[lo - a:hi - a], "f32", what=f"{name} v @{a} r{rank}")
                    if mp_:
                        compare(wh[lo:hi], we[lo - a:hi - a], "f32", what=f"{name} master r{rank}")
                state[a] = (we, ve)
                checked += WIN
            gdraa.gdraa_deregister(g)
            del g
        gdraa.gdraa_deregister(model if mp_ else w)
        del w, v, model
        torch.cuda.empty_cache()
    st = gdraa.gdraa_get_stats()
    assert st["ll_calls"] == 0 and st["sync_waits"] == 2 * st["calls"], st
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"full{rank}.json"), "w") as f:
        json.dump({"checked": checked}, f)


def test_multiprocess_full_size_sampled(tmp_path):
    """Configs 2, 3, 4 (+ NEXT-1) at full size through the multi-process path, two chained
    steps, bit-exact on windows at every shard boundary, the ragged end, the all-ranks
    -0.0 segment (AMB-3) and random places."""
    from paper_1802_02326_b200 import jobserver
    world = mp_world()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    try:
        mp.start_processes(_full_worker, args=(world, sock, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        js.communicate(timeout=120)
    for r in range(world):
        assert json.load(open(tmp_path / f"full{r}.json"))["checked"] > 0


def _c5_worker(rank, world, sock, out_dir):
    """Config 5 sizes through the multi-process path: allreduce_mean of fp32 buffers of
    2^k bytes, k = 10..30 (the small-message kernel below its threshold, the two-shot
    kernel above), against the oracle -- whole buffers up to 4 MiB, sampled windows at
    every shard boundary, the ragged end, the all-ranks -0.0 segment and random places
    above."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1802_02326_b200 import gdraa
    from tests._parity import compare
    from tests.test_gpu_parity import from_dev, to_dev

    from tests.conftest import rank_device
    dev = rank_device(rank)
    os.environ["GDRAA_JOBSERVER"] = sock
    gdraa.gdraa_init(world, rank)
    checked = 0
    for k in range(10, 31):
        L = (1 << k) // 4
        seed = 500 + k
        gh = synth.grad_like_full(seed, rank, L)
        buf = to_dev(gh, dev=dev)
        del gh
        gdraa.gdraa_register(buf)
        gdraa.gdraa_allreduce_mean(buf)
        torch.cuda.synchronize()
        if L <= (1 << 20):
            gs = [synth.grad_like_full(seed, p, L) for p in range(world)]
            compare(from_dev(buf), oracle.allreduce_mean(gs), "f32", what=f"c5 2^{k} B r{rank}")
            checked += L
        else:
            for a in _windows(L, world, seed):
                got = from_dev(buf[a:a + WIN])
                compare(got, oracle.allreduce_mean(_window_grads(seed, world, a, L, False)),
                        "f32", what=f"c5 2^{k} B @{a} r{rank}")
                checked += WIN
        gdraa.gdraa_deregister(buf)
        del buf
        torch.cuda.empty_cache()
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"c5_{rank}.json"), "w") as f:
        json.dump({"checked": checked}, f)


def test_multiprocess_config5_sizes(tmp_path):
    """Config 5 (allreduce message-size sweep 1 KiB - 1 GiB) bit-exact against the oracle
    through the multi-process path at every size of the sweep."""
    from paper_1802_02326_b200 import jobserver
    world = mp_world()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    try:
        mp.start_processes(_c5_worker, args=(world, sock, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        js.communicate(timeout=300)
    for r in range(world):
        assert json.load(open(tmp_path / f"c5_{r}.json"))["checked"] > 0


def test_multiprocess_config4_world8(tmp_path):
    """Config 4 as BASELINE.json states it -- ResNet-50 bf16 gradients, fp32 accumulation
    and master weights, 8 ranks -- at full size through the multi-process path (+ the
    NEXT-1 bf16 model-copy form), two chained steps, sampled windows bit-exact against the
    oracle.  Eight processes on whatever GPUs the box has (time-sliced when fewer than 8)."""
    from paper_1802_02326_b200 import jobserver
    world = 8
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    cfg = [("r50", "bf16", False), ("r50", "bf16", True)]
    try:
        mp.start_processes(_full_worker, args=(world, sock, str(tmp_path), cfg), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        out, _ = js.communicate(timeout=300)
    line = json.loads(out.strip().splitlines()[-1])["jobserver"]
    assert line["ok"] and line["ranks_joined"] == 8 and line["data_bytes"] == 0, line
    for r in range(world):
        assert json.load(open(tmp_path / f"full{r}.json"))["checked"] > 0


# ---------------------------------------------------------------------------------------
# World 8 on fewer GPUs: two or more ranks per GPU (all eight on a one-GPU box), each its
# own process and CUDA context, time-sliced by the GPU.  It runs the whole N = 8
# multi-process path -- job server with 8 ranks, 7 IPC peers per registration (same-GPU
# and cross-GPU), 8-way barriers, the LL slots at N = 8 -- on any box (17 s on one GPU,
# profiles/r76_pytest_world8_one_gpu.log).
# ---------------------------------------------------------------------------------------

def _over_worker(rank, world, ndev, sock, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1802_02326_b200 import gdraa
    from tests._parity import compare
    from tests.test_gpu_parity import from_dev, make_grads, to_dev

    d = rank % ndev
    torch.cuda.set_device(d)
    dev = f"cuda:{d}"
    os.environ["GDRAA_JOBSERVER"] = sock
    gdraa.gdraa_init(world, rank)
    calls = 0
    for L in (1000, 70_001, 1 << 20, 3_000_017):       # LL and two-shot paths at N = 8
        for bf16 in (False, True):
            gs = make_grads("like", 81 + L % 89, world, L, bf16)
            dt = "bf16" if bf16 else "f32"
            buf = to_dev(gs[rank], bf16, dev)
            gdraa.gdraa_register(buf)
            gdraa.gdraa_allreduce_mean(buf)
            calls += 1
            torch.cuda.synchronize()
            compare(from_dev(buf), oracle.allreduce_mean(gs), dt, what=f"w8 mean L={L} r{rank}")
            w0, v0 = synth.w_like(82, L), synth.w_like(83, L)
            g = to_dev(gs[rank], bf16, dev)
            w, v = to_dev(w0, dev=dev), to_dev(v0, dev=dev)
            gdraa.gdraa_register(w)
            gdraa.gdraa_register(g)
            off, ln = gdraa.gdraa_shard(world, rank, L)
            for it in range(2):
                w0, v0 = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
                gdraa.gdraa_sgd_step_ex(w, g, v, 0.1, 0.9, 0.001)
                calls += 1
            torch.cuda.synchronize()
            compare(from_dev(w), w0, "f32", what=f"w8 sgd w L={L} {dt} r{rank}")
            compare(from_dev(v)[off:off + ln], v0[off:off + ln], "f32", what=f"w8 v r{rank}")
            for t in (buf, w, g):
                gdraa.gdraa_deregister(t)
    st = gdraa.gdraa_get_stats()
    assert st["calls"] == calls and st["iter_done"] == calls, (st, calls)
    gdraa.gdraa_finalize()
    with open(os.path.join(out_dir, f"w8_{rank}.json"), "w") as f:
        json.dump({"calls": calls, "device": d, "stats": st}, f)


def test_multiprocess_world8_oversubscribed(tmp_path):
    from paper_1802_02326_b200 import jobserver
    world, ndev = 8, torch.cuda.device_count()
    sock = str(tmp_path / "js.sock")
    js = jobserver.start(world, sock)
    try:
        mp.start_processes(_over_worker, args=(world, ndev, sock, str(tmp_path)), nprocs=world,
                           join=True, start_method="spawn")
    finally:
        out, err = js.communicate(timeout=300)
    line = json.loads(out.strip().splitlines()[-1])["jobserver"]
    reps = [json.load(open(tmp_path / f"w8_{r}.json")) for r in range(world)]
    assert line["ok"] and line["data_bytes"] == 0 and line["ranks_joined"] == 8, line
    assert line["done"] == [reps[0]["calls"]] * world, line


def test_soak_short(tmp_path):
    """tools/soak.py for 15 s: random calls of every entry point (sets, streamed sets, two
    streams, both size classes) through the multi-process path, each checked bit for bit
    (time-sliced ranks on a one-GPU box)."""
    import socket
    import subprocess
    import sys
    world = mp_world()
    with socket.socket() as t:
        t.bind(("127.0.0.1", 0))
        port = t.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(root, "tools", "soak.py"), "--seconds", "15", "--max-elems", "1000000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["iterations"] > 0 and d["mismatches"] == 0, d
