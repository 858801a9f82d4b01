#!/usr/bin/env python
"""Soak test of the multi-process path: thousands of randomly chosen collective calls
(every entry point, both kernels' size classes, bucket sets per call and streamed, calls
on two streams), each checked bit for bit.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/soak.py [--seconds 300]

Inputs are integer-valued (SURVEY §8(c) integer family) and N is a power of two, so every
result is exact in any summation order: the expected values are computed on the device
with plain torch ops (an independent check of the library's bits, not part of it).  Each
rank reports its counts; rank 0 prints one JSON line (calls per kind, mismatches, elapsed).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--max-elems", type=int, default=3_000_000)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1802_02326_b200 import gdraa, jobserver

    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    assert world & (world - 1) == 0, "world must be a power of two (exact integer family)"
    # ranks share GPUs (time-sliced) when there are fewer GPUs than ranks: gloo plumbing
    shared = torch.cuda.device_count() < world
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    js = jobserver.setup_for_rank(world, rank, int(os.environ["LOCAL_RANK"]),
                                  tag="soak" + os.environ["MASTER_PORT"])
    gdraa.gdraa_init(world, rank)

    M = args.max_elems
    lr, mom = 0.125, 0.5                          # dyadic: the update is exact
    # registered buffers, reused by every call (ranges of them)
    g = torch.empty(M, device=dev)
    gb = torch.empty(M, dtype=torch.bfloat16, device=dev)
    w = torch.empty(M, device=dev)
    model = torch.empty(M, dtype=torch.bfloat16, device=dev)
    buf = torch.empty(M, device=dev)
    for t in (g, gb, w, model, buf):
        gdraa.gdraa_register(t)
    v = torch.zeros(M, device=dev)
    wm = torch.empty(M, device=dev)
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    rng = np.random.default_rng(args.seed)         # same sequence on every rank

    def ints(seed, r, n, lo, hi, dtype=torch.float32):
        gen = torch.Generator(device=dev).manual_seed(seed * 1000 + r)
        return torch.randint(lo, hi, (n,), generator=gen, device=dev).to(dtype)

    counts, bad, fails = {}, 0, []
    t_end = time.time() + args.seconds
    it = 0
    while True:
        stop = torch.tensor([1 if time.time() > t_end else 0], device="cpu" if shared else dev)
        dist.all_reduce(stop, op=dist.ReduceOp.MAX)   # every rank stops at the same call
        if stop.item():
            break
        it += 1
        kind = rng.choice(["sgd", "sgd_bf16", "mp", "mean", "mean_bf16", "set", "streamed"])
        n = int(rng.choice([rng.integers(1, 4096), rng.integers(4096, 1 << 18),
                            rng.integers(1 << 18, M)]))
        n = max(8, n // 8 * 8)
        seed = int(rng.integers(1 << 30))
        stream = side if rng.random() < 0.3 else torch.cuda.current_stream()
        gs = [ints(seed, p, n, -128, 128) for p in range(world)]     # every rank's gradient
        mean = sum(gs[1:], gs[0]) / world                            # exact (power of two)
        w0 = ints(seed, 99, n, -4096, 4096)
        v0 = ints(seed, 98, n, -1024, 1024)
        off, ln = gdraa.gdraa_shard(world, rank, n)
        ok = True
        if kind in ("sgd", "sgd_bf16", "set", "streamed"):
            gsrc = gb if kind == "sgd_bf16" else g
            gsrc[:n].copy_(gs[rank].to(gsrc.dtype))
            w[:n].copy_(w0)
            v[:n].copy_(v0)
            stream.wait_stream(main)          # the input copies above
            with torch.cuda.stream(stream):
                if kind in ("sgd", "sgd_bf16"):
                    gdraa.gdraa_sgd_step_range(w, gsrc, v, 0, n, lr, mom, 0.0, stream=stream)
                else:
                    cut = max(8, n // 2 // 8 * 8) if n > 8 else n
                    if kind == "set":
                        gdraa.gdraa_bucket_set_begin()
                    else:
                        gdraa.gdraa_bucket_set_begin_streamed(int(rng.choice([16, 64])))
                    for a, c in ((cut, n - cut), (0, cut)):
                        if c > 0:
                            gdraa.gdraa_sgd_step_range(w, gsrc, v, a, c, lr, mom, 0.0,
                                                       stream=stream)
                    gdraa.gdraa_bucket_set_end(stream=stream)
            main.wait_stream(stream)
            v1 = mom * v0 + mean
            w1 = w0 - lr * v1
            ok = torch.equal(w[:n], w1)
            if kind in ("sgd", "sgd_bf16"):
                ok &= torch.equal(v[off:off + ln], v1[off:off + ln])
        elif kind == "mp":
            gb[:n].copy_(gs[rank].to(torch.bfloat16))
            wm[:n].copy_(w0)
            v[:n].copy_(v0)
            stream.wait_stream(main)          # the input copies above
            with torch.cuda.stream(stream):
                gdraa.gdraa_sgd_step_mp_range(wm, model, gb, v, 0, n, lr, mom, 0.0,
                                              stream=stream)
            main.wait_stream(stream)
            v1 = mom * v0 + mean
            w1 = w0 - lr * v1
            ok = torch.equal(model[:n], w1.to(torch.bfloat16))
            ok &= torch.equal(wm[off:off + ln], w1[off:off + ln])
        else:
            b = buf if kind == "mean" else gb
            b[:n].copy_(gs[rank].to(b.dtype))
            stream.wait_stream(main)          # the input copies above
            with torch.cuda.stream(stream):
                gdraa.gdraa_allreduce_mean_range(b, 0, n, stream=stream)
            main.wait_stream(stream)
            ok = torch.equal(b[:n], mean.to(b.dtype))
        counts[kind] = counts.get(kind, 0) + 1
        if not bool(ok):
            bad += 1
            if len(fails) < 20:
                fails.append({"it": it, "kind": str(kind), "n": n, "side": stream is side})
    torch.cuda.synchronize()
    st = gdraa.gdraa_get_stats()
    rep = [None] * world
    dist.all_gather_object(rep, {"rank": rank, "bad": bad, "fails": fails, "calls": counts,
                                 "device_calls": st["calls"], "ll_calls": st["ll_calls"]})
    if rank == 0:
        print(json.dumps({"soak": True, "n_gpus": world, "seconds": args.seconds,
                          "iterations": it, "mismatches": sum(r["bad"] for r in rep),
                          "per_rank": rep}), file=out, flush=True)
    gdraa.gdraa_finalize()
    if js is not None:
        js.communicate(timeout=60)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
