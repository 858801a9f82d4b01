#!/usr/bin/env python
"""NEXT-3 measurement: overlap of the bucketed GDRAA step with a backward pass.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/overlap.py [--buckets 8]

A synthetic backward of K bf16 GEMMs (sized so the whole backward takes about as long as
one full-buffer step) produces the ResNet-50 gradient buffer bucket by bucket, last
bucket first.  Four timings per rank, max over ranks, CUDA events:
  bwd      the K GEMMs alone
  comm     one gdraa_sgd_step over the whole buffer alone
  serial   the K GEMMs, then the whole-buffer step (no overlap)
  overlap  after GEMM k, bucket k is reduced and applied by gdraa_sgd_step_range on a
           side stream while GEMM k+1 runs (synchronisations "as late as the DL
           needs")
Prints one JSON line on rank 0.  GDRAA_MAX_CTAS caps the collective's grid.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--buckets", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--gemm", type=int, default=0, help="GEMM size (0: calibrate)")
    ap.add_argument("--set", action="store_true",
                    help="issue the buckets of one iteration as a bucket set "
                         "(gdraa_bucket_set_begin/_end: one deferred exit barrier per set)")
    ap.add_argument("--nccl", action="store_true",
                    help="reference point: each bucket as torch.distributed all_reduce(AVG) "
                         "(NCCL) followed by torch's momentum-SGD ops on the bucket, the "
                         "DDP-plus-optimizer pattern, instead of the library")
    ap.add_argument("--comm-only", action="store_true",
                    help="time only the whole-buffer and the bucketed step (no backward)")
    ap.add_argument("--streamed", type=int, default=0, metavar="CTAS",
                    help="issue the buckets as a STREAMED bucket set: one persistent kernel "
                         "of CTAS CTAs per rank serves all of them")
    args = ap.parse_args()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)

    import torch
    import torch.distributed as dist

    import synth
    from paper_1802_02326_b200 import gdraa, jobserver

    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    js = jobserver.setup_for_rank(world, rank, local, tag="ovl" + os.environ["MASTER_PORT"])
    gdraa.gdraa_init(world, rank)

    L = synth.L_R50
    g = torch.from_numpy(synth.grad_like(7, rank, L)).to(dev)
    w = torch.from_numpy(synth.w_like(7, L)).to(dev)
    v = torch.zeros(L, device=dev)
    gdraa.gdraa_register(w)
    gdraa.gdraa_register(g)
    K = args.buckets
    edges = [(L * k // K) // 64 * 64 for k in range(K)] + [L]
    buckets = [(edges[k], edges[k + 1] - edges[k]) for k in range(K)][::-1]   # last first
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    lr, mom = synth.PAPER_LR, synth.PAPER_MOM

    def t_max(ms):
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main_s)
        for _ in range(iters):
            fn()
        e1.record(main_s)
        torch.cuda.synchronize()
        return t_max(e0.elapsed_time(e1) / iters)

    def nccl_step(first, count, stream):
        with torch.cuda.stream(stream):
            gb, vb, wb = g[first:first + count], v[first:first + count], w[first:first + count]
            dist.all_reduce(gb, op=dist.ReduceOp.AVG)
            vb.mul_(mom).add_(gb)
            wb.add_(vb, alpha=-lr)

    def step_range(first, count, stream):
        if args.nccl:
            nccl_step(first, count, stream)
        else:
            gdraa.gdraa_sgd_step_range(w, g, v, first, count, lr, mom, 0.0, stream=stream)

    def comm():
        if args.nccl:
            nccl_step(0, L, main_s)
        else:
            gdraa.gdraa_sgd_step(w, g, v, lr, mom)

    t_comm = timed(comm, args.iters)

    # one GEMM per bucket, sized so that the K GEMMs take ~ one full step
    n = args.gemm
    if n == 0:
        n = 512
        while True:
            a = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
            t = timed(lambda: a @ a, 5)
            if t * K >= t_comm or n >= 16384:
                break
            n += 256
    A = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    C = torch.empty_like(A)

    def bwd():
        for _ in range(K):
            torch.mm(A, A, out=C)

    def serial():
        bwd()
        comm()

    evs = [torch.cuda.Event() for _ in range(K)]

    def set_begin():
        if args.nccl:
            return
        if args.streamed:
            gdraa.gdraa_bucket_set_begin_streamed(args.streamed)
        elif args.set:
            gdraa.gdraa_bucket_set_begin()

    in_set = (args.set or args.streamed > 0) and not args.nccl

    def overlap():
        set_begin()
        for k, (first, count) in enumerate(buckets):
            torch.mm(A, A, out=C)               # "produces" bucket k
            evs[k].record(main_s)
            side.wait_event(evs[k])
            step_range(first, count, side)
        if in_set:
            gdraa.gdraa_bucket_set_end(stream=side)
        main_s.wait_stream(side)

    def comm_buckets():
        set_begin()
        for first, count in buckets:
            step_range(first, count, main_s)
        if in_set:
            gdraa.gdraa_bucket_set_end()

    t_comm_b = timed(comm_buckets, args.iters)
    if args.comm_only:
        t_bwd = t_serial = t_overlap = float("nan")
    else:
        t_bwd = timed(bwd, args.iters)
        t_serial = timed(serial, args.iters)
        t_overlap = timed(overlap, args.iters)
    if rank == 0:
        hidden = (t_serial - t_overlap) / min(t_bwd, t_comm)
        line = {"n_gpus": world, "L": L, "buckets": K, "gemm_n": n,
                "max_ctas": os.environ.get("GDRAA_MAX_CTAS", "all"),
                "kernel": os.environ.get("GDRAA_KERNEL", "default"), "bucket_set": "streamed" if args.streamed else args.set,
                "streamed_ctas": args.streamed, "impl": "nccl+torch" if args.nccl else "gdraa",
                "bwd_us": t_bwd * 1e3, "comm_us": t_comm * 1e3,
                "comm_bucketed_us": t_comm_b * 1e3, "serial_us": t_serial * 1e3,
                "overlap_us": t_overlap * 1e3, "speedup": t_serial / t_overlap,
                "fraction_of_shorter_phase_hidden": hidden}
        print(json.dumps(line), file=out, flush=True)
    gdraa.gdraa_finalize()
    if js is not None:
        js.communicate(timeout=60)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
