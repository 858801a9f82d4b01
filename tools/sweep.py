#!/usr/bin/env python
"""Config 5: allreduce message-size sweep, 1 KiB - 1 GiB fp32, gdraa_allreduce_mean vs
torch.distributed NCCL all_reduce(AVG) on the same box and the same buffers.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/sweep.py [--max-log2 30]

Prints one JSON line per size on rank 0: time per call (max over ranks, CUDA events)
and bus GB/s per rank, busBW = 2 (N-1)/N * S / t (NCCL's definition).  Every size is
also checked against NCCL's result (within 1e-6 relative: different summation order, so
not bitwise) on the first call.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--out", default=None)
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays")
    ap.add_argument("--nccl-op", choices=["avg", "sum"], default="avg",
                    help="NCCL op timed (the result check always uses AVG)")
    args = ap.parse_args()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)

    import torch
    import torch.distributed as dist
    from paper_1802_02326_b200 import gdraa, jobserver

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    js = jobserver.setup_for_rank(world, rank, local, tag="sweep" + os.environ["MASTER_PORT"])
    gdraa.gdraa_init(world, rank)
    stream = torch.cuda.current_stream()
    cap_stream = torch.cuda.Stream()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    lines = []

    def timed(fn, iters):
        """Per-call device time (max over ranks).  With --graph the `iters` calls are
        captured into one CUDA graph and replayed, so host launch cost is excluded."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        graph = None
        if args.graph:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap_stream):   # fn uses the current stream
                for _ in range(iters):
                    fn()
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for _ in range(iters):
                fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for k in range(args.min_log2, args.max_log2 + 1):
        nbytes = 1 << k
        n = nbytes // 4
        x = torch.randn(n, device=dev, generator=gen)
        ours = x.clone()
        ref = x.clone()
        gdraa.gdraa_register(ours)
        gdraa.gdraa_allreduce_mean(ours)
        dist.all_reduce(ref, op=dist.ReduceOp.AVG)
        torch.cuda.synchronize()
        rel = float(((ours - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item())
        iters = 1000 if nbytes <= (1 << 20) else (200 if nbytes <= (1 << 26) else 20)
        t_ours = timed(lambda: gdraa.gdraa_allreduce_mean(ours), iters)   # current stream
        # timed op: AVG (same semantics) or SUM (lets NCCL pick NVLS in-switch reduction)
        nop = dist.ReduceOp.SUM if args.nccl_op == "sum" else dist.ReduceOp.AVG
        t_nccl = timed(lambda: dist.all_reduce(ref, op=nop), iters)
        gdraa.gdraa_deregister(ours)
        bus = lambda ms: 2 * (world - 1) / world * nbytes / (ms * 1e-3) / 1e9  # noqa: E731
        line = {"n_gpus": world, "bytes": nbytes, "iters": iters,
                "timing": "cuda_graph_replay" if args.graph else "eager_python_loop",
                "gdraa_us": t_ours * 1e3, "gdraa_busbw_gbs": bus(t_ours),
                "nccl_us": t_nccl * 1e3, "nccl_busbw_gbs": bus(t_nccl),
                "speedup_vs_nccl": t_nccl / t_ours, "max_rel_diff_vs_nccl": rel,
                "nccl_op": args.nccl_op,
                "nccl_env": {k: os.environ[k] for k in ("NCCL_ALGO", "NCCL_PROTO",
                                                         "NCCL_NVLS_ENABLE")
                             if k in os.environ}}
        assert rel <= 1e-5, line
        if rank == 0:
            print(json.dumps(line), file=out, flush=True)
            lines.append(line)
        del x, ours, ref   # (no empty_cache: the allocator keeps the exported segments)
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            for line in lines:
                f.write(json.dumps(line) + "\n")
    gdraa.gdraa_finalize()
    if js is not None:
        js.communicate(timeout=60)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
