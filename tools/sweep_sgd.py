#!/usr/bin/env python
"""Crossover sweep of gdraa_sgd_step: the small-message (LL) SGD kernel vs the two-shot
fused kernel, fp32 (or bf16) gradients of 1 KiB - 64 MiB per rank.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/sweep_sgd.py --path ll [--graph]
    torchrun ... tools/sweep_sgd.py --path two_shot [--graph]

The path is fixed at gdraa_init from GDRAA_LL_SGD_MAX_BYTES (huge: the LL kernel wherever
the receive slot holds the shard; 0: the two-shot kernel), so each path is one run.
Prints one JSON line per size on rank 0 (max over ranks, CUDA events); both paths give
the same bits (tests/test_gpu_parity.py).
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
    ap.add_argument("--max-log2", type=int, default=26)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays")
    ap.add_argument("--path", default="ll", choices=["ll", "two_shot"])
    args = ap.parse_args()
    os.environ["GDRAA_LL_SGD_MAX_BYTES"] = str(1 << 40) if args.path == "ll" else "0"
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
    js = jobserver.setup_for_rank(world, rank, local, tag="swsgd" + os.environ["MASTER_PORT"])
    gdraa.gdraa_init(world, rank)
    stream = torch.cuda.current_stream()
    cap_stream = torch.cuda.Stream()
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + rank)
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    es = 4 if args.dtype == "f32" else 2
    code = gdraa.GDRAA_F32 if args.dtype == "f32" else gdraa.GDRAA_BF16

    def timed(fn, iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        graph = None
        if args.graph:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap_stream):
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

    cap = gdraa.gdraa_small_message_bytes(world)   # LL slot bytes per sender
    for k in range(args.min_log2, args.max_log2 + 1):
        nbytes = 1 << k
        n = nbytes // es
        g = (torch.randn(n, device=dev, generator=gen) * 1e-3).to(tdt)
        w0 = torch.randn(n, device=dev, generator=torch.Generator(device=dev).manual_seed(7))
        if args.path == "ll" and gdraa.gdraa_small_step_bytes(world, code) < nbytes:
            break                                          # the shard no longer fits a slot
        w = w0.clone()
        v = torch.zeros(n, device=dev)
        gdraa.gdraa_register(w)
        gdraa.gdraa_register(g)
        gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9)
        torch.cuda.synchronize()
        iters = 1000 if nbytes <= (1 << 20) else 200
        t = timed(lambda: gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9), iters)
        gdraa.gdraa_deregister(w)
        gdraa.gdraa_deregister(g)
        bus = (world - 1) / world * n * (es + 4) / (t * 1e-3) / 1e9
        line = {"n_gpus": world, "dtype": args.dtype, "g_bytes": nbytes, "n": n,
                "path": args.path,
                "timing": "cuda_graph_replay" if args.graph else "eager_python_loop",
                "us": t * 1e3, "busbw_gbs": bus, "ll_slot_bytes": cap}
        if rank == 0:
            print(json.dumps(line), file=out, flush=True)
        del g, w0
    gdraa.gdraa_finalize()
    if js is not None:
        js.communicate(timeout=60)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
