#!/usr/bin/env python
"""Per-call timing of gdraa_sgd_step when the calls rotate over S buffer sets (debug aid
for the small-message SGD path).  torchrun --nproc-per-node 2 tools/ll_debug.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
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
    js = jobserver.setup_for_rank(world, rank, local, tag="lldbg" + os.environ["MASTER_PORT"])
    gdraa.gdraa_init(world, rank)
    stream = torch.cuda.current_stream()
    n = int(os.environ.get("LLDBG_N", str(1 << 20)))
    for S in (1, 2, 3, 8):
        for shared in ("none", "g", "wv"):
            if S == 1 and shared != "none":
                continue
            g0 = torch.randn(n, device=dev) * 1e-3
            w0 = torch.randn(n, device=dev)
            v0 = torch.zeros(n, device=dev)
            sets = []
            for s in range(S):
                g = g0 if shared == "g" else torch.randn(n, device=dev) * 1e-3
                w = w0 if shared == "wv" else torch.randn(n, device=dev)
                v = v0 if shared == "wv" else torch.zeros(n, device=dev)
                if shared != "wv" or s == 0:
                    gdraa.gdraa_register(w)
                if shared != "g" or s == 0:
                    gdraa.gdraa_register(g)
                sets.append((w, g, v))
            for k in range(20):
                w, g, v = sets[k % S]
                gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9, stream)
            dist.barrier(device_ids=[local])
            torch.cuda.synchronize()
            K = 100
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
            evs[0].record(stream)
            for k in range(K):
                w, g, v = sets[k % S]
                gdraa.gdraa_sgd_step(w, g, v, 0.1, 0.9, stream)
                evs[k + 1].record(stream)
            torch.cuda.synchronize()
            ts = sorted(evs[k].elapsed_time(evs[k + 1]) * 1e3 for k in range(K))
            tot = evs[0].elapsed_time(evs[K]) * 1e3 / K
            line = {"rank": rank, "n": n, "sets": S, "shared": shared, "mean_us": tot,
                    "p10": ts[K // 10], "p50": ts[K // 2], "p90": ts[9 * K // 10], "max": ts[-1]}
            print(json.dumps(line), file=out, flush=True)
            for w, g, v in sets:
                for t in (w, g):
                    try:
                        gdraa.gdraa_deregister(t)
                    except gdraa.GdraaError:
                        pass
            dist.barrier(device_ids=[local])
    gdraa.gdraa_finalize()
    if js is not None:
        js.communicate(timeout=60)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
