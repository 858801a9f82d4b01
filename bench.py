#!/usr/bin/env python
"""Benchmark of the GDRAA hot path: the fused gradient allreduce + momentum-SGD step
(gdraa_sgd_step) on ResNet-sized gradient buffers, 1 process per B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config r50|r101|r50bf16|c1]
                    [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One "step" = one gdraa_sgd_step over the whole gradient buffer (= one kernel launch:
reduce -> average -> update -> broadcast, two device synchronisations).  Prints ONE JSON
line on rank 0 (contract in DESIGN.md "Measurement").  Metric (BASELINE.json): bus GB/s
of the fused allreduce+SGD and its fraction of the NVLink roofline; N = 1 has no NVLink
traffic and reports the kernel's algorithmic HBM GB/s against the measured HBM copy peak.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

OUT = sys.stdout

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "allreduce+SGD bus GB/s and % NVLink roofline at 1/2/4/8 B200 (ResNet-50 grads)"
CONFIGS = {
    # name: (L, g dtype, description)
    "c1": (synth.L_C1, "f32", "config 1: 1M-element fp32 gradient"),
    "r50": (synth.L_R50, "f32", "config 2: ResNet-50 fp32 gradient buffer (25,557,032)"),
    "r101": (synth.L_R101, "f32", "config 3: ResNet-101 fp32 gradient buffer (44,549,160)"),
    "r50bf16": (synth.L_R50, "bf16", "config 4: ResNet-50 bf16 gradients, fp32 master w/v"),
    "r50bf16mp": (synth.L_R50, "bf16", "config 4 + NEXT-1: bf16 gradients, fp32 master "
                  "sharded like v, bf16 model copy all-gathered, weight decay 0.001"),
}
MP_CONFIGS = {"r50bf16mp"}
PAPER_WD = 0.001               # P:246 "weight decay is 0.001"
NVLINK_NOMINAL_GBS = 900.0     # NVLink 5, per direction per GPU
NVLINK_MEASURED_GBS = 770.0    # B200_PROFILING.md: measured peer copy per direction


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(L, N, s_g, s_w=4):
    """Per-rank algorithmic bytes of one step (DESIGN.md §6 "Roofline").
    N = 1: HBM bytes of the local fused SGD, (s_g + 16) * L (read g, w, v; write w, v),
    plus s_w * L for the separate model copy of the mixed-precision variant (s_w = 2).
    N >= 2: NVLink bus bytes per rank per direction, B_nv = (N-1)/N * L * (s_g + s_w)
    (reduce ingress of g + broadcast ingress of w' or its bf16 copy; NCCL busBW
    convention)."""
    if N == 1:
        return (s_g + 16 + (s_w if s_w != 4 else 0)) * L
    return (N - 1) / N * L * (s_g + s_w)


# ---------------------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------------------
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, torch_dev):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            uuid = str(torch.cuda.get_device_properties(torch_dev).uuid)
            try:
                self.h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(torch_dev)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:   # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            self._stop.wait(0.005)

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in REASONS.items():
                if mask & bit:
                    self.reasons.add(name)
        except Exception:   # noqa: BLE001
            pass

    def start(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self):
        self._stop.set()
        self.t.join()
        self.sample()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons - {"gpu_idle"}),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------
# the oracle as a CPU baseline (rank 0 only)
# ---------------------------------------------------------------------------------------
class OracleSample:
    """The CPU oracle (single-threaded C, as it stands) on a bounded sample of the
    workload: the first n elements of every one of the N rank buffers (all N ranks are
    simulated in one process, as the oracle defines the method)."""

    def __init__(self, L, N, g_dt, mp=False, n=1 << 20):
        import oracle
        self.oracle, self.L, self.N, self.n, self.mp = oracle, L, N, min(L, n), mp
        self.gs = [synth.grad_like(0, p, self.n) for p in range(N)]
        if g_dt == "bf16":
            self.gs = [synth.to_bf16_bits_trunc(g) for g in self.gs]
        self.w, self.v = synth.w_like(0, self.n), np.zeros(self.n, np.float32)
        s_g = 2 if g_dt == "bf16" else 4
        # the metric's per-rank bytes for one step of this sample (as `value`: one step of
        # all N ranks takes the measured time, so per-rank bytes / that time)
        self.bytes = algorithmic_bytes(self.n, N, s_g, 2 if mp else 4)

    def step(self):
        t0 = time.perf_counter()
        if self.mp:
            self.w, self.v, _ = self.oracle.sgd_step_wd(
                self.gs, self.w, self.v, synth.PAPER_LR, synth.PAPER_MOM, PAPER_WD,
                model_dtype=self.oracle.BF16)
        else:
            self.w, self.v = self.oracle.sgd_step(self.gs, self.w, self.v, synth.PAPER_LR,
                                                  synth.PAPER_MOM)
        return time.perf_counter() - t0

    def step_mt(self, pool, k):
        """The same oracle call on k contiguous pieces of the sample, one per thread
        (ctypes drops the GIL; the pieces are independent, so the result is identical)."""
        cuts = [self.n * i // k for i in range(k + 1)]

        def piece(i):
            a, b = cuts[i], cuts[i + 1]
            gs = [g[a:b] for g in self.gs]
            if self.mp:
                w, v, _ = self.oracle.sgd_step_wd(gs, self.w[a:b], self.v[a:b], synth.PAPER_LR,
                                                  synth.PAPER_MOM, PAPER_WD,
                                                  model_dtype=self.oracle.BF16)
            else:
                w, v = self.oracle.sgd_step(gs, self.w[a:b], self.v[a:b], synth.PAPER_LR,
                                            synth.PAPER_MOM)
            return a, b, w, v

        t0 = time.perf_counter()
        for a, b, w, v in pool.map(piece, range(k)):
            self.w[a:b], self.v[a:b] = w, v
        return time.perf_counter() - t0

    def describe(self, reps):
        return (f"{reps} oracle sgd_step calls over the first {self.n} elements of each of "
                f"the {self.N} rank buffers (L={self.L}); single thread")


def oracle_baseline(L, N, g_dt, budget_s, mp=False):
    """(bytes/s, sample description, s/step) of the oracle over ~budget_s seconds."""
    s = OracleSample(L, N, g_dt, mp)
    s.step()
    reps, total = 0, 0.0
    while total < budget_s:
        total += s.step()
        reps += 1
    return s.bytes / (total / reps), s.describe(reps), total / reps


def oracle_baseline_mt(L, N, g_dt, budget_s, mp=False):
    """The labelled k-thread variant: k = host cores, same sample."""
    from concurrent.futures import ThreadPoolExecutor
    k = os.cpu_count() or 1
    s = OracleSample(L, N, g_dt, mp, n=1 << 23)    # 8M elements: enough work per thread
    with ThreadPoolExecutor(max_workers=k) as pool:
        s.step_mt(pool, k)
        reps, total = 0, 0.0
        while total < budget_s:
            total += s.step_mt(pool, k)
            reps += 1
    return s.bytes / (total / reps), k, reps, s.n


def run_reference(args):
    """--impl reference: the CPU oracle on the same config and metric.  Each step is one
    oracle call over a bounded sample of the workload (OracleSample)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    L, g_dt, desc = CONFIGS[args.config]
    N = args.gpus
    s = OracleSample(L, N, g_dt, args.config in MP_CONFIGS)
    for _ in range(args.warmup):
        s.step()
    dts = [s.step() for _ in range(args.steps)]
    sample = s.describe(args.steps)
    value = s.bytes / float(np.mean(dts)) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(dts)) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_dict(args, L, g_dt, desc, N, "oracle (CPU)"),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu_model": cpu_model(),
                         "host_cores": os.cpu_count()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=OUT, flush=True)
    return 0


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as t:
        t.bind(("127.0.0.1", 0))
        return t.getsockname()[1]


def self_launch(n, argv):
    """Re-run this script as N ranks under torch.distributed.run (one process per GPU,
    NCCL plumbing, rendezvous on 127.0.0.1).  Every rank sends library output to stderr;
    rank 0 alone prints the JSON line, on the stdout inherited from this process."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.join(ROOT, "bench.py"), *argv]
    return subprocess.run(cmd, cwd=ROOT).returncode


def dry_launch(args):
    """The launch path alone (CPU test of self_launch): N ranks meet in a gloo group;
    rank 0 prints what every rank saw."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    me = {"rank": rank, "local_rank": int(os.environ.get("LOCAL_RANK", "0")),
          "master_addr": os.environ.get("MASTER_ADDR")}
    table = [me]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        table = [None] * world
        dist.all_gather_object(table, me)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_launch": True, "n_gpus": args.gpus, "world": world,
                          "ranks": table}), file=OUT, flush=True)
    return 0


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or None


def config_dict(args, L, g_dt, desc, N, path=None):
    mp = args.config in MP_CONFIGS
    s_g = 2 if g_dt == "bf16" else 4
    return {"workload": args.config, "description": desc, "L": L, "g_dtype": g_dt,
            "w_dtype": "f32 master sharded + bf16 model copy" if mp else "f32",
            "v_dtype": "f32", "lr": synth.PAPER_LR, "mom": synth.PAPER_MOM,
            "wd": PAPER_WD if mp else 0.0,
            "parallelism": f"dp{N}", "buffer_sets": args.sets,
            "l2": ("n/a: the CPU oracle on host memory" if args.sets <= 0 else
                   f"inputs larger than L2: {args.sets} rotating (g, w, v) sets per rank "
                   f"({args.sets * L * (s_g + 8 + (2 if mp else 0)) / 1e6:.0f} MB)"),
            "path": path,
            "timing": ("host wall clock of the CPU oracle per step" if args.impl == "reference"
                       else "one CUDA-graph replay of the K steps" if args.graph
                       else "eager Python loop of the K steps")}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="r50", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sets", type=int, default=0,
                    help="rotating (g, w, v) sets per rank; 0 = enough to exceed 2x L2")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--eager", dest="graph", action="store_false",
                    help="time an eager Python loop of the K steps instead of one CUDA-graph "
                         "replay of them (the default: host launch cost out of the step)")
    ap.add_argument("--graph", dest="graph", action="store_true")
    ap.set_defaults(graph=True)
    ap.add_argument("--dry-launch", action="store_true",
                    help="check the process launch only: every rank joins a gloo group, rank "
                         "0 prints the rank table as the JSON line (no GPU work)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # `python bench.py --gpus N` without a launcher: start the N ranks ourselves
        # (torchrun on a free loopback port); rank 0's JSON line reaches our stdout.
        return self_launch(args.gpus, sys.argv[1:])
    # Exactly one JSON line on stdout: anything libraries print (NCCL banners, ...) goes
    # to stderr; the result line goes to the saved stdout.
    global OUT
    OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.dry_launch:
        return dry_launch(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_1802_02326_b200 import gdraa, jobserver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun")
    # GDRAA_BENCH_OVERSUBSCRIBE=1: a functional check of the N-rank path on a box with
    # fewer GPUs (ranks share GPUs round-robin, time-sliced; gloo plumbing, no NCCL
    # reference).  Its times are meaningless and the JSON line says so.
    oversub = os.environ.get("GDRAA_BENCH_OVERSUBSCRIBE") == "1"
    if oversub:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    js = None
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
            args.no_nccl = True
        else:
            dist.init_process_group("nccl", device_id=dev)
        js = jobserver.setup_for_rank(world, rank, int(os.environ.get("LOCAL_RANK", "0")))
    gdraa.gdraa_init(world, rank)

    L, g_dt, desc = CONFIGS[args.config]
    mp = args.config in MP_CONFIGS
    N = world
    s_g = 2 if g_dt == "bf16" else 4
    s_w = 2 if mp else 4
    tdt = torch.bfloat16 if g_dt == "bf16" else torch.float32
    off, ln = gdraa.gdraa_shard(N, rank, L)
    lr, mom = synth.PAPER_LR, synth.PAPER_MOM
    wd = PAPER_WD if mp else 0.0
    stream = torch.cuda.current_stream()

    class StepSet:
        """One (g, w, v) buffer set and the public call that steps it."""

        def __init__(self, s):
            g_h = synth.grad_like(100 + s, rank, L)
            if g_dt == "bf16":
                g_h = synth.to_bf16_bits_trunc(g_h).view(np.int16)
            self.g = torch.from_numpy(g_h).to(dev)
            self.g = self.g.view(tdt) if g_dt == "bf16" else self.g
            self.w = torch.from_numpy(synth.w_like(100 + s, L)).to(dev)   # fp32 (master)
            self.v = torch.zeros(L, dtype=torch.float32, device=dev)
            if mp:   # NEXT-1: replicated bf16 model copy, fp32 master sharded like v
                self.model = torch.zeros(L, dtype=torch.bfloat16, device=dev)
                gdraa.gdraa_register(self.model)
            else:
                gdraa.gdraa_register(self.w)
            gdraa.gdraa_register(self.g)

        def step(self, s=None):
            s = stream if s is None else s
            if mp:
                gdraa.gdraa_sgd_step_mp(self.w, self.model, self.g, self.v, lr, mom, wd, s)
            else:
                gdraa.gdraa_sgd_step(self.w, self.g, self.v, lr, mom, s)

        def result_shard(self):
            """This rank's share of the step's result (read back by the e2e leg)."""
            return (self.model if mp else self.w)[off:off + ln]

    # synthetic inputs (host), then resident in HBM; S rotating sets so that no step
    # finds its inputs in the 126 MB L2 (>= 3 sets, and >= 2x L2 of them in total).
    if args.sets <= 0:
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        set_bytes = L * (s_g + 4 + 4 + (2 if mp else 0))
        args.sets = max(3, -(-2 * l2 // set_bytes))
    sets = [StepSet(s) for s in range(args.sets)]
    # which kernel serves the step (both give the same bits): N = 1 is a local fused
    # SGD, small steps take the LL kernel (no device barrier), the rest the two-shot one
    code = gdraa.GDRAA_BF16 if g_dt == "bf16" else gdraa.GDRAA_F32
    path = ("local" if N == 1 else
            "ll_sgd" if L * s_g <= gdraa.gdraa_small_step_bytes(N, code, mp) else "two_shot")

    def barrier():
        if world > 1:
            dist.barrier() if oversub else dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for k in range(args.warmup):
        sets[k % len(sets)].step()
    barrier()

    graph = None
    if args.graph:
        # the K timed steps captured once into a CUDA graph (host launch cost out of the
        # step time; the library's epochs live in device memory, so replays are valid)
        cap = torch.cuda.Stream()
        g0 = gdraa.gdraa_get_stats()["launches"]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            for k in range(args.steps):
                sets[k % len(sets)].step(cap)
        graph_launches = gdraa.gdraa_get_stats()["launches"] - g0
        graph.replay()   # untimed warm-up replay
        barrier()

    st0 = gdraa.gdraa_get_stats()
    clocks = ClockSampler(local) if rank == 0 else None
    barrier()
    if clocks:
        clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for k in range(args.steps):
            sets[k % len(sets)].step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    barrier()
    st1 = gdraa.gdraa_get_stats()
    launches = st1["launches"] - st0["launches"]
    if graph is not None:   # replays do not pass through the host launch counter
        launches = graph_launches
    ms_step = ms / args.steps
    per_rank = algorithmic_bytes(L, N, s_g, s_w)
    achieved = per_rank / (ms_step * 1e-3) / 1e9            # per rank = per launch
    job_total = per_rank * N / (ms_step * 1e-3) / 1e9       # summed over ranks
    # the metric is bus GB/s (NCCL's busBW convention): B_nv / t per rank;
    # N = 1 has no bus and reports the launch's HBM rate
    value = achieved

    # ---- per-call distribution (untimed pass; an event pair around every call) ----
    M = min(args.steps, 200)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(M)]
    barrier()
    for k in range(M):
        evs[k][0].record(stream)
        sets[k % len(sets)].step()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    per = torch.tensor([a.elapsed_time(b) * 1e3 for a, b in evs], device=dev)
    if world > 1:
        dist.all_reduce(per, op=dist.ReduceOp.MAX)   # a call lasts until its slowest rank
    per = per.cpu().numpy()
    percall = {"calls": M, "median_us": float(np.median(per)),
               "p10_us": float(np.percentile(per, 10)), "p90_us": float(np.percentile(per, 90)),
               "note": "an event pair around each call (max over ranks per call); the pairs "
                       "break programmatic dependent launch between calls, so the median "
                       "sits above ms_per_step"}

    # ---- e2e: host buffers through the public API, copies inside the timed region ----
    # Every step copies its gradient H2D from pinned memory, runs the step and copies this
    # rank's shard of the updated weights D2H.  The copies of neighbouring steps overlap
    # (double-buffered gradients and D2H staging on their own streams), as a training
    # loop prefetching the next batch would.
    st = sets[0]
    g_bufs = [st.g, st.g.clone()]
    gdraa.gdraa_register(g_bufs[1])
    g_host = [torch.empty(L, dtype=tdt, pin_memory=True) for _ in range(2)]
    for h in g_host:
        h.copy_(st.g.cpu())
    out_dev = st.result_shard()
    stage = [torch.empty_like(out_dev) for _ in range(2)]
    out_host = [torch.empty(ln, dtype=out_dev.dtype, pin_memory=True) for _ in range(2)]
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("h2d", "step", "d2h")}
    start = torch.cuda.Event()

    def e2e_step(k):
        b = k % 2
        if k >= 2:
            s_h2d.wait_event(ev["step"][b])          # g_bufs[b] consumed by step k-2
        with torch.cuda.stream(s_h2d):
            g_bufs[b].copy_(g_host[b], non_blocking=True)
        ev["h2d"][b].record(s_h2d)
        stream.wait_event(ev["h2d"][b])
        if mp:
            gdraa.gdraa_sgd_step_mp(st.w, st.model, g_bufs[b], st.v, lr, mom, wd, stream)
        else:
            gdraa.gdraa_sgd_step(st.w, g_bufs[b], st.v, lr, mom, stream)
        if k >= 2:
            stream.wait_event(ev["d2h"][b])           # stage[b] drained by step k-2's D2H
        stage[b].copy_(out_dev, non_blocking=True)
        ev["step"][b].record(stream)
        s_d2h.wait_event(ev["step"][b])
        with torch.cuda.stream(s_d2h):
            out_host[b].copy_(stage[b], non_blocking=True)
        ev["d2h"][b].record(s_d2h)

    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    start.record(stream)
    s_h2d.wait_event(start)
    s_d2h.wait_event(start)
    for k in range(args.e2e_steps):
        e2e_step(k)
    stream.wait_stream(s_d2h)
    e1.record(stream)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ems], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    e2e_val = per_rank / (ems / args.e2e_steps * 1e-3) / 1e9   # same definition as value

    # the same per-step copies alone (H2D and D2H concurrently, no step): the PCIe bound
    # the e2e figure is held to
    barrier()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    s_h2d.wait_event(c0)
    s_d2h.wait_event(c0)
    for k in range(args.e2e_steps):
        with torch.cuda.stream(s_h2d):
            g_bufs[k % 2].copy_(g_host[k % 2], non_blocking=True)
        with torch.cuda.stream(s_d2h):
            out_host[k % 2].copy_(stage[k % 2], non_blocking=True)
    stream.wait_stream(s_h2d)
    stream.wait_stream(s_d2h)
    c1.record(stream)
    torch.cuda.synchronize()
    cms = c0.elapsed_time(c1)
    if world > 1:
        t = torch.tensor([cms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        cms = float(t.item())
    copy_bound = per_rank / (cms / args.e2e_steps * 1e-3) / 1e9

    # ---- NCCL all_reduce(AVG) of the same gradient buffer (reference point) ----
    nccl = None
    if world > 1 and not args.no_nccl:
        buf = sets[0].g.clone()
        for _ in range(5):
            dist.all_reduce(buf, op=dist.ReduceOp.AVG)
        barrier()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0.record(stream)
        for _ in range(20):
            dist.all_reduce(buf, op=dist.ReduceOp.AVG)
        n1.record(stream)
        torch.cuda.synchronize()
        nms = n0.elapsed_time(n1) / 20
        t = torch.tensor([nms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nms = float(t.item())
        nccl = {"op": "torch.distributed.all_reduce(AVG)", "bytes": L * s_g,
                "ms": nms, "bus_gbs_per_rank": 2 * (N - 1) / N * L * s_g / (nms * 1e-3) / 1e9,
                "nccl": ".".join(map(str, torch.cuda.nccl.version()))}

    if rank == 0:
        peaks, peak_src = measured_peaks()
        if N == 1:
            roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "peak_source": peak_src,
                    "bytes_per_launch": per_rank, "bytes_per_element": per_rank / L}
        else:
            roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_MEASURED_GBS,
                    "unit": "GB/s", "frac": achieved / NVLINK_MEASURED_GBS,
                    "peak_source": "measured B200 peer copy per direction (B200_PROFILING.md)",
                    "frac_of_nominal_900": achieved / NVLINK_NOMINAL_GBS,
                    "bytes_per_launch": per_rank}
            # the HBM side of the same launch: all of g read once (locally
            # or by peers), the owner shard's w / master and v read+written, and every
            # w' (or bf16 copy) element written once into this rank's memory
            hb = (s_g * L + (16 if mp else 12) * L / N + s_w * L)
            roof["hbm_side"] = {"bytes_per_launch": hb,
                                "achieved_gbs": hb / (ms_step * 1e-3) / 1e9,
                                "frac_of_peak": hb / (ms_step * 1e-3) / 1e9 / peaks["hbm_gbs"]}
        tr = ncu_traffic(args.config, N)
        if isinstance(tr, dict):   # N >= 2: the solo rank-0 capture
            roof["traffic"] = tr["dram_bytes"]
            roof["traffic_nvlink"] = {k: tr[k] for k in (
                "kind", "nvlink_rx_user_bytes", "nvlink_tx_user_bytes", "nvlink_rx_bytes",
                "nvlink_tx_bytes", "algorithmic_nvlink_bytes_own_share_per_direction",
                "nvlink_user_over_algorithmic", "source") if k in tr}
        else:
            roof["traffic"] = tr
        roof["kernel_ms"] = ms_step
        cpu = None
        if N == 1 and not args.no_cpu_baseline:
            cv, sample, _ = oracle_baseline(L, N, g_dt, 10.0, mp)
            cpu = {"value": cv / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
                   "sample": sample, "cpu_model": cpu_model(), "host_cores": os.cpu_count()}
            mv, k, mreps, mn = oracle_baseline_mt(L, N, g_dt, 5.0, mp)
            cpu["threaded_variant"] = {
                "value": mv / 1e9, "unit": "GB/s", "cores": k,
                "note": f"same oracle on the first {mn} elements of each rank buffer, split "
                        f"into {k} contiguous pieces on {k} threads ({mreps} steps); a "
                        f"labelled variant, not the baseline"}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, L, g_dt, desc, N, path),
            "value_definition": ("per-rank algorithmic bytes of one step / step time (max "
                                 "over ranks); "
                                 + (f"N=1: HBM bytes {per_rank / L:g}*L" if N == 1 else
                                    f"N>=2: bus bytes B_nv = (N-1)/N*L*({s_g}+{s_w}) per rank "
                                    "per direction (NCCL busBW convention)")),
            "bus_gbs_per_rank": achieved if N > 1 else 0.0,
            "job_total_gbs": job_total,
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "GB/s", "steps": args.e2e_steps,
                    "h2d_bytes_per_step": L * s_g * N, "d2h_bytes_per_step": L * s_w,
                    "note": "all ranks: H2D of each rank's gradient from pinned host memory, "
                            "the step through the public API, D2H of each rank's shard of "
                            "the updated weights (via a device staging copy); copies of "
                            "neighbouring steps overlap on separate streams",
                    "copies_only_value": copy_bound,
                    "frac_of_copies_only": e2e_val / copy_bound,
                    "copies_only_note": "the same H2D + D2H copies alone, no step: the PCIe "
                                        "bound of this e2e figure, in the same units"},
            "per_call": percall,
            "gpu_launches": launches, "clocks": clocks.summary() if clocks else None,
            "nccl_reference": nccl,
        }
        if oversub:
            line["oversubscribed"] = ("functional check only: %d ranks time-sliced on %d GPUs; "
                                      "the times are not a measurement"
                                      % (N, torch.cuda.device_count()))
        print(json.dumps(line), file=OUT, flush=True)

    barrier()
    gdraa.gdraa_finalize()
    if js is not None:
        js.communicate(timeout=60)
    if world > 1:
        dist.destroy_process_group()
    return 0


def ncu_traffic(config, N):
    """dram bytes per launch from the committed ncu --set full summary, if one matches."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            tab = json.load(f)
        return tab.get(f"{config}_n{N}")
    except OSError:
        return None


if __name__ == "__main__":
    sys.exit(main())
