#!/usr/bin/env python
"""Summarise ncu output for profiles/: the launch list (per-kernel share of device time)
and the key counters of one `--set full` capture.

    python tools/ncu_summary.py launches <launches.csv>            > profiles/…_launches.json
    python tools/ncu_summary.py full <prof.ncu-rep | raw.csv> [algorithmic_bytes] > profiles/…_ncu.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__inst_executed.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "nvlrx__bytes.sum", "nvltx__bytes.sum", "nvlrx__bytes_data_user.sum",
    "nvltx__bytes_data_user.sum",
]

SCALE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1}


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1))
    tot = sum(sum(v) for v in agg.values())
    return {"source": path, "total_device_s": tot,
            "kernels": [{"name": k, "launches": len(v), "avg_us": sum(v) / len(v) * 1e6,
                         "share": sum(v) / tot} for k, v in
                        sorted(agg.items(), key=lambda kv: -sum(kv[1]))]}


def full(path, algorithmic=None):
    """path: an .ncu-rep, or the CSV of `ncu -i <rep> --page raw --csv` (reduced on the
    GPU box to keep gpurun_out small)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    d[k] = r[i]
        if "dram__bytes_read.sum" in d:
            d["traffic_bytes"] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
            if algorithmic:
                d["algorithmic_bytes"] = algorithmic
                d["traffic_over_algorithmic"] = d["traffic_bytes"] / algorithmic
        res.append(d)
    return {"source": path, "captures": res}


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
        print(json.dumps(full(sys.argv[2], alg), indent=1))
