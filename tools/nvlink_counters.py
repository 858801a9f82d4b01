"""Calibrate NVML's NVLink byte counters against a known transfer (2 GPUs, one process).

Reads, per link, the NVLink5-era counters NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES /
RCV_BYTES (fields 202 / 204) and the older THROUGHPUT_DATA_TX / RX (138 / 139, KiB)
before and after a 1 GiB device-to-device copy GPU0 -> GPU1, and prints one JSON line per
counter family with the bytes each GPU saw, so bench.py can report measured NVLink bytes
per launch beside the algorithmic ones.  Usage: python tools/nvlink_counters.py
"""
import json
import time

import pynvml
import torch

FIELDS = {"count_bytes": (202, 204, 1), "throughput_kib": (138, 139, 1024),
          "throughput_raw_kib": (140, 141, 1024)}


def handle(dev):
    uuid = str(torch.cuda.get_device_properties(dev).uuid)
    try:
        return pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
    except Exception:   # noqa: BLE001
        return pynvml.nvmlDeviceGetHandleByIndex(dev)


def read(h, nlinks):
    out = {}
    for name, (tx, rx, scale) in FIELDS.items():
        ids = [(tx, l) for l in range(nlinks)] + [(rx, l) for l in range(nlinks)]
        try:
            vals = pynvml.nvmlDeviceGetFieldValues(h, ids)
        except pynvml.NVMLError as e:
            out[name] = {"error": str(e)}
            continue
        t = r = 0
        bad = 0
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                bad += 1
                continue
            x = int(v.value.ullVal) * scale
            if i < nlinks:
                t += x
            else:
                r += x
        out[name] = {"tx": t, "rx": r, "failed_fields": bad}
    return out


def main():
    pynvml.nvmlInit()
    hs = [handle(d) for d in range(2)]
    nl = []
    for h in hs:
        v = pynvml.nvmlDeviceGetFieldValues(h, [91])[0]
        nl.append(int(v.value.uiVal) if v.nvmlReturn == 0 else 18)
    n = 1 << 28   # 1 GiB of fp32
    a = torch.randn(n, device="cuda:0")
    b = torch.empty(n, device="cuda:1")
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    time.sleep(0.5)
    before = [read(h, k) for h, k in zip(hs, nl)]
    reps = 4
    for _ in range(reps):
        b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    time.sleep(1.5)   # counters may update lazily
    after = [read(h, k) for h, k in zip(hs, nl)]
    moved = reps * n * 4
    for name in FIELDS:
        row = {"family": name, "bytes_moved": moved, "links": nl}
        for d in range(2):
            if "error" in before[d][name] or "error" in after[d][name]:
                row[f"gpu{d}"] = before[d][name].get("error") or after[d][name].get("error")
                continue
            row[f"gpu{d}"] = {k: (after[d][name][k] - before[d][name][k]) / moved
                              for k in ("tx", "rx")}
            row[f"gpu{d}"]["failed_fields"] = after[d][name]["failed_fields"]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
