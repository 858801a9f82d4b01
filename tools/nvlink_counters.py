"""Calibrate NVML's NVLink byte counters against a known transfer (2 GPUs, one process).

Two NVML sources are tried around 4 x 1 GiB device-to-device copies GPU0 -> GPU1:
(1) the per-link field values NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / RCV_BYTES (202 / 204)
and THROUGHPUT_DATA_TX / RX (138 / 139, KiB); (2) GPU Performance Monitoring (GPM)
samples, NVML_GPM_METRIC_NVLINK_TOTAL_{RX,TX}_PER_SEC, whose average rate between two
samples times the wall time between them gives bytes.  One JSON line per source with the
measured bytes divided by the bytes copied (1.0 = exact), so bench.py can report measured
NVLink bytes per launch.  Usage: python tools/nvlink_counters.py
"""
import json
import time

import pynvml
import torch

FIELDS = {"count_bytes": (202, 204, 1), "throughput_kib": (138, 139, 1024)}


def handle(dev):
    uuid = str(torch.cuda.get_device_properties(dev).uuid)
    try:
        return pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
    except Exception:   # noqa: BLE001
        return pynvml.nvmlDeviceGetHandleByIndex(dev)


def read_fields(h, nlinks):
    out = {}
    for name, (tx, rx, scale) in FIELDS.items():
        ids = [(tx, l) for l in range(nlinks)] + [(rx, l) for l in range(nlinks)]
        try:
            vals = pynvml.nvmlDeviceGetFieldValues(h, ids)
        except pynvml.NVMLError as e:
            out[name] = {"error": str(e)}
            continue
        codes = sorted({int(v.nvmlReturn) for v in vals})
        t = sum(int(v.value.ullVal) for v in vals[:nlinks] if v.nvmlReturn == 0) * scale
        r = sum(int(v.value.ullVal) for v in vals[nlinks:] if v.nvmlReturn == 0) * scale
        out[name] = {"tx": t, "rx": r, "return_codes": codes}
    return out


class Gpm:
    def __init__(self, h):
        self.h, self.err = h, None
        try:
            sup = pynvml.nvmlGpmQueryDeviceSupport(h)
            self.ok = bool(sup.isSupportedDevice)
            if not self.ok:
                self.err = "GPM not supported on this device"
        except Exception as e:   # noqa: BLE001
            self.ok, self.err = False, f"nvmlGpmQueryDeviceSupport: {e}"

    def sample(self):
        try:
            s = pynvml.nvmlGpmSampleAlloc()
            pynvml.nvmlGpmSampleGet(self.h, s)
        except Exception as e:   # noqa: BLE001
            self.ok, self.err = False, f"nvmlGpmSampleGet: {e}"
            return None
        return s, time.perf_counter()

    def rates(self, a, b):
        mg = pynvml.c_nvmlGpmMetricsGet_t()
        mg.version = pynvml.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1, mg.sample2 = a[0], b[0]
        mg.metrics[0].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        mg.metrics[1].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        pynvml.nvmlGpmMetricsGet(mg)
        m = mg.metrics
        return {"tx_rate": m[0].value, "rx_rate": m[1].value,
                "codes": [int(m[0].nvmlReturn), int(m[1].nvmlReturn)],
                "unit": str(m[0].metricInfo.unit) if hasattr(m[0], "metricInfo") else None,
                "seconds": b[1] - a[1]}


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
    reps = 4
    moved = reps * n * 4

    gpms = [Gpm(h) for h in hs]
    time.sleep(0.5)
    before = [read_fields(h, k) for h, k in zip(hs, nl)]
    g0 = [g.sample() if g.ok else None for g in gpms]
    for _ in range(reps):
        b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    g1 = [g.sample() if g.ok else None for g in gpms]
    time.sleep(1.5)   # field counters may update lazily
    after = [read_fields(h, k) for h, k in zip(hs, nl)]

    for name in FIELDS:
        row = {"source": "fields:" + name, "bytes_moved": moved, "links": nl}
        for d in range(2):
            x, y = before[d][name], after[d][name]
            if "error" in x or "error" in y:
                row[f"gpu{d}"] = x.get("error") or y.get("error")
                continue
            row[f"gpu{d}"] = {k: (y[k] - x[k]) / moved for k in ("tx", "rx")}
            row[f"gpu{d}"]["return_codes"] = y["return_codes"]
        print(json.dumps(row), flush=True)
    row = {"source": "gpm:NVLINK_TOTAL_{TX,RX}_PER_SEC", "bytes_moved": moved}
    for d in range(2):
        if not gpms[d].ok or g0[d] is None or g1[d] is None:
            row[f"gpu{d}"] = gpms[d].err
            continue
        try:
            r = gpms[d].rates(g0[d], g1[d])
            r["tx_bytes_if_MiBps"] = r["tx_rate"] * 2**20 * r["seconds"] / moved
            r["rx_bytes_if_MiBps"] = r["rx_rate"] * 2**20 * r["seconds"] / moved
            row[f"gpu{d}"] = r
        except Exception as e:   # noqa: BLE001
            row[f"gpu{d}"] = f"nvmlGpmMetricsGet: {e}"
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
