"""Summarise which algorithm / protocol NCCL chose per all_reduce size from an
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING log (stderr of tools/sweep.py), plus the
init lines that say whether NVLS (NVSwitch multicast/in-switch reduction) is in use.

    python tools/nccl_algos.py sweep.err > summary.json
"""
import collections
import json
import re
import sys


def main(path):
    init, raw, choices = [], [], collections.OrderedDict()
    pat = re.compile(r"(AllReduce)\D*?(\d+)\s*Bytes.*?[Aa]lgo\s*(\w+).*?[Pp]roto\s*(\w+)")
    for line in open(path, errors="replace"):
        if "NCCL INFO" not in line:
            continue
        low = line.lower()
        if "nvls" in low or "version" in low or "channels" in low or "collnet" in low:
            if len(init) < 60:
                init.append(line.split("NCCL INFO", 1)[1].strip())
        if "allreduce" in low and len(raw) < 12:
            raw.append(line.split("NCCL INFO", 1)[1].strip())
        m = pat.search(line)
        if m:
            choices.setdefault(int(m.group(2)), collections.Counter())[
                f"{m.group(3)}/{m.group(4)}"] += 1
    print(json.dumps({"log": path, "init": init, "allreduce_lines": raw,
                      "allreduce_choices": {str(k): dict(v) for k, v in choices.items()}},
                     indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
