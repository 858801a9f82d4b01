"""SASS evidence for the default-path kernels of lib/libgdraa.so (cuobjdump -sass).

For each kernel instance the runtime launches on its default path, counts the
instruction classes that back the DESIGN.md claims (128-bit peer loads / stores, bulk
copies + mbarriers, system fences, the FP ops of the fold / update, and where the FFMA
come from), and saves a short excerpt of the inner loop.

    python tools/sass_summary.py [out_prefix]     # e.g. profiles/r98_sass
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1802_02326_b200", "lib", "libgdraa.so")

# (label, mangled-name regex): the kernels bench.py's configs and the small-message path run
DEFAULT_PATH = [
    ("N=1 local fused SGD, fp32 (gdraa_kernel<float,1,kSgd,U4,512,1>)",
     r"12gdraa_kernelIfLi1ELi1ELi4ELi512ELi1EEE"),
    ("N=2 two-shot fused SGD, fp32, TMA-staged (gdraa_tma_kernel<float,2,kSgd>)",
     r"16gdraa_tma_kernelIfLi2ELi1ELi16ELi4ELi4ELi4ELi0ELi0ELi40EEE"),
    ("N=4 two-shot fused SGD, fp32, TMA-staged (gdraa_tma_kernel<float,4,kSgd>)",
     r"16gdraa_tma_kernelIfLi4ELi1ELi16ELi4ELi4ELi4ELi0ELi0ELi40EEE"),
    ("N=2 two-shot fused SGD, bf16 g, TMA-staged (gdraa_tma_kernel<bf16,2,kSgd>)",
     r"16gdraa_tma_kernelI13__nv_bfloat16Li2ELi1ELi16ELi4ELi4ELi4ELi0ELi0ELi40EEE"),
    ("N=4 two-shot mixed-precision SGD, bf16 g (gdraa_tma_kernel<bf16,4,kSgdMp>)",
     r"16gdraa_tma_kernelI13__nv_bfloat16Li4ELi2ELi16ELi4ELi4ELi4ELi0ELi0ELi40EEE"),
    ("N=2 small-message SGD, fp32 (gdraa_ll_sgd_kernel<float,2,kSgd>)",
     r"19gdraa_ll_sgd_kernelIfLi2ELi1EEE"),
    ("N=2 small-message mean, fp32 (gdraa_ll_kernel<float,2>)",
     r"15gdraa_ll_kernelIfLi2EEE"),
    ("N=2 streamed bucket set, fp32 sgd (gdraa_tma_set_kernel<float,2,kSgd>)",
     r"20gdraa_tma_set_kernelIfLi2ELi1EEE"),
    ("bucket-set exit barrier (gdraa_exit_kernel)",
     r"17gdraa_exit_kernel"),
]

CLASSES = {
    "LDG.128 (incl. peer pulls)": r"\bLDG\.E[.\w]*\.128\b",
    "LDG.64": r"\bLDG\.E[.\w]*\.64\b",
    "STG.128 (incl. peer pushes)": r"\bSTG\.E[.\w]*\.128\b",
    "STG.64": r"\bSTG\.E[.\w]*\.64\b",
    "UBLKCP (cp.async.bulk)": r"\bUBLKCP\b",
    "SYNCS (mbarrier)": r"\bSYNCS\b",
    "MEMBAR.ALL.SYS / .SC.SYS": r"\bMEMBAR\.\w+\.SYS\b",
    "FENCE.VIEW.ASYNC": r"\bFENCE\.VIEW\.ASYNC",
    "FADD": r"\bFADD\b",
    "FMUL": r"\bFMUL\b",
    "FFMA": r"\bFFMA\b",
    "MUFU.RCP": r"\bMUFU\.RCP\b",
    "CALL (slow-path subroutine)": r"\bCALL\.",
    "ACQBULK": r"\bACQBULK\b",
    "PREEXIT": r"\bPREEXIT\b",
    "NANOSLEEP": r"\bNANOSLEEP\b",
}


def functions(sass):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur and re.match(r"\s+/\*[0-9a-f]{4}\*/", line):
            body.append(line.strip())
    if cur:
        yield cur, body


def main():
    prefix = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r62_sass")
    sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True,
                          check=True).stdout
    funcs = dict(functions(sass))
    summary = {"library": os.path.relpath(SO, ROOT), "kernels_in_library": len(funcs),
               "ll128_kernels": sum("ll128" in f for f in funcs), "default_path": []}
    excerpts = []
    for label, rx in DEFAULT_PATH:
        name = next((f for f in funcs if re.search(rx, f)), None)
        if name is None:
            summary["default_path"].append({"kernel": label, "missing": rx})
            continue
        body = funcs[name]
        counts = collections.OrderedDict()
        for k, pat in CLASSES.items():
            counts[k] = sum(1 for l in body if re.search(pat, l))
        # where the FFMA sit: inside __fdiv_rn's correctly-rounded reciprocal refinement
        # (next to MUFU.RCP / the slow-path CALL) vs anywhere else
        ffma_lines = [i for i, l in enumerate(body) if re.search(CLASSES["FFMA"], l)]
        rcp_lines = [i for i, l in enumerate(body) if re.search(r"MUFU\.RCP|CALL\.", l)]
        near = sum(1 for i in ffma_lines if any(abs(i - j) <= 12 for j in rcp_lines))
        summary["default_path"].append({
            "kernel": label, "mangled": name, "instructions": len(body),
            "counts": counts, "ffma_within_12_of_rcp_or_call": near,
            "ffma_total": len(ffma_lines)})
        # excerpt: the first 40 instructions around the first peer-store / bulk-copy site
        pos = next((i for i, l in enumerate(body) if re.search(r"UBLKCP|STG\.E[.\w]*\.128", l)), 0)
        excerpts.append(f"==== {label}\n==== {name}\n" + "\n".join(body[max(0, pos - 20):pos + 20]))
    with open(prefix + "_summary.json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(prefix + "_excerpts.txt", "w") as f:
        f.write("\n\n".join(excerpts) + "\n")
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
