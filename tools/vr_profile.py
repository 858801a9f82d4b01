"""One virtual-rank call of the hot path on one GPU, for an ncu capture of the N >= 2
kernels' on-chip and HBM behaviour (all N ranks' buffers in this GPU's HBM, the same
kernel code as the multi-process path; DESIGN.md §6 "Virtual ranks").

    ncu --set full -k regex:gdraa_tma_kernel --launch-skip 2 -c 1 \
        python tools/vr_profile.py [N=4] [config=r50] [calls=3]

config: r50 (fp32 sgd_step), r50bf16mp (bf16 g, sgd_step_mp with weight decay), r101.
Prints the algorithmic HBM bytes of one launch (every rank's g read once by its owner,
the owner shards of w/master and v read and written, every rank's w' / bf16 copy written
once): the figure ncu's dram bytes are compared with.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1802_02326_b200 import gdraa  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = sys.argv[2] if len(sys.argv) > 2 else "r50"
    calls = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    L = synth.L_R101 if cfg == "r101" else synth.L_R50
    mp = cfg == "r50bf16mp"
    dev = torch.device("cuda:0")
    gdt = torch.bfloat16 if mp else torch.float32
    g = [torch.randn(L, device=dev).to(gdt) * 1e-3 for _ in range(N)]
    v = [torch.zeros(L, device=dev) for _ in range(N)]
    if mp:
        wm = [torch.randn(L, device=dev) * 0.05 for _ in range(N)]
        model = [torch.zeros(L, dtype=torch.bfloat16, device=dev) for _ in range(N)]
    else:
        w0 = torch.randn(L, device=dev) * 0.05
        w = [w0.clone() for _ in range(N)]
    for _ in range(calls):
        if mp:
            gdraa.gdraa_vr_sgd_step_mp(wm, model, g, v, synth.PAPER_LR, synth.PAPER_MOM, 0.001)
        else:
            gdraa.gdraa_vr_sgd_step(w, g, v, synth.PAPER_LR, synth.PAPER_MOM)
    torch.cuda.synchronize()
    s_g, s_w = (2, 2) if mp else (4, 4)
    hbm = L * (N * s_g + (16 if mp else 12) + N * s_w)
    print(json.dumps({"vr_profile": cfg, "N": N, "L": L, "calls": calls,
                      "algorithmic_hbm_bytes_per_launch": hbm,
                      "note": "every g byte read once by its owner; owner shards of "
                              + ("master w and v read+written (16 B/elt); " if mp else
                                 "w read and v read+written (12 B/elt); ")
                              + f"w' ({s_w} B) written into all N ranks"}))


if __name__ == "__main__":
    main()
