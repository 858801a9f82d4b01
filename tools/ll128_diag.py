"""Locate the LL128 SGD transition fault: virtual ranks on one GPU run
LL-format small-message SGD steps, then LL128 steps (GDRAA_LL128=auto must be set), and
every mismatch with the oracle is mapped to (block owner, line, lane, element in lane).

    GDRAA_LL128=auto python tools/ll128_diag.py [N=4] [tries=5] [--full]
"""
import json
import os
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1802_02326_b200 import gdraa  # noqa: E402


def main():
    assert os.environ.get("GDRAA_LL128") == "auto"
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    N = int(args[0]) if args else 4
    tries = int(args[1]) if len(args) > 1 else 5
    lim = gdraa.gdraa_small_step_bytes(N) // 4
    dev = "cuda:0"
    for t in range(tries):
        # the failing test's exact sequence (tests/test_gpu_parity.py::
        # test_vr_sgd_latency_path): every size 3 times, LL-format up to 65537
        sizes = [1, 3, 63, 65, 127, 4097, 65_537] if "--full" in sys.argv else [65_537]
        seq = [L for L in sizes for _ in range(3)] + [lim - 1] * 3
        w = synth.w_like(901 + t, 1)  # placeholder, reset per size below
        size_prev = None
        for step, L in enumerate(seq):
            if L != size_prev:
                w, v = synth.w_like(901, L), synth.w_like(902, L)
                w_d = [torch.from_numpy(w).to(dev) for _ in range(N)]
                v_d = [torch.from_numpy(v).to(dev) for _ in range(N)]
                size_prev = L
            it = step % 3
            from tests.test_gpu_parity import make_grads
            gs = make_grads("like", (900 + L % 13) if it == 0 else (910 + it), N, L, False)
            g_d = [torch.from_numpy(g).to(dev) for g in gs]
            gdraa.gdraa_vr_sgd_step_ex(w_d, g_d, v_d, 0.1, 0.9, 0.001)
            torch.cuda.synchronize()
            w, v_new = oracle.sgd_step_wd(gs, w, v, 0.1, 0.9, 0.001)
            blk = gdraa.gdraa_shard(N, 0, L)[1]
            out = {"try": t, "step": step, "L": L, "path": "ll128" if L == lim - 1 else "ll"}
            for r in range(N):
                got = w_d[r].cpu().numpy()
                bad = np.nonzero(got.view(np.uint32) != w.view(np.uint32))[0]
                if len(bad) == 0:
                    continue
                owner = bad // blk
                rel = bad - owner * blk
                line, within = rel // 30, rel % 30
                lane = np.minimum(within // 4, 7)
                out[f"r{r}"] = {"bad": int(len(bad)), "owners": dict(Counter(owner.tolist())),
                                "lanes": dict(Counter(lane.tolist())),
                                "lines_min_max": [int(line.min()), int(line.max())],
                                "first": int(bad[0]),
                                "got_first": float(got[bad[0]]), "exp_first": float(w[bad[0]])}
                off, ln = gdraa.gdraa_shard(N, r, L)
                out[f"r{r}"]["own_v_bad"] = int(np.count_nonzero(
                    v_d[r].cpu().numpy()[off:off + ln].view(np.uint32)
                    != v_new[off:off + ln].view(np.uint32)))
            v = v_new
            print(json.dumps(out), flush=True)
            # keep going from the GPU state so later steps show whether errors persist
            w = w_d[0].cpu().numpy().copy()


if __name__ == "__main__":
    main()
