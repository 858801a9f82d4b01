#!/usr/bin/env python
"""A small sweep over every kernel of the library (two-shot LSU / TMA per GDRAA_KERNEL,
the LL mean, the LL SGD step, every mode and dtype) through the single-GPU virtual-rank
entry points, for compute-sanitizer:

    GDRAA_KERNEL=tma compute-sanitizer --tool memcheck python tools/sanitize_run.py
    GDRAA_KERNEL=lsu compute-sanitizer --tool racecheck python tools/sanitize_run.py

Results are checked against the CPU oracle, so a clean sanitizer run is also a parity run.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1802_02326_b200 import gdraa  # noqa: E402
from tests._parity import compare  # noqa: E402
from tests.test_gpu_parity import from_dev, make_grads, to_dev  # noqa: E402

DEV = "cuda:0"


def main():
    n_cases = 0
    # 777 and 3001: LL paths; 200_003: two-shot (above the LL limits once disabled below)
    for N in (2, 3, 4):
        for dt in ("f32", "bf16"):
            bf16 = dt == "bf16"
            for L in (777, 3001, 200_003):
                gs = make_grads("like", 50 + N, N, L, bf16)
                w0, v0 = synth.w_like(51, L), synth.w_like(52, L)
                w_exp, v_exp, m_exp = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001,
                                                         model_dtype=oracle.BF16)
                g_d = [to_dev(g, bf16) for g in gs]
                w_d = [to_dev(w0) for _ in range(N)]
                v_d = [to_dev(v0) for _ in range(N)]
                gdraa.gdraa_vr_sgd_step_ex(w_d, g_d, v_d, 0.1, 0.9, 0.001)
                wm_d = [to_dev(w0) for _ in range(N)]
                vm_d = [to_dev(v0) for _ in range(N)]
                mo_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
                gdraa.gdraa_vr_sgd_step_mp(wm_d, mo_d, g_d, vm_d, 0.1, 0.9, 0.001)
                bufs = [to_dev(g, bf16) for g in gs]
                gdraa.gdraa_vr_allreduce_mean(bufs)
                torch.cuda.synchronize()
                mean_exp = oracle.allreduce_mean(gs)
                for r in range(N):
                    off, ln = gdraa.gdraa_shard(N, r, L)
                    compare(from_dev(w_d[r]), w_exp, "f32", what=f"w N={N} {dt} L={L} r{r}")
                    compare(from_dev(v_d[r])[off:off + ln], v_exp[off:off + ln], "f32", what="v")
                    compare(from_dev(mo_d[r]), m_exp, "bf16", what="mp model")
                    compare(from_dev(wm_d[r])[off:off + ln], w_exp[off:off + ln], "f32",
                            what="mp master")
                    compare(from_dev(bufs[r]), mean_exp, dt, what="mean")
                    assert np.array_equal(from_dev(g_d[r]), gs[r])
                n_cases += 1
    print(f"sanitize_run OK: {n_cases} cases, kernel={os.environ.get('GDRAA_KERNEL', 'auto')}")


if __name__ == "__main__":
    main()
