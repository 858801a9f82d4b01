"""Run by test_gpu_kernels.py in a subprocess with GDRAA_KERNEL forced (the choice is
read once per process): a compact virtual-rank parity sweep of every mode through the
forced data-movement variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1802_02326_b200 import gdraa  # noqa: E402
from tests._parity import compare  # noqa: E402
from tests.test_gpu_parity import from_dev, make_grads, to_dev  # noqa: E402

DEV = "cuda:0"


def main():
    count = 0
    for N in (1, 2, 3, 4, 8):
        for dt in ("f32", "bf16"):
            bf16 = dt == "bf16"
            for L in (257, 70_001, 1_000_003):
                gs = make_grads("like", 800 + N, N, L, bf16)
                # sgd (+ weight decay)
                w0, v0 = synth.w_like(800, L), synth.w_like(801, L)
                w_exp, v_exp, m_exp = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001,
                                                         model_dtype=oracle.BF16)
                g_d = [to_dev(g, bf16) for g in gs]
                w_d = [to_dev(w0) for _ in range(N)]
                v_d = [to_dev(v0) for _ in range(N)]
                gdraa.gdraa_vr_sgd_step_ex(w_d, g_d, v_d, 0.1, 0.9, 0.001)
                # mixed precision
                wm_d = [to_dev(w0) for _ in range(N)]
                vm_d = [to_dev(v0) for _ in range(N)]
                mo_d = [torch.zeros(L, dtype=torch.bfloat16, device=DEV) for _ in range(N)]
                gdraa.gdraa_vr_sgd_step_mp(wm_d, mo_d, g_d, vm_d, 0.1, 0.9, 0.001)
                # mean (sizes above the latency-path threshold use the two-shot kernel)
                bufs = [to_dev(g, bf16) for g in gs]
                gdraa.gdraa_vr_allreduce_mean(bufs)
                torch.cuda.synchronize()
                mean_exp = oracle.allreduce_mean(gs)
                for r in range(N):
                    off, ln = gdraa.gdraa_shard(N, r, L)
                    compare(from_dev(w_d[r]), w_exp, "f32", what=f"w N={N} {dt} L={L} r{r}")
                    compare(from_dev(v_d[r])[off:off + ln], v_exp[off:off + ln], "f32",
                            what="v")
                    compare(from_dev(mo_d[r]), m_exp, "bf16", what="mp model")
                    compare(from_dev(wm_d[r])[off:off + ln], w_exp[off:off + ln], "f32",
                            what="mp master")
                    compare(from_dev(bufs[r]), mean_exp, dt, what="mean")
                # the same step as two buckets inside a bucket set (deferred exit barrier)
                w_d = [to_dev(w0) for _ in range(N)]
                v_d = [to_dev(v0) for _ in range(N)]
                half = L // 2 // 8 * 8
                gdraa.gdraa_vr_bucket_set_begin(N)
                for first, cnt in ((half, L - half), (0, half)):
                    if cnt:
                        gdraa.gdraa_vr_sgd_step_range(w_d, g_d, v_d, first, cnt, 0.1, 0.9, 0.001)
                gdraa.gdraa_vr_bucket_set_end(N)
                torch.cuda.synchronize()
                for r in range(N):
                    compare(from_dev(w_d[r]), w_exp, "f32", what=f"set w N={N} {dt} L={L} r{r}")
                count += 1
    print(f"OK {os.environ.get('GDRAA_KERNEL')} {count} cases")


if __name__ == "__main__":
    main()
