"""Run by test_gpu_kernels.py in a subprocess with GDRAA_LL128=1 (read once per process):
virtual-rank parity of the LL128 line format of the small-message allreduce_mean -- every
world size, both dtypes, ragged sizes around the 120-byte line and up to the LL
threshold, and chains of calls (the two slot parities alternate)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1802_02326_b200 import gdraa  # noqa: E402
from tests._parity import compare  # noqa: E402
from tests.test_gpu_parity import from_dev, make_grads, to_dev  # noqa: E402


def main():
    assert os.environ.get("GDRAA_LL128") == "1"
    count = 0
    for N in range(2, 9):
        lim = gdraa.gdraa_small_message_bytes(N)
        for dt in ("f32", "bf16"):
            bf16 = dt == "bf16"
            es = 2 if bf16 else 4
            sizes = [1, 2, 3, 29, 30, 31, 59, 60, 61, 257, 4097, 70_001, lim // es]
            if bf16:
                sizes += [119, 120, 121]
            for i, L in enumerate(sizes):
                for fam in ("like", "int"):
                    for step in range(3 if L == 4097 else 1):   # chained: both parities
                        gs = make_grads(fam, 900 + 10 * N + i + 100 * step, N, L, bf16)
                        bufs = [to_dev(g, bf16) for g in gs]
                        gdraa.gdraa_vr_allreduce_mean(bufs)
                        torch.cuda.synchronize()
                        exp = oracle.allreduce_mean(gs)
                        for r in range(N):
                            compare(from_dev(bufs[r]), exp, dt,
                                    what=f"ll128 mean N={N} {dt} L={L} {fam} r{r}")
                        count += 1
    # the LL128 form of the small-message SGD step (fp32 g, fp32 w, with weight decay)
    import synth
    for N in range(2, 9):
        lim = gdraa.gdraa_small_step_bytes(N) // 4
        for i, L in enumerate([1, 29, 30, 31, 61, 64 * N + 1, 257, 4097, 70_001, lim]):
            gs = make_grads("like" if i % 2 else "int", 700 + 10 * N + i, N, L, False)
            w0, v0 = synth.w_like(700 + N, L), synth.w_like(701 + N, L)
            w_exp, v_exp = oracle.sgd_step_wd(gs, w0, v0, 0.1, 0.9, 0.001)
            g_d = [to_dev(g) for g in gs]
            w_d = [to_dev(w0) for _ in range(N)]
            v_d = [to_dev(v0) for _ in range(N)]
            gdraa.gdraa_vr_sgd_step_ex(w_d, g_d, v_d, 0.1, 0.9, 0.001)
            torch.cuda.synchronize()
            for r in range(N):
                off, ln = gdraa.gdraa_shard(N, r, L)
                compare(from_dev(w_d[r]), w_exp, "f32", what=f"ll128 sgd w N={N} L={L} r{r}")
                compare(from_dev(v_d[r])[off:off + ln], v_exp[off:off + ln], "f32",
                        what=f"ll128 sgd v N={N} L={L} r{r}")
                outside = np.concatenate([from_dev(v_d[r])[:off], from_dev(v_d[r])[off + ln:]])
                assert np.array_equal(outside.view(np.uint32), np.concatenate(
                    [v0[:off], v0[off + ln:]]).view(np.uint32)), "v outside the shard"
                assert np.array_equal(from_dev(g_d[r]).view(np.uint32), gs[r].view(np.uint32))
            count += 1

    # LL128 mean calls interleaved with small-message SGD steps on the same
    # receive slots (fp32 steps: LL128 lines, the bf16 step: LL entries): each result must
    # still be the oracle's
    for N in (2, 3, 4, 8):
        L = 4097
        w0, v0 = synth.w_like(950 + N, L), synth.w_like(951 + N, L)
        w_d = [to_dev(w0) for _ in range(N)]
        v_d = [to_dev(v0) for _ in range(N)]
        w_ref, v_ref = w0.copy(), v0.copy()
        for step in range(6):
            bf = step == 3   # one step with bf16 gradients: LL entries, not LL128 lines
            gs = make_grads("like", 960 + 10 * N + step, N, L, bf)
            if step % 2 == 0:
                bufs = [to_dev(g) for g in gs]
                gdraa.gdraa_vr_allreduce_mean(bufs)
                torch.cuda.synchronize()
                exp = oracle.allreduce_mean(gs)
                for r in range(N):
                    compare(from_dev(bufs[r]), exp, "f32", what=f"mixed mean N={N} s{step} r{r}")
            else:
                g_d = [to_dev(g, bf) for g in gs]
                gdraa.gdraa_vr_sgd_step(w_d, g_d, v_d, 0.1, 0.9)
                torch.cuda.synchronize()
                w_ref, v_new = oracle.sgd_step(gs, w_ref, v_ref, 0.1, 0.9)
                for r in range(N):
                    off, ln = gdraa.gdraa_shard(N, r, L)
                    compare(from_dev(w_d[r]), w_ref, "f32", what=f"mixed sgd w N={N} s{step}")
                    compare(from_dev(v_d[r])[off:off + ln], v_new[off:off + ln], "f32",
                            what=f"mixed sgd v N={N} s{step}")
                v_ref = v_new
            count += 1
    print(f"OK ll128 {count} cases")


if __name__ == "__main__":
    main()
