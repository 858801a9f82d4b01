"""Second workload through the library on the GPU (S:418-426,
S:480): synchronous data-parallel momentum SGD on a synthetic least-squares problem.
Each of N ranks computes the gradient of its own b samples (the "training task part"
of Algorithm 1, here plain torch on the GPU), and gdraa_vr_sgd_step averages and
applies them.  The trajectory must match serial float64 SGD on batches of N*b samples
within 1e-5, and every rank must hold bitwise identical weights.
"""
import numpy as np
import pytest
import torch

from synth.least_squares import Problem
from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs a CUDA GPU")]

if has_cuda():
    from paper_1802_02326_b200 import gdraa

DEV = "cuda:0"


def serial_trajectory(P, iters, N, b, lr, mom):
    w, v, out = np.zeros(P.d), np.zeros(P.d), []
    for it in range(iters):
        X, y = P.batch(it, N, b)
        v = mom * v + X.T @ (X @ w - y) / X.shape[0]
        w = w - lr * v
        out.append(w.copy())
    return out


@pytest.mark.parametrize("N,b", [(4, 8), (2, 16), (8, 4)])
def test_least_squares_ssgd_matches_serial(N, b):
    P = Problem(seed=3)
    lr, mom, iters = 0.05, 0.9, 100
    ref = serial_trajectory(P, iters, N, b, lr, mom)
    w = [torch.zeros(P.d, device=DEV) for _ in range(N)]
    v = [torch.zeros(P.d, device=DEV) for _ in range(N)]
    g = [torch.zeros(P.d, device=DEV) for _ in range(N)]
    gap = 0.0
    for it in range(iters):
        for r in range(N):
            X, y = P.batch(it, N, b, rank=r)
            Xt = torch.from_numpy(X.astype(np.float32)).to(DEV)
            yt = torch.from_numpy(y.astype(np.float32)).to(DEV)
            g[r].copy_(Xt.T @ (Xt @ w[r] - yt) / b)
        gdraa.gdraa_vr_sgd_step(w, g, v, lr, mom)
        torch.cuda.synchronize()
        w0 = w[0].cpu().numpy()
        for r in range(1, N):
            assert np.array_equal(w[r].cpu().numpy().view(np.uint32), w0.view(np.uint32))
        gap = max(gap, float(np.max(np.abs(w0 - ref[it]))))
    assert gap < 1e-5, gap
    r = P.X @ ref[-1] - P.y
    assert 0.5 * np.mean(r * r) < 1e-3
