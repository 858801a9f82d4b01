"""Second workload data: a synthetic
least-squares problem for synchronous data-parallel SGD, whose serial large-batch run
must coincide with the N-rank GDRAA run (each rank: b samples of the same N*b).

Data only -- no gradient, no mean, no update: each side of a test computes those itself.
"""
import numpy as np

from . import normal


class Problem:
    """X (M x d) ~ N(0,1), y = X w* + 0.01 noise; global batches are taken in order."""

    def __init__(self, seed=0, M=4096, d=16):
        self.M, self.d = M, d
        self.X = normal(seed, 0, 201, M * d).reshape(M, d)
        self.w_star = normal(seed, 0, 202, d)
        self.y = self.X @ self.w_star + 0.01 * normal(seed, 0, 203, M)

    def batch(self, it, N, b, rank=None):
        """Iteration it's global batch of N*b rows (or rank's b-row slice of it): the
        deterministic sharding S:420 asks for (rank r gets rows [r*b, (r+1)*b))."""
        B = N * b
        idx = (it * B + np.arange(B)) % self.M
        if rank is not None:
            idx = idx[rank * b:(rank + 1) * b]
        return self.X[idx], self.y[idx]
