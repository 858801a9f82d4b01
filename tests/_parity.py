"""Comparison helpers for GPU-vs-oracle parity (AMB-14).

The pass bar is the north star's tolerance: max relative error 1e-6 (fp32) and 1e-2
(bf16), rel = max_i |x_i - y_i| / max(|y_i|, FLT_MIN).  Because the kernel pins the
summation order and every rounding, the path is expected to be bit-exact, so `exact=True`
(the default) additionally requires zero mismatching bit patterns.
"""
import numpy as np

TOL = {"f32": 1e-6, "bf16": 1e-2}
FLT_MIN = np.float32(1.17549435e-38)


def as_f32(x, dtype):
    x = np.asarray(x)
    if dtype == "bf16":
        return (x.astype(np.uint32) << np.uint32(16)).view(np.float32)
    return x.astype(np.float32, copy=False)


def compare(got, exp, dtype="f32", exact=True, what=""):
    got = np.ascontiguousarray(got)
    exp = np.ascontiguousarray(exp)
    assert got.shape == exp.shape, (what, got.shape, exp.shape)
    gf, ef = as_f32(got, dtype), as_f32(exp, dtype)
    denom = np.maximum(np.abs(ef), FLT_MIN)
    rel = float(np.max(np.abs(gf.astype(np.float64) - ef) / denom)) if got.size else 0.0
    assert rel <= TOL[dtype], f"{what}: max rel err {rel:.3g} > {TOL[dtype]}"
    if exact:
        gb = got.view(np.uint16 if dtype == "bf16" else np.uint32)
        eb = exp.view(np.uint16 if dtype == "bf16" else np.uint32)
        bad = np.flatnonzero(gb != eb)
        assert bad.size == 0, (f"{what}: {bad.size} of {got.size} elements differ bitwise "
                               f"(first at {bad[:5].tolist()}: got {gf[bad[:5]]} exp {ef[bad[:5]]})")
    return rel
