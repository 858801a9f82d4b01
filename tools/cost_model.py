#!/usr/bin/env python
"""alpha-beta cost model of one GDRAA allreduce (the simulator
idea of S:269-300, here in closed form) fitted to the config-5 sweep.

    t(S) = alpha + B_nv(S) / beta,   B_nv(S) = 2 (N-1)/N * S   (bytes per rank per direction)

alpha collects the per-call constants (launch gap, the two device synchronisations,
pipeline fill/drain); beta is the NVLink rate the data phase sustains.  Paper assumption
1 ("latency is tiny compared to transfer") holds where B_nv/beta >> alpha.

    python tools/cost_model.py profiles/r06_sweep_c5_n4.jsonl [...]  > profiles/cost_model.json
"""
import json
import sys

import numpy as np


def fit(lines, min_bytes=1 << 22):
    N = lines[0]["n_gpus"]
    S = np.array([l["bytes"] for l in lines], float)
    t = np.array([l["gdraa_us"] for l in lines], float) * 1e-6
    bnv = 2 * (N - 1) / N * S
    sel = S >= min_bytes
    A = np.stack([np.ones(sel.sum()), bnv[sel]], 1)
    (alpha, inv_beta), *_ = np.linalg.lstsq(A, t[sel], rcond=None)
    small = t[S <= 1 << 16]
    pred = alpha + bnv * inv_beta
    out = {
        "n_gpus": N,
        "alpha_us_fit": alpha * 1e6,
        "alpha_us_small_msgs": float(np.median(small)) * 1e6 if small.size else None,
        "beta_gbs_fit": 1 / inv_beta / 1e9,
        "fit_range_bytes": [int(S[sel].min()), int(S[sel].max())],
        "max_rel_err_fit_range": float(np.max(np.abs(pred[sel] - t[sel]) / t[sel])),
        "half_efficiency_bytes": float(alpha / inv_beta * N / (2 * (N - 1))),
        "rows": [{"bytes": int(s), "measured_us": float(a * 1e6), "model_us": float(p * 1e6)}
                 for s, a, p in zip(S, t, pred)],
    }
    # NCCL on the same sizes, same model
    if "nccl_us" in lines[0]:
        tn = np.array([l["nccl_us"] for l in lines], float) * 1e-6
        (an, ibn), *_ = np.linalg.lstsq(A, tn[sel], rcond=None)
        out["nccl"] = {"alpha_us_fit": an * 1e6, "beta_gbs_fit": 1 / ibn / 1e9}
    return out


def main():
    res = []
    for path in sys.argv[1:]:
        lines = [json.loads(l) for l in open(path) if l.strip()]
        r = fit(lines)
        r["source"] = path
        res.append(r)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
