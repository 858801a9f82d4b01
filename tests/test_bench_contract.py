"""bench.py's JSON line keeps the driver's contract: the reference arm on
the CPU here, our arm on a GPU (small config, few steps, both timing modes)."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         env=env, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "3", "--warmup", "3"], 600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "c1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == d["value"]
    assert cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["graph", "eager"])
def test_our_arm_line(mode):
    steps = 20
    d = _run(["--config", "c1", "--steps", str(steps), "--warmup", "3", "--e2e-steps", "3",
              "--no-cpu-baseline"] + (["--eager"] if mode == "eager" else []), 900)
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["config"]["path"] == "local"
    assert ("graph" in d["config"]["timing"]) == (mode == "graph")
    assert d["gpu_launches"] == steps                     # one fused kernel per step
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert r["achieved"] == pytest.approx(r["bytes_per_launch"] / (d["ms_per_step"] * 1e-3) / 1e9)
    assert d["value"] == pytest.approx(r["achieved"])     # N = 1: whole job = one rank
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    pc = d["per_call"]
    assert pc["p10_us"] <= pc["median_us"] <= pc["p90_us"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
