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


def test_self_launch_without_torchrun():
    """`python bench.py --gpus N` with no WORLD_SIZE in the environment starts its own N
    ranks (torch.distributed.run on a free 127.0.0.1 port); exactly one JSON line comes
    back, from rank 0, with every rank present."""
    d = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--dry-launch"], 300)
    assert d["dry_launch"] and d["world"] == 2 and d["n_gpus"] == 2
    assert sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert sorted(r["local_rank"] for r in d["ranks"]) == [0, 1]
    assert all(r["master_addr"] == "127.0.0.1" for r in d["ranks"])


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
    assert d["value"] == pytest.approx(r["achieved"])     # per-rank rate of the launch
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    pc = d["per_call"]
    assert pc["p10_us"] <= pc["median_us"] <= pc["p90_us"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.skipif(not __import__("tests.conftest", fromlist=["x"]).has_cuda()
                    or __import__("torch").cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_our_arm_self_launched_n2():
    """The driver's form `python bench.py --gpus 2` (no torchrun): NVLink roofline line."""
    d = _run(["--gpus", "2", "--steps", "20", "--warmup", "5", "--e2e-steps", "3"], 900)
    assert d["n_gpus"] == 2 and d["config"]["path"] == "two_shot"
    r = d["roofline"]
    assert r["bound"] == "nvlink" and r["peak"] == 770.0 and 0 < r["frac"] < 1.2
    assert "frac_of_nominal_900" in r
    assert d["value"] == pytest.approx(r["achieved"]) == pytest.approx(d["bus_gbs_per_rank"])
    assert d["job_total_gbs"] == pytest.approx(2 * d["value"])
    assert d["nccl_reference"]["bus_gbs_per_rank"] > 0
