import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run via gpurun")
    config.addinivalue_line("markers", "multigpu: multi-process path (one rank per GPU; time-sliced ranks on a one-GPU box)")


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)


def mp_world():
    """World size of the multi-process tests: one rank per visible GPU (at most 8), or two
    ranks sharing the only GPU -- separate processes and CUDA contexts, time-sliced by
    the GPU -- so that a one-GPU box still runs the cross-process path (job server, CUDA
    IPC mappings, cross-process flag barriers), if not NVLink."""
    import torch
    return max(2, min(torch.cuda.device_count(), 8))


def rank_device(rank):
    """Select and return the device of `rank` in a multi-process test (rank mod GPUs)."""
    import torch
    d = rank % torch.cuda.device_count()
    torch.cuda.set_device(d)
    return f"cuda:{d}"
