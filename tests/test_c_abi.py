"""The boundary from plain C: tests/c_abi_smoke.c and tests/c_abi_mp.c include only
include/gdraa.h and the CUDA runtime header and link only lib/libgdraa.so and libcudart
-- no Python binding, no torch.  CPU: the header compiles as strict C11 and both programs
link.  GPU: four virtual ranks through gdraa_vr_sgd_step, and the job server plus forked
rank processes through gdraa_init / register / sgd_step / allreduce_mean / finalize, each
checked against the exact closed form of integer-valued inputs."""
import os
import subprocess

import pytest

from tests.conftest import has_cuda

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1802_02326_b200", "lib")
CUDA = "/usr/local/cuda"


def _cudart_dir():
    for d in (os.path.join(CUDA, "lib64"), os.path.join(CUDA, "targets", "x86_64-linux", "lib")):
        if os.path.exists(os.path.join(d, "libcudart.so")):
            return d
    return None


def build(out, src="c_abi_smoke.c"):
    rt = _cudart_dir()
    if rt is None or not os.path.exists(os.path.join(LIB, "libgdraa.so")):
        pytest.skip("CUDA runtime or lib/libgdraa.so missing")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-pedantic",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           os.path.join(ROOT, "tests", src), "-o", out,
           "-L", LIB, "-lgdraa", "-L", rt, "-lcudart", f"-Wl,-rpath,{LIB}:{rt}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_abi_compiles_and_links(tmp_path):
    build(str(tmp_path / "c_abi_smoke"))
    build(str(tmp_path / "c_abi_mp"), "c_abi_mp.c")


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA GPU")
def test_c_abi_runs(tmp_path):
    exe = build(str(tmp_path / "c_abi_smoke"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA GPU")
def test_c_abi_multiprocess(tmp_path):
    """Job server + `world` forked rank processes, all from C (world 4 on a 4-GPU box,
    else 2; ranks share GPUs round-robin, time-sliced)."""
    import torch
    exe = build(str(tmp_path / "c_abi_mp"), "c_abi_mp.c")
    world = 4 if torch.cuda.device_count() >= 4 else 2
    js = os.path.join(LIB, "gdraa_jobserver")
    r = subprocess.run([exe, js, str(world)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
