"""The boundary from plain C: tests/c_abi_smoke.c includes only include/gdraa.h and the
CUDA runtime header and links only lib/libgdraa.so and libcudart -- no Python binding,
no torch.  CPU: the header compiles as strict C11 and the program links.  GPU: it runs
four virtual ranks through gdraa_vr_sgd_step and checks the exact closed form."""
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


def build(out):
    rt = _cudart_dir()
    if rt is None or not os.path.exists(os.path.join(LIB, "libgdraa.so")):
        pytest.skip("CUDA runtime or lib/libgdraa.so missing")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-pedantic",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           os.path.join(ROOT, "tests", "c_abi_smoke.c"), "-o", out,
           "-L", LIB, "-lgdraa", "-L", rt, "-lcudart", f"-Wl,-rpath,{LIB}:{rt}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_abi_compiles_and_links(tmp_path):
    build(str(tmp_path / "c_abi_smoke"))


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA GPU")
def test_c_abi_runs(tmp_path):
    exe = build(str(tmp_path / "c_abi_smoke"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr
