"""Build the native parts of the package, in-tree (so the .so travels with gpurun):

  lib/libgdraa.so      C-ABI library (include/gdraa.h): runtime + sm_100a kernels
  lib/gdraa_jobserver  job-server control plane (no CUDA)

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo (cross-compiles without a GPU).
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
SO = os.path.join(LIB, "libgdraa.so")
JOBSERVER = os.path.join(LIB, "gdraa_jobserver")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-Wall",
              "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]

SOURCES = ["gdraa_runtime.cu", "gdraa_kernels.cu"]
HEADERS = ["gdraa_internal.h", "jobserver_proto.h"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    os.makedirs(LIB, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + \
        [os.path.join(ROOT, "include", "gdraa.h"), __file__]
    if force or _stale(SO, deps):
        cmd = [NVCC, *NVCC_FLAGS, "-shared", "-o", SO + ".tmp",
               *[os.path.join(CSRC, f) for f in SOURCES], "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(LIB, "build.log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libgdraa.so (see %s)" % log)
        if verbose:
            sys.stdout.write(r.stderr)
        os.replace(SO + ".tmp", SO)
    jdeps = [os.path.join(CSRC, "jobserver.cpp"), os.path.join(CSRC, "jobserver_proto.h"), __file__]
    if force or _stale(JOBSERVER, jdeps):
        cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-o", JOBSERVER + ".tmp",
               os.path.join(CSRC, "jobserver.cpp"), "-lrt"]
        subprocess.run(cmd, check=True)
        os.replace(JOBSERVER + ".tmp", JOBSERVER)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
