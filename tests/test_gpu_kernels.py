"""Both data-movement variants of the fused kernel -- the LSU (register-staged) and the
TMA (shared-memory-staged, cp.async.bulk) kernel -- must produce the oracle's bits for
every mode, world size and dtype.  The runtime picks one per call by a measured rule;
here each is forced in a subprocess (GDRAA_KERNEL is read once per process)."""
import os
import subprocess
import sys

import pytest

from tests.conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs a CUDA GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kernel", ["lsu", "tma", "tma-thread-fence", "lsu-thread-fence"])
def test_forced_kernel_parity(kernel):
    """Each data-movement variant, with the default per-CTA exit fence and with the
    per-thread one (GDRAA_EXIT_FENCE=thread), gives the oracle's bits."""
    env = dict(os.environ, GDRAA_KERNEL=kernel.split("-")[0], GDRAA_LL_MAX_BYTES="0")
    if kernel.endswith("thread-fence"):
        env["GDRAA_EXIT_FENCE"] = "thread"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_kernel_parity_worker.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"OK {kernel.split('-')[0]}" in r.stdout

