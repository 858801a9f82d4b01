"""Start / locate the job-server control plane (lib/gdraa_jobserver).

One job server per job.  Under torchrun, local rank 0 starts it at a socket path derived
from MASTER_PORT; every rank exports GDRAA_JOBSERVER=<path> before gdraa_init, which
retries the connection until the server is up.
"""
import os
import subprocess

from .gdraa import PKG

BINARY = os.path.join(PKG, "lib", "gdraa_jobserver")


def default_socket_path(tag=None) -> str:
    if tag is None:
        tag = os.environ.get("MASTER_PORT", str(os.getpid()))
    return f"/tmp/gdraa_js_{os.getuid()}_{tag}.sock"


def start(world: int, socket_path: str = None, gated: bool = False, timeout_ms: int = 120000,
          stats_path: str = None) -> subprocess.Popen:
    """Spawn the job server; returns the Popen (its stdout carries the exit JSON line)."""
    if not os.path.exists(BINARY):
        raise FileNotFoundError(f"{BINARY} missing: run __graft_entry__.build()")
    socket_path = socket_path or default_socket_path()
    cmd = [BINARY, "--socket", socket_path, "--world", str(world),
           "--timeout-ms", str(timeout_ms)]
    if gated:
        cmd.append("--gated")
    if stats_path:
        cmd += ["--stats", stats_path]
    proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    proc.socket_path = socket_path
    return proc


def setup_for_rank(world: int, rank: int, local_rank: int = None, gated: bool = False,
                   tag=None):
    """Torchrun helper: local rank 0 starts the server; all ranks set GDRAA_JOBSERVER.
    Returns the Popen on the starting rank, else None."""
    if local_rank is None:
        local_rank = rank
    path = default_socket_path(tag)
    os.environ["GDRAA_JOBSERVER"] = path
    if world > 1 and local_rank == 0:
        return start(world, path, gated=gated)
    return None
