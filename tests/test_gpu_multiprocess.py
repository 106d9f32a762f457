"""One process per GPU (torchrun, NCCL control plane, IPC-mapped pools): the
PS step in every schedule vs the oracle on each rank's variables."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest

from paper_1805_08430_b200 import _lib

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.skipif(_lib.device_count() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("pools", ["ipc", "vmm"])
def test_two_process_ps_schedules_match_oracle(pools):
    """Pools exported as CUDA IPC handles, or as VMM allocations whose POSIX
    fd the peer duplicates (pidfd_getfd)."""
    env = dict(os.environ, NCCL_DEBUG="WARN", SRFLOW_ALLOC_VMM="1" if pools == "vmm" else "0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_ps_worker.py")]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert out.count(": OK") == 2, out[-4000:]
