"""One process per GPU (torchrun, IPC-mapped pools): the PS step in every
schedule and the Send/Recv endpoints, each rank's results vs the oracle.

With two GPUs the ranks use NCCL for the control plane and NVLink for the
data plane.  On a one-GPU box both ranks run on GPU 0 with a gloo control
plane (SRFLOW_MP_ONE_GPU=1): CUDA IPC between two processes of one device
still exercises pool export/import, proxy spaces, system-scope flags on
imported pools and the doorbell's device-read fallback."""
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


def _run(worker: str, pools: str) -> str:
    one_gpu = _lib.device_count() < 2
    env = dict(os.environ, NCCL_DEBUG="WARN", SRFLOW_ALLOC_VMM="1" if pools == "vmm" else "0",
               SRFLOW_MP_ONE_GPU="1" if one_gpu else "0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", worker)]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert out.count(": OK") == 2, out[-4000:]
    return out


@pytest.mark.parametrize("pools", ["ipc", "vmm"])
def test_two_process_ps_schedules_match_oracle(pools):
    """Pools exported as CUDA IPC handles, or as VMM allocations whose POSIX
    fd the peer duplicates (pidfd_getfd)."""
    _run("mp_ps_worker.py", pools)


@pytest.mark.parametrize("pools", ["ipc", "vmm"])
def test_two_process_sendrecv_endpoints(pools):
    """Static and dynamic Send/Recv between processes through the reference
    endpoints (StaticSender/Receiver, DynSender/Receiver)."""
    _run("mp_sendrecv_worker.py", pools)


@pytest.mark.parametrize("pools", ["ipc", "vmm"])
def test_two_process_pipelined_and_pulled_edges(pools):
    """One edge between processes (configs[1]'s one-way layout): the push
    edge storing into the peer's mapped slots and the pull edge reading the
    peer's mapped payloads; every round's consumer checksum equals the
    sender's payload."""
    _run("mp_edge_worker.py", pools)
