"""Torch tensors allocated inside a registered pool and
sent zero-copy; run in a subprocess because torch's allocator can only be
replaced before the first CUDA allocation."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_torch_allocations_live_in_the_registered_pool():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "torch_pool_worker.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "torch-pool OK" in out, out[-4000:]
