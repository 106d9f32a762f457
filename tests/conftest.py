"""Test configuration: repo root on sys.path, the `gpu` marker, golden fixtures."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 (runs the sm_100a kernels through libsrflow.so)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        doc = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return doc, arrays
