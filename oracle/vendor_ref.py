"""Vendor the reference package into oracle/_ref/ (TEST INFRASTRUCTURE ONLY).

The reference (rdmaflow) is pure Python with numpy as its only dependency, so
"building" it is copying its package: /root/reference/pkg/src/rdmaflow ->
oracle/_ref/rdmaflow, plus its test suite -> oracle/_ref/ref_tests (run
against this package by tests/test_gpu_ref_suite.py).  oracle/_ref/ is
git-ignored (no reference source enters the history) but travels with the
gpurun snapshot, so the GPU box can time the real reference as the CPU arm
(bench.py --impl reference, cpu_baseline kind "reference") and run its tests.
Run here (where /root/reference exists): python -m oracle.vendor_ref
"""
from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
OUT = os.path.join(HERE, "_ref")


def vendor(ref_pkg: str = REF_PKG, out: str = OUT) -> bool:
    src = os.path.join(ref_pkg, "src", "rdmaflow")
    if not os.path.isdir(src):
        return False
    os.makedirs(out, exist_ok=True)
    ignore = shutil.ignore_patterns("__pycache__", "*.pyc")
    for name, from_ in (("rdmaflow", src), ("ref_tests", os.path.join(ref_pkg, "tests"))):
        dst = os.path.join(out, name)
        if os.path.isdir(from_):
            shutil.rmtree(dst, ignore_errors=True)
            shutil.copytree(from_, dst, ignore=ignore)
    with open(os.path.join(out, "README"), "w") as fh:
        fh.write("Vendored copy of the reference (rdmaflow) made by oracle/vendor_ref.py.\n"
                 "Test infrastructure only: never imported by paper_1805_08430_b200.\n")
    return True


if __name__ == "__main__":
    ok = vendor()
    print(OUT if ok else "reference not found; nothing vendored")
    sys.exit(0 if ok else 1)
