"""bench.sweep (configs[1] on one GPU) alone, one JSON row per size."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1805_08430_b200 import _lib  # noqa: E402

_lib.load()
for r in bench.sweep(int(os.environ.get("PROBE_MAX", str(256 << 20))), 0):
    print(json.dumps(r), flush=True)
