"""bench.bench_ps_session alone (configs[2]-[4] through Session.run)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1805_08430_b200 import _lib  # noqa: E402

_lib.load()
out = bench.bench_ps_session(0, 1, 0, 20, 3, "sgd", False)
for k, v in out.items():
    print(json.dumps({"cfg": k, "steps_per_s": v.get("steps_per_s"), "e2e": v.get("e2e", {}).get("value"),
                      "verified": v.get("verified"), "replay": v.get("replay")}), flush=True)
