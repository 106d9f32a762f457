"""N=1 VGG-16 (16 MiB slices and unsliced) with the fused push: GenGrad unit
size x exchange lag sweep (SRFLOW_GEN_UNIT_KIB / SRFLOW_PS_EXCHANGE_LAG)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1805_08430_b200 import _lib  # noqa: E402
from paper_1805_08430_b200.ps import PsLayout  # noqa: E402
from paper_1805_08430_b200.workloads import vgg16_shapes  # noqa: E402

_lib.load()
for sl in (16, 0):
    for unit in (64, 128, 512):
        for lag in (1, 3, 6):
            _lib.tune("gen_unit_kib", unit)
            os.environ["SRFLOW_PS_EXCHANGE_LAG"] = str(lag)
            L = PsLayout(vgg16_shapes(), 1, 1, slice_bytes=(sl << 20) if sl else None)
            r = bench.bench_ps(0, 1, 0, 20, 3, op="sgd", cpu=False, layout=L, label="probe")
            print(json.dumps({"slice": sl, "gen_unit_kib": unit, "lag": lag,
                              "steps_per_s": r["steps_per_s"], "verified": r["verified"],
                              "best": min(r["autotune_ms_per_5"], key=r["autotune_ms_per_5"].get)}),
                  flush=True)
