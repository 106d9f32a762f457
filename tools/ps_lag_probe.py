"""VGG-16 reference placement (co-located) with the fused push, exchange lag
and order sweep (SRFLOW_PS_EXCHANGE_LAG / _ORDER read per PsStep)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_1805_08430_b200 import _lib  # noqa: E402
from paper_1805_08430_b200.distributed import env_world, init_process_group  # noqa: E402

rank, world, local = env_world()
_lib.load()
torch.cuda.set_device(local)
init_process_group("nccl")
for order in ("size", "index"):
    for lag in (0, 1, 2, 3, 5, 8):
        os.environ["SRFLOW_PS_EXCHANGE_LAG"] = str(lag)
        os.environ["SRFLOW_PS_EXCHANGE_ORDER"] = order
        r = bench.bench_ps(rank, world, local, 20, 3, op="sgd", cpu=False)
        if rank == 0:
            print(json.dumps({"order": order, "lag": lag, "steps_per_s": r["steps_per_s"],
                              "verified": r["verified"],
                              "best": min(r["autotune_ms_per_5"], key=r["autotune_ms_per_5"].get),
                              "autotune": r["autotune_ms_per_5"]}), flush=True)
