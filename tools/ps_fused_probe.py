"""PS device engine with the fused weight push in the autotune: the N=1
configs (VGG-16, FCN-5, LSTM, MLP) through bench.bench_ps, printing the
chosen schedule and every candidate's time for 5 steps.  torchrun for N>1."""
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
rows = {"vgg16": bench.bench_ps(rank, world, local, 20, 3, op="sgd", cpu=False)}
rows.update(bench.bench_ps_configs(rank, world, local, 20, 3, "sgd", False))
if rank == 0:
    for k, r in rows.items():
        if isinstance(r, dict) and "steps_per_s" in r:
            print(json.dumps({"cfg": k, "world": world, "steps_per_s": r["steps_per_s"],
                              "fused_push": r.get("fused_push"), "frac": r["roofline"]["frac"],
                              "verified": r["verified"], "autotune": r["autotune_ms_per_5"]}),
                  flush=True)
