"""configs[1] one direction (rank 0 -> rank 1): push vs pull edge per size,
through bench.sweep_nvlink_one_way.  torchrun --nproc-per-node 2."""
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
mx = int(os.environ.get("PROBE_MAX", str(256 << 20)))
rows = bench.sweep_nvlink_one_way(mx, rank, world, local)
if rank == 0:
    for r in rows:
        print(json.dumps(r), flush=True)
