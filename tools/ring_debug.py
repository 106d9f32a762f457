"""N>1 pipelined ring, step by step with progress prints (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.distributed import init_process_group

rank, world, local = init_process_group("nccl")
torch.cuda.set_device(local)
_lib.tune("put_timeout_ms", 3000)
mirror = os.environ.get("RING_MIRROR", "1") == "1"


def say(*a):
    print(f"[rank {rank} {time.time():.3f}]", *a, flush=True)


for S in (1 << 20, 4 << 20):
    say("ring", S)
    ring = bench.PipelinedRing(S, rank, world, local, slots=4)
    if not mirror:
        ring.credit_for_consumer = None
    say("created", ring.info)
    ring.launch(8)
    say("launched")
    try:
        ring.sync()
        say("synced")
    except Exception as exc:
        say("sync error", exc)
    buf = (bench.C.c_uint32 * 14)()
    _lib.call("srf_edge_state", ring.edge._h, buf, 14)
    say("state", list(buf))
    bench.barrier_sync()
    say("verify", ring.verify())
    ring.close()
say("done")
