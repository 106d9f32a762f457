"""Cross-process copy-engine put vs activity of the destination process: rank 0
pushes 256 MiB into rank 1's pool (copy engine or SM stores) while rank 1 is
idle, runs a long compute kernel, or runs a kernel spinning on a flag."""
import ctypes as C
import json
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
S = 256 << 20
ring = bench.SendRecvRing(S, rank, world, local)
R = 10
res = {}


def put():
    _lib.call("srf_put", ring.src.handle, ring.args_addr, ring.args_len, ring.args_tok, 2,
              ring.dst.handle, ring.dst_region[0], ring.dst_region[1], 0, ring.stream, None)


def busy_compute():
    a = torch.randn(8192, 8192, device="cuda")
    for _ in range(60):
        a = a @ a
        a = a / a.norm()
    return a


for engine in ("ce", "sm"):
    _lib.tune("peer_ce_kib", 1024 if engine == "ce" else 0)
    for mode in ("idle", "compute", "spin"):
        bench.barrier_sync()
        if rank == 1:
            if mode == "compute":
                busy_compute()
            elif mode == "spin":
                # a flag nobody sets: 1 warp spinning for ~1.5 s (times out)
                _lib.call("srf_flag_wait", ring.rcv.handle, ring.recv.base_addr + 64, 7, 0,
                          1_500_000_000, ring.stream)
        time.sleep(0.05)
        if rank == 0:
            put()
            ring.sync()
            t0 = time.perf_counter()
            for _ in range(R):
                put()
            ring.sync()
            res[f"{engine}_{mode}"] = round(S * R / (time.perf_counter() - t0) / 1e9, 1)
        torch.cuda.synchronize()
        try:
            ring.sync()
        except Exception:
            pass
        bench.barrier_sync()
if rank == 0:
    print(json.dumps(res), flush=True)
