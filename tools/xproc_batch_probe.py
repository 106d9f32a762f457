"""Cross-process: K1 put vs the PS put batch (k_put_batch) moving the same
256 MiB into the next rank's pool (SM stores, copy engine off)."""
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
_lib.tune("peer_ce_kib", 0)
S = 256 << 20
ring = bench.SendRecvRing(S, rank, world, local)
P, u64 = C.c_void_p, _lib.u64_array
b = C.c_void_p()
_lib.call("srf_batch_put_create", 1, (P * 1)(ring.src.handle.value), u64([ring.payload.base_addr]),
          u64([S]), u64([ring.payload.access_token]), u64([ring.flag.base_addr]),
          (P * 1)(ring.dst.handle.value), u64([ring.dst_region[0]]), u64([ring.dst_region[1]]), 0,
          C.byref(b))
R = 20


def timed(fn):
    fn()
    ring.sync()
    bench.barrier_sync()
    t0 = time.perf_counter()
    if rank == 0:
        for _ in range(R):
            fn()
        ring.sync()
    bench.barrier_sync()
    return round(S * R / (time.perf_counter() - t0) / 1e9, 1)


def k1():
    _lib.call("srf_put", ring.src.handle, ring.args_addr, ring.args_len, ring.args_tok, 2,
              ring.dst.handle, ring.dst_region[0], ring.dst_region[1], 0, ring.stream, None)


def batch(cap=0):
    _lib.call("srf_batch_launch", b, ring.stream, 0, 0, cap)


res = {"k1": timed(k1), "batch": timed(batch), "batch_cap296": timed(lambda: batch(296)),
       "batch_cap148": timed(lambda: batch(148)), "batch_cap592": timed(lambda: batch(592))}
for ctas, thr in ((2, 256), (4, 512), (8, 512)):
    _lib.tune("ctas_per_sm", ctas)
    _lib.tune("copy_threads", thr)
    res[f"k1_{ctas}x{thr}"] = timed(k1)
if rank == 0:
    print(json.dumps(res), flush=True)
