"""Cross-process NVLink store probe: unidirectional vs bidirectional SM puts
through the imported peer pool, grid-geometry sweep."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.distributed import init_process_group

rank, world, local = init_process_group("nccl")
torch.cuda.set_device(local)
if os.environ.get("PEER_CTX"):
    for d in range(torch.cuda.device_count()):
        torch.empty(1, device=f"cuda:{d}")  # primary context on every GPU
    torch.cuda.set_device(local)
    for d in range(torch.cuda.device_count()):
        _lib.call("srf_enable_peer", local, d)
S = 256 << 20
ring = bench.SendRecvRing(S, rank, world, local)
R = 20
res = {}


def timed(body, active=True):
    a, b = ring.event(), ring.event()
    bench.barrier_sync()
    ring.record(a)
    if active:
        for _ in range(R):
            body()
    ring.record(b)
    ring.sync()
    bench.barrier_sync()
    return ring.elapsed_ms(a, b) / R


def put():
    _lib.call("srf_put", ring.src.handle, ring.args_addr, ring.args_len, ring.args_tok, 2,
              ring.dst.handle, ring.dst_region[0], ring.dst_region[1], 0, ring.stream, None)


for ctas, threads, vec32 in ((8, 512, 0), (8, 512, 1), (2, 512, 1), (4, 256, 1)):
    _lib.tune("ctas_per_sm", ctas)
    _lib.tune("copy_threads", threads)
    _lib.tune("vec32", vec32)
    t_uni = timed(put, active=(rank == 0))
    t_bi = bench.dist_max(timed(put))
    if rank == 0:
        rec = {"ctas": ctas, "threads": threads, "vec32": vec32, "uni_gbps": S / t_uni / 1e6,
               "bi_gbps": S / t_bi / 1e6}
        print(json.dumps(rec), flush=True)
