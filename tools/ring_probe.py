"""Multi-process ring probe (torchrun): isolates the cost of the static
protocol (credit wait + consumer flag wait) from raw IPC peer stores."""
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
if os.environ.get("PROBE_PEER_FIRST"):
    _lib.call("srf_enable_peer", local, (local + 1) % world)
    _lib.call("srf_enable_peer", local, (local - 1) % world)
S = int(os.environ.get("PROBE_BYTES", 256 << 20))
ring = bench.SendRecvRing(S, rank, world, local)
R = 30
res = {}


def timed(body):
    a, b = ring.event(), ring.event()
    for _ in range(3):
        body()
    ring.sync()
    bench.barrier_sync()
    ring.record(a)
    for _ in range(R):
        body()
    ring.record(b)
    ring.sync()
    bench.barrier_sync()
    return bench.dist_max(ring.elapsed_ms(a, b) / R)


def put_nowait():
    _lib.call("srf_put", ring.src.handle, ring.args_addr, ring.args_len, ring.args_tok, 2,
              ring.dst.handle, ring.dst_region[0], ring.dst_region[1], 0, ring.stream, None)


def clear_own():
    # consume without waiting (the flag is set by the peer's completed put)
    _lib.call("srf_flag_wait", ring.rcv.handle, ring.recv.base_addr + S, 1, 1, 10**10, ring.stream)


res["put_only_ms"] = timed(put_nowait)
# pull: each rank reads the next rank's payload (mapped as ring.dst) into its own recv
def pull_next():
    _lib.call("srf_get", ring.src.handle, ring.recv.base_addr, ring.recv.access_token,
              ring.dst.handle, ring.payload.base_addr, ring.dst_region[1], S, ring.stream, None)
res["gbps_pull_only"] = S / (timed(pull_next) / 1e3) / 1e9
# reset flags
ring.sync(); bench.barrier_sync()
ring.rcv.write_at(ring.recv, S, b"\x00"); bench.barrier_sync()
res["protocol_ms"] = timed(lambda: (ring.put(), ring.consume()))
res["gbps_put_only"] = S / (res["put_only_ms"] / 1e3) / 1e9
res["gbps_protocol"] = S / (res["protocol_ms"] / 1e3) / 1e9
for impl in (1,):
    _lib.tune("put_impl", impl)
    res[f"protocol_ms_impl{impl}"] = timed(lambda: (ring.put(), ring.consume()))
    res[f"gbps_protocol_impl{impl}"] = S / (res[f"protocol_ms_impl{impl}"] / 1e3) / 1e9
    _lib.tune("put_impl", 0)
if rank == 0:
    print(json.dumps(res), flush=True)

# --- comparators: copy engine into the IPC mapping, NCCL send/recv --------------
import time
import torch.distributed as dist
from paper_1805_08430_b200.memspace import device_view
remote = device_view(ring.dst.device_base + ring.dst_region[0], S, local)
local_src = ring.src.view(ring.payload, 0, S)
for _ in range(3):
    remote.copy_(local_src)
torch.cuda.synchronize(); bench.barrier_sync()
t0 = time.perf_counter()
for _ in range(R):
    remote.copy_(local_src)
torch.cuda.synchronize(); bench.barrier_sync()
res["copy_engine_ipc_gbps"] = S * R / bench.dist_max(time.perf_counter() - t0) / 1e9
x = torch.empty(S, dtype=torch.uint8, device="cuda")
y = torch.empty(S, dtype=torch.uint8, device="cuda")
peer = (rank + 1) % world
prev = (rank - 1) % world
def xchg():
    reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, x, peer), dist.P2POp(dist.irecv, y, prev)])
    for r in reqs:
        r.wait()
for _ in range(3):
    xchg()
torch.cuda.synchronize(); bench.barrier_sync()
t0 = time.perf_counter()
for _ in range(R):
    xchg()
torch.cuda.synchronize(); bench.barrier_sync()
res["nccl_sendrecv_gbps"] = S * R / bench.dist_max(time.perf_counter() - t0) / 1e9
if rank == 0:
    print(json.dumps(res), flush=True)
