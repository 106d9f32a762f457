"""Where the ~67 us of one small dynamic transfer through the host API go."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: F401
from paper_1805_08430_b200.analyzer import PlanEntry
from paper_1805_08430_b200.fabric import Fabric
from paper_1805_08430_b200.graph import Tensor, shape_of
from paper_1805_08430_b200.memspace import ArenaAllocator, BufferRef, MemorySpace
from paper_1805_08430_b200.runtime.protocol import DynReceiver, DynSender
from paper_1805_08430_b200.wire import ElemType, Mechanism, meta_block_size

size = 4096
fab = Fabric()
sp = {s: MemorySpace(s, 16 << 20, device=0) for s in (0, 1)}
ar = {s: ArenaAllocator(sp[s], sp[s].allocate_region(8 << 20, True)) for s in (0, 1)}
dv = {s: fab.create_device(sp[s], qps_per_peer=2) for s in (0, 1)}
fwd = dv[0].connect(dv[1].endpoint)
back = dv[1].channels_to(dv[0].endpoint)
e = PlanEntry(0, 0, 1, Mechanism.DYNAMIC, shape_of(size // 4), ElemType.F32, 1)
mb = ar[1].alloc(meta_block_size(1))
sp[1].write_at(mb, mb.length - 1, b"\x00")
e.recv_buffer = mb
e.remote_addr, e.remote_token, e.remote_len = mb.base_addr, mb.access_token, mb.length
snd = DynSender(e, sp[0], ar[0], fwd[1])
rcv = DynReceiver(e, sp[1], ar[1], back[1])
t = Tensor((size // 4,), ElemType.F32, BufferRef(ar[0].alloc(size), ar[0]), 0)
acc = {"send": 0.0, "poll": 0.0, "fetch": 0.0, "release": 0.0, "polls": 0}
R = 300
for k in range(R + 20):
    a = time.perf_counter()
    snd.send(t, stage_copy=False)
    b = time.perf_counter()
    m, n = None, 0
    while m is None:
        m = rcv.poll()
        n += 1
    c = time.perf_counter()
    got = rcv.fetch(m)
    d = time.perf_counter()
    got.buffer.release()
    f = time.perf_counter()
    if k >= 20:
        acc["send"] += (b - a) / R * 1e6
        acc["poll"] += (c - b) / R * 1e6
        acc["fetch"] += (d - c) / R * 1e6
        acc["release"] += (f - d) / R * 1e6
        acc["polls"] += n / R
print(json.dumps({k: round(v, 2) for k, v in acc.items()}), flush=True)
