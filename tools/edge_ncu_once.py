"""One k_put_stream launch for an ncu capture: `slots` rounds (no credit
waits, so it runs alone under a serialising profiler), then its consumer.
Usage: python tools/edge_ncu_once.py [hbm|nvl|pull] [S] [slots]
  hbm: server 0 -> server 1 on GPU 0; nvl: GPU 0 -> GPU 1 (one process);
  pull: the pull edge, k_pull_stream on GPU 1 reading GPU 0's payloads
  (rounds posted up front, consumer after it in stream order)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace
from paper_1805_08430_b200.runtime.protocol import PipelinedStaticEdge, PulledStaticEdge

mode = sys.argv[1] if len(sys.argv) > 1 else "hbm"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 256 << 20
slots = int(sys.argv[3]) if len(sys.argv) > 3 else 4
st, sl = (S + 255) & ~255, (S + 1 + 255) & ~255
a = MemorySpace(0, 2 * st + (8 << 20), device=0)
b = MemorySpace(1, slots * sl + (8 << 20), device=1 if mode in ("nvl", "pull") else 0)
_lib.call("srf_connect", a.handle, b.handle)
ra = a.allocate_region(2 * st, register=True)
rb = b.allocate_region(slots * sl, register=True)
for i in range(2):
    _lib.call("srf_gen_reference", a.handle, ra.base_addr + i * st, S // 4, 0, 0, 0, 2 + i,
              None, None)
for i in range(slots):
    b.write_raw(rb.base_addr + i * sl + S, b"\x00")
a.sync(), b.sync()
if mode == "pull":
    posted = b.allocate_region(8)
    e = PulledStaticEdge(a, ra.base_addr, ra.access_token, S, 2, st, b, rb, slots, sl,
                         posted.base_addr, tma=os.environ.get("PROBE_TMA", "1") == "1")
    for k in range(2):
        PulledStaticEdge.post(a, b, posted.base_addr, (k + 1) * slots)
        a.sync()
        e.recv(slots)
        PipelinedStaticEdge.consume(b, rb.base_addr, slots, sl, S, k * slots, slots)
        b.sync()
    print("edge_ncu_once ok", e.info(), flush=True)
    e.close()
    sys.exit(0)
e = PipelinedStaticEdge(a, ra, S, 2, st, b, rb.base_addr, rb.access_token, slots, sl)
for _ in range(2):   # the first pass warms; ncu -s 1 -c 1 captures the second
    e.send(slots)
    PipelinedStaticEdge.consume(b, rb.base_addr, slots, sl, S, e.info()["next_round"] - slots,
                                slots)
    a.sync(), b.sync()
print("edge_ncu_once ok", e.info(), flush=True)
e.close()
