"""One k_dyn_pull_stream launch for an ncu capture: GPU 0's payloads
announced by k_dyn_send_stream (rounds <= slots, so no credit waits), GPU 1
pulls them through the pipelined dynamic edge (ring arena of `slots` rounds,
consumer afterwards in stream order).  Usage: python tools/dyn_ncu_once.py [S] [slots]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib  # noqa: E402
from paper_1805_08430_b200.memspace import MemorySpace  # noqa: E402
from paper_1805_08430_b200.runtime.protocol import PipelinedDynamicEdge  # noqa: E402
from paper_1805_08430_b200.wire import ElemType  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256 << 20
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 4
stride = (S + 255) & ~255
ms = PipelinedDynamicEdge.meta_stride(1)
dev_b = 1 if _lib.device_count() > 1 else 0
a = MemorySpace(0, 2 * stride + (8 << 20), device=0)
b = MemorySpace(1, slots * stride + slots * ms + (8 << 20), device=dev_b)
_lib.call("srf_connect", a.handle, b.handle)
src = a.allocate_region(2 * stride, register=True)
for i in range(2):
    _lib.call("srf_gen_reference", a.handle, src.base_addr + i * stride, S // 4, 0, 0, 0, 2 + i,
              None, None)
ring = b.allocate_region(slots * stride, register=True)
meta = b.allocate_region(slots * ms, register=True)
a.sync(), b.sync()
e = PipelinedDynamicEdge(a, src.base_addr, src.base_addr + 2 * stride, src.access_token, S, 1, b,
                         meta.base_addr, ms, slots, ring.base_addr, slots * stride)
for k in range(2):   # ncu -s 1 -c 1 captures the second receiver launch
    PipelinedDynamicEdge.send(a, b, meta.base_addr, ms, slots, (S // 4,), ElemType.F32,
                              src.base_addr, stride, 2, src.access_token, k * slots, slots)
    a.sync()
    e.recv(slots)
    b.sync()
    e.consume(k * slots, slots)
    b.sync()
print("dyn_ncu_once ok", flush=True)
e.close()
