"""Same-GPU pipelined edge: sender and consumer on GPU 0; on a timeout print
the edge state and slot flags."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib, errors
from paper_1805_08430_b200.memspace import MemorySpace
from paper_1805_08430_b200.runtime.protocol import PipelinedStaticEdge

_lib.tune("put_timeout_ms", 300)
cases = []
for thr in (32, 64, 128, 1024):
    for S, slots, mode, rounds in [(1024, 1, 0, 10), (1024, 1, 0, 200), (1024, 1, 1, 200),
                                   (1024, 2, 0, 200), (1 << 20, 1, 0, 50), (1 << 20, 4, 0, 50)]:
        cases.append((thr, S, slots, mode, rounds))
for thr, S, slots, mode, rounds in cases:
    _lib.tune("consume_threads", thr)
    st, sl = (S + 255) & ~255, (S + 1 + 255) & ~255
    a = MemorySpace(10, 8 * st + (4 << 20), seed=1, device=0)
    b = MemorySpace(20, slots * sl + 4096 + (4 << 20), seed=2, device=0)
    ra = a.allocate_region(8 * st, register=True)
    rb = b.allocate_region(slots * sl, register=True)
    sums = b.allocate_region(8 * rounds)
    for i in range(slots):
        b.write_raw(rb.base_addr + i * sl + S, b"\x00")
    a.sync(), b.sync()
    sa, sb = C.c_void_p(), C.c_void_p()
    _lib.call("srf_stream_create", a.handle, C.byref(sa))
    _lib.call("srf_stream_create", b.handle, C.byref(sb))
    e = PipelinedStaticEdge(a, ra, S, 8, st, b, rb.base_addr, rb.access_token, slots, sl)
    PipelinedStaticEdge.consume(b, rb.base_addr, slots, sl, S, 0, rounds,
                                checksums_addr=sums.base_addr if mode else None, stream=sb)
    e.send(rounds, sa)
    res = "ok"
    for s in (sa, sb):
        _lib.call("srf_stream_sync", s)
    for sp in (a, b):
        try:
            sp.sync()
        except errors.Timeout as exc:
            res = f"timeout {exc}"
    buf = (C.c_uint32 * (3 * slots + 2))()
    _lib.call("srf_edge_state", e._h, buf, 3 * slots + 2)
    flags = [b.read_raw(rb.base_addr + i * sl + S, 1)[0] for i in range(slots)]
    print("thr", thr, S, slots, mode, rounds, res, "state", list(buf), "flags", flags, e.info(), flush=True)
    e.close()
    a.close(), b.close()
