"""Copy-engine peer copy rate vs buffer alignment (GPU0 -> GPU1, one
process): K1 with knob 6 on, source/destination offsets from 2-MiB-aligned
pool bases."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

S = 256 << 20
a = MemorySpace(0, S + (16 << 20), device=0)
b = MemorySpace(1, S + (16 << 20), device=1)
_lib.call("srf_connect", a.handle, b.handle)
ra = a.allocate_region(S + (12 << 20), register=True)
rb = b.allocate_region(S + (12 << 20), register=True)
u = _lib.u64_array
st = C.c_void_p()
_lib.call("srf_stream_create", a.handle, C.byref(st))
print("pool bases", hex(a.device_base), hex(b.device_base), "regions", ra.base_addr, rb.base_addr)


def rate(so, do, n, ce, R=10):
    _lib.tune("peer_ce_kib", 1024 if ce else 0)
    flag = ra.base_addr + so + n
    a.write_raw(flag, b"\x01")
    def go():
        _lib.call("srf_put", a.handle, u([ra.base_addr + so, flag]), u([n - 1, 1]),
                  u([ra.access_token] * 2), 2, b.handle, rb.base_addr + do, rb.access_token, 0,
                  st, None)
    go(); _lib.call("srf_stream_sync", st)
    t0 = time.perf_counter()
    for _ in range(R):
        go()
    _lib.call("srf_stream_sync", st)
    return round(n * R / (time.perf_counter() - t0) / 1e9, 1)


out = []
for off in (0, 32, 256, 4096, 65536, 1 << 20, 2 << 20):
    for n in (S, 64 << 20):
        out.append({"src_off": off, "dst_off": off, "bytes": n, "ce": rate(off, off, n, True),
                    "sm": rate(off, off, n, False)})
        print(json.dumps(out[-1]), flush=True)
for so, do in ((0, 256), (256, 0), (4096, 0), (0, 4096)):
    print(json.dumps({"src_off": so, "dst_off": do, "bytes": S, "ce": rate(so, do, S, True),
                      "sm": rate(so, do, S, False)}), flush=True)
