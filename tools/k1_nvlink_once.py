"""A few K1 puts (SM stores) GPU0 -> GPU1 and K4 pulls GPU1 -> GPU0 (one
process, peer access) for ncu."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

_lib.tune("peer_ce_kib", 0)   # the SM kernels, not the copy engine

S = 256 << 20
a = MemorySpace(0, S + (16 << 20), device=0)
b = MemorySpace(1, S + (16 << 20), device=1 if _lib.device_count() > 1 else 0)
_lib.call("srf_connect", a.handle, b.handle)
ra, rb = a.allocate_region(S + (8 << 20), True), b.allocate_region(S + (8 << 20), True)
flag = ra.base_addr + S + 64
a.write_raw(flag, b"\x01")
for _ in range(6):
    _lib.call("srf_put", a.handle, _lib.u64_array([ra.base_addr, flag]), _lib.u64_array([S, 1]),
              _lib.u64_array([ra.access_token] * 2), 2, b.handle, rb.base_addr, rb.access_token,
              0, None, None)
a.sync()
for _ in range(6):  # K4: GPU0 reads GPU1's block
    _lib.call("srf_get", a.handle, ra.base_addr, ra.access_token, b.handle, rb.base_addr,
              rb.access_token, S, None, None)
a.sync()
print("ok")
