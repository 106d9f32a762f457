"""A few K1 puts GPU0 -> GPU1 (one process, peer access) for ncu."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

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
print("ok")
