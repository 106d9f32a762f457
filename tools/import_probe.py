"""Single process, two GPUs: SM puts GPU0 -> GPU1 through (a) the owning
mapping and (b) a VMM re-import of the same allocation (fd), to separate
'imported mapping' from 'other process' effects."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

_lib.load()
_lib.tune("alloc_vmm", 1)
S = 256 << 20
a = MemorySpace(0, S + (64 << 20), device=0)
b = MemorySpace(1, S + (64 << 20), device=1)
_lib.call("srf_connect", a.handle, b.handle)
ra = a.allocate_region(S + (32 << 20), True)
rb = b.allocate_region(S + (32 << 20), True)
flag = ra.base_addr + S + 64
a.write_raw(flag, b"\x01")
desc = b.export()
proxy = MemorySpace.import_remote(desc, 0)
st = C.c_void_p()
_lib.call("srf_stream_create", a.handle, C.byref(st))
e0, e1 = C.c_void_p(), C.c_void_p()
_lib.call("srf_timing_event_create", a.handle, C.byref(e0))
_lib.call("srf_timing_event_create", a.handle, C.byref(e1))


def rate(dst):
    def put():
        _lib.call("srf_put", a.handle, _lib.u64_array([ra.base_addr, flag]), _lib.u64_array([S, 1]),
                  _lib.u64_array([ra.access_token] * 2), 2, dst.handle, rb.base_addr,
                  rb.access_token, 0, st, None)
    for _ in range(3):
        put()
    _lib.call("srf_stream_sync", st)
    _lib.call("srf_event_record_on", e0, st)
    for _ in range(20):
        put()
    _lib.call("srf_event_record_on", e1, st)
    _lib.call("srf_stream_sync", st)
    ms = C.c_float()
    _lib.call("srf_event_elapsed_ms", e0, e1, C.byref(ms))
    return S * 20 / (ms.value / 1e3) / 1e9


print(json.dumps({"owning_mapping_gbps": rate(b), "vmm_reimport_gbps": rate(proxy)}), flush=True)
