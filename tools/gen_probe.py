"""Device GenGrad (srf_gen_reference, the reference PCG64 stream) throughput
vs the HBM write rate of a plain fill, at VGG-16 (138.4 M fp32) and FCN-5
slab sizes; a window of each result is checked against numpy."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import port
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

out = []
for n in (138_357_544, 5_111_750, 641_607):
    sp = MemorySpace(0, 4 * n + (8 << 20), device=0)
    reg = sp.allocate_region(4 * n + 64, register=True)
    st = C.c_void_p()
    _lib.call("srf_stream_create", sp.handle, C.byref(st))
    ev = [C.c_void_p(), C.c_void_p()]
    for e in ev:
        _lib.call("srf_timing_event_create", sp.handle, C.byref(e))

    def timed(fn, R):
        fn()
        _lib.call("srf_stream_sync", st)
        _lib.call("srf_event_record_on", ev[0], st)
        for _ in range(R):
            fn()
        _lib.call("srf_event_record_on", ev[1], st)
        _lib.call("srf_stream_sync", st)
        ms = C.c_float()
        _lib.call("srf_event_elapsed_ms", ev[0], ev[1], C.byref(ms))
        return ms.value / R * 1e3

    R = 20 if n > 10**7 else 200
    it = [0]

    def gen():
        it[0] += 1
        _lib.call("srf_gen_reference", sp.handle, reg.base_addr, n, 0, 0, 29, it[0], st, None)

    us = timed(gen, R)
    got = np.frombuffer(sp.read_raw(reg.base_addr + 4 * (n - 4096), 4 * 4096), np.float32)
    ok = got.tobytes() == port.reference_values(0, 29, it[0], n - 4096, 4096).tobytes()
    # a plain HBM fill of the same bytes (zero-copy K5 of the first half onto
    # the second is a read+write; use the pool zero-fill via a local copy)
    usc = timed(lambda: _lib.call("srf_copy", sp.handle, reg.base_addr, reg.base_addr + 4 * (n // 2),
                                  4 * (n // 2), st, None), R)
    row = {"n": n, "bytes": 4 * n, "gen_us": round(us, 2), "gen_gbps": round(4 * n / us / 1e3, 1),
           "copy_half_us": round(usc, 2),
           "copy_half_gbps_rw": round(2 * 4 * (n // 2) / usc / 1e3, 1), "verified": ok}
    print(json.dumps(row), flush=True)
    out.append(row)
    _lib.call("srf_stream_destroy", st)
    sp.close()
