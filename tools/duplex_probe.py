"""NVLink duplex probe (one process, GPU0 <-> GPU1): does GPU0 push (stores
out) and pull (loads in) at the same time at full rate?  SM and copy-engine
variants of each direction."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

S = 256 << 20
a = MemorySpace(0, 3 * S + (8 << 20), device=0)
b = MemorySpace(1, 3 * S + (8 << 20), device=1)
_lib.call("srf_connect", a.handle, b.handle)
ra = a.allocate_region(3 * S + (4 << 20), register=True)
rb = b.allocate_region(3 * S + (4 << 20), register=True)
sa = [C.c_void_p(), C.c_void_p()]
for st in sa:
    _lib.call("srf_stream_create", a.handle, C.byref(st))
u = _lib.u64_array
a.write_raw(ra.base_addr + S, b"\x01")


def push(st):
    _lib.call("srf_put", a.handle, u([ra.base_addr, ra.base_addr + S]), u([S - 1, 1]),
              u([ra.access_token] * 2), 2, b.handle, rb.base_addr, rb.access_token, 0, st, None)


def pull(st):
    _lib.call("srf_get", a.handle, ra.base_addr + 2 * S, ra.access_token, b.handle,
              rb.base_addr + 2 * S, rb.access_token, S, st, None)


def timed(fns, R=20):
    for f, st in fns:
        f(st)
    for st in sa:
        _lib.call("srf_stream_sync", st)
    t0 = time.perf_counter()
    for _ in range(R):
        for f, st in fns:
            f(st)
    for st in sa:
        _lib.call("srf_stream_sync", st)
    dt = (time.perf_counter() - t0) / R
    return round(len(fns) * S / dt / 1e9, 1)


res = {}
for name, ce in (("sm", 0), ("ce", 1)):
    _lib.tune("peer_ce_kib", 1024 if ce else 0)
    res[f"push_{name}"] = timed([(push, sa[0])])
    res[f"pull_{name}"] = timed([(pull, sa[0])])
    res[f"push+pull_{name}"] = timed([(push, sa[0]), (pull, sa[1])])
# mixed: CE push with SM pull (get below threshold is SM... use threshold above S for pulls)
_lib.tune("peer_ce_kib", 1024)
def pull_sm(st):
    _lib.tune("peer_ce_kib", 0)
    pull(st)
    _lib.tune("peer_ce_kib", 1024)
res["push_ce+pull_sm"] = timed([(push, sa[0]), (pull_sm, sa[1])])
def push_sm(st):
    _lib.tune("peer_ce_kib", 0)
    push(st)
    _lib.tune("peer_ce_kib", 1024)
res["push_sm+pull_ce"] = timed([(push_sm, sa[0]), (pull, sa[1])])
print(json.dumps(res), flush=True)

# round 2: the pull through the async proxy (TMA cp.async.bulk peer global ->
# shared -> local global, put_impl 1) beside SM-store pushes, SM engines only
_lib.tune("peer_ce_kib", 0)
res2 = {}
def pull_tma(st):
    _lib.tune("put_impl", 1)
    pull(st)
    _lib.tune("put_impl", 0)
def push_tma(st):
    _lib.tune("put_impl", 1)
    push(st)
    _lib.tune("put_impl", 0)
res2["pull_tma"] = timed([(pull_tma, sa[0])])
res2["push_sm+pull_tma"] = timed([(push, sa[0]), (pull_tma, sa[1])])
res2["push_tma+pull_sm"] = timed([(push_tma, sa[0]), (pull, sa[1])])
res2["push_tma+pull_tma"] = timed([(push_tma, sa[0]), (pull_tma, sa[1])])
res2["push_sm+pull_sm"] = timed([(push, sa[0]), (pull, sa[1])])
print(json.dumps(res2), flush=True)
