"""NVLink pull probe (one process, GPU0 <-> GPU1): per-direction GB/s when
both GPUs PULL from each other at once (each GPU's SMs issue only loads; the
outbound data are read responses), against both pushing at once.  SM loads
(k_put with a peer source) and the TMA variant (put_impl 1)."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

_lib.tune("peer_ce_kib", 0)
sizes = [int(x) << 20 for x in os.environ.get("PROBE_MIB", "4,16,64,256").split(",")]
S_MAX = max(sizes)
sp = [MemorySpace(i, 2 * S_MAX + (8 << 20), device=i) for i in (0, 1)]
_lib.call("srf_connect", sp[0].handle, sp[1].handle)
rg = [s.allocate_region(2 * S_MAX + (4 << 20), register=True) for s in sp]
st = []
for s in sp:
    h = C.c_void_p()
    _lib.call("srf_stream_create", s.handle, C.byref(h))
    st.append(h)
u = _lib.u64_array


def push(i, S):  # GPU i stores its [0, S) into the peer's [S_MAX, S_MAX + S)
    j = 1 - i
    _lib.call("srf_put", sp[i].handle, u([rg[i].base_addr]), u([S]), u([rg[i].access_token]), 1,
              sp[j].handle, rg[j].base_addr + S_MAX, rg[j].access_token, 0, st[i], None)


def pull(i, S):  # GPU i loads the peer's [0, S) into its own [S_MAX, S_MAX + S)
    j = 1 - i
    _lib.call("srf_get", sp[i].handle, rg[i].base_addr + S_MAX, rg[i].access_token,
              sp[j].handle, rg[j].base_addr, rg[j].access_token, S, st[i], None)


def timed(fn, who, S):
    R = max(4, min(200, (8 << 30) // S))
    for i in who:
        fn(i, S)
    for h in st:
        _lib.call("srf_stream_sync", h)
    t0 = time.perf_counter()
    for _ in range(R):
        for i in who:
            fn(i, S)
    for h in st:
        _lib.call("srf_stream_sync", h)
    dt = (time.perf_counter() - t0) / R
    return round(S / dt / 1e9, 1)  # per direction


for S in sizes:
    res = {"mib": S >> 20}
    for impl in (0, 1):
        _lib.tune("put_impl", impl)
        tag = "tma" if impl else "sm"
        res[f"push1_{tag}"] = timed(push, [0], S)
        res[f"pull1_{tag}"] = timed(pull, [0], S)
        res[f"push2_{tag}"] = timed(push, [0, 1], S)
        res[f"pull2_{tag}"] = timed(pull, [0, 1], S)
    _lib.tune("put_impl", 0)
    print(json.dumps(res), flush=True)
