"""Is the cross-process SM-store 'cap' an alignment effect?  K1 SM stores
GPU0 -> GPU1, 256 MiB, source/destination offsets co-aligned mod 32 or not,
one process (peer access) and two processes (IPC import)."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

_lib.tune("peer_ce_kib", 0)
S = 256 << 20
u = _lib.u64_array
mode = sys.argv[1] if len(sys.argv) > 1 else "inproc"


def rate(src_sp, rs, dst_sp, dst_addr, dst_tok, soff, doff, st, R=10):
    flag = rs.base_addr + S + 4096
    src_sp.write_raw(flag, b"\x01")
    def go():
        _lib.call("srf_put", src_sp.handle, u([rs.base_addr + soff, flag]), u([S, 1]),
                  u([rs.access_token] * 2), 2, dst_sp.handle, dst_addr + doff, dst_tok, 0, st,
                  None)
    go(); _lib.call("srf_stream_sync", st)
    t0 = time.perf_counter()
    for _ in range(R):
        go()
    _lib.call("srf_stream_sync", st)
    return round(S * R / (time.perf_counter() - t0) / 1e9, 1)


def pull_rate(dst_sp, rd, src_sp, src_addr, src_tok, soff, doff, st, R=10):
    def go():
        _lib.call("srf_get", dst_sp.handle, rd.base_addr + doff, rd.access_token, src_sp.handle,
                  src_addr + soff, src_tok, S, st, None)
    go(); _lib.call("srf_stream_sync", st)
    t0 = time.perf_counter()
    for _ in range(R):
        go()
    _lib.call("srf_stream_sync", st)
    return round(S * R / (time.perf_counter() - t0) / 1e9, 1)


if mode == "inproc":
    a = MemorySpace(0, S + (16 << 20), device=0)
    b = MemorySpace(1, S + (16 << 20), device=1)
    _lib.call("srf_connect", a.handle, b.handle)
    ra, rb = a.allocate_region(S + (8 << 20), True), b.allocate_region(S + (8 << 20), True)
    st = C.c_void_p()
    _lib.call("srf_stream_create", a.handle, C.byref(st))
    res = {}
    for soff, doff in ((0, 0), (0, 8), (8, 0), (0, 16), (0, 4), (3, 5)):
        res[f"s{soff}_d{doff}"] = rate(a, ra, b, rb.base_addr, rb.access_token, soff, doff, st)
        res[f"pull_s{soff}_d{doff}"] = pull_rate(a, ra, b, rb.base_addr, rb.access_token,
                                                 soff, doff, st)
    print(json.dumps({"mode": mode, **res}), flush=True)
else:
    import bench
    from paper_1805_08430_b200.distributed import gather_descriptors, init_process_group
    rank, world, local = init_process_group("nccl")
    torch.cuda.set_device(local)
    a = MemorySpace(rank, S + (16 << 20), device=local)
    ra = a.allocate_region(S + (8 << 20), True)
    table = gather_descriptors(a.export())
    peer = MemorySpace.import_remote(table[(rank + 1) % world], local)
    _rid, pbase, _plen, _r, ptok = table[(rank + 1) % world]["regions"][0]
    st = C.c_void_p()
    _lib.call("srf_stream_create", a.handle, C.byref(st))
    res = {}
    for soff, doff in ((0, 0), (0, 8), (8, 0), (0, 16), (0, 4), (3, 5)):
        bench.barrier_sync()
        r = rate(a, ra, peer, pbase, ptok, soff, doff, st) if rank == 0 else None
        bench.barrier_sync()
        res[f"s{soff}_d{doff}"] = r
    if rank == 0:
        print(json.dumps({"mode": mode, **res}), flush=True)
