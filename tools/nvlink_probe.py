"""Probe: K1 push vs K4 pull, vector vs TMA-bulk implementation, one and two
directions over NVLink, next to the copy engine.  Device time via CUDA events."""
import ctypes as C
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

S = int(os.environ.get("PROBE_BYTES", 256 << 20))
REPS = 20
ndev = torch.cuda.device_count()
out = {"bytes": S, "devices": ndev, "results": []}


class Side:
    def __init__(self, sid, dev):
        self.sp = MemorySpace(sid, 2 * S + (64 << 20), device=dev)
        self.r = self.sp.allocate_region(2 * S + (32 << 20), True)
        self.src = self.r.base_addr
        self.dst = self.r.base_addr + S + 4096
        self.flag = self.r.base_addr + 2 * S + 8192
        self.sp.write_raw(self.flag, b"\x01")
        self.st = C.c_void_p()
        _lib.call("srf_stream_create", self.sp.handle, C.byref(self.st))
        self.ev = [C.c_void_p(), C.c_void_p()]
        for e in self.ev:
            _lib.call("srf_timing_event_create", self.sp.handle, C.byref(e))

    def push_to(self, other):
        _lib.call("srf_put", self.sp.handle, _lib.u64_array([self.src, self.flag]),
                  _lib.u64_array([S, 1]), _lib.u64_array([self.r.access_token] * 2), 2,
                  other.sp.handle, other.dst, other.r.access_token, 0, self.st, None)

    def pull_from(self, other):
        _lib.call("srf_get", self.sp.handle, self.dst, self.r.access_token, other.sp.handle,
                  other.src, other.r.access_token, S, self.st, None)

    def elapsed(self):
        ms = C.c_float()
        _lib.call("srf_event_elapsed_ms", self.ev[0], self.ev[1], C.byref(ms))
        return ms.value / 1e3


def run(sides_ops):
    """sides_ops: list of (side, fn) issued concurrently; returns per-op GB/s."""
    for side, fn in sides_ops:
        for _ in range(3):
            fn()
    for side, _ in sides_ops:
        _lib.call("srf_stream_sync", side.st)
    for side, fn in sides_ops:
        _lib.call("srf_event_record_on", side.ev[0], side.st)
    for _ in range(REPS):
        for side, fn in sides_ops:
            fn()
    for side, _ in sides_ops:
        _lib.call("srf_event_record_on", side.ev[1], side.st)
    for side, _ in sides_ops:
        _lib.call("srf_stream_sync", side.st)
    return [S * REPS / side.elapsed() / 1e9 for side, _ in sides_ops]


pairs = [(0, 1)] if ndev > 1 else []
pairs.append((0, 0))
for d0, d1 in pairs:
    a, b = Side(0, d0), Side(1, d1)
    _lib.call("srf_connect", a.sp.handle, b.sp.handle)
    for impl in (0, 1):
        _lib.tune("put_impl", impl)
        for ctas in ((1, 2, 4) if impl == 0 else (2,)):
            _lib.tune("ctas_per_sm", ctas)
            rec = {"devs": [d0, d1], "impl": ["vector", "tma_bulk"][impl], "ctas_per_sm": ctas}
            rec["push_1dir"] = run([(a, lambda: a.push_to(b))])[0]
            rec["pull_1dir"] = run([(b, lambda: b.pull_from(a))])[0]
            if d0 != d1:
                rec["push_2dir"] = run([(a, lambda: a.push_to(b)), (b, lambda: b.push_to(a))])
                rec["pull_2dir"] = run([(a, lambda: a.pull_from(b)), (b, lambda: b.pull_from(a))])
            out["results"].append(rec)
            print(json.dumps(rec), flush=True)
    # verify the bulk path moved the right bytes
    _lib.tune("put_impl", 1)
    data = torch.randint(0, 255, (S,), dtype=torch.uint8, device=f"cuda:{d0}")
    a.sp.view(a.r, a.src - a.r.base_addr, S).copy_(data)
    torch.cuda.synchronize(d0)
    a.push_to(b)
    _lib.call("srf_stream_sync", a.st)
    ok = torch.equal(b.sp.view(b.r, b.dst - b.r.base_addr, S).cpu(), data.cpu())
    ok &= b.sp.read_raw(b.dst + S, 1) == b"\x01"
    b.pull_from(a)
    _lib.call("srf_stream_sync", b.st)
    print("bulk verify", d0, d1, ok, flush=True)
    out.setdefault("bulk_verified", []).append(bool(ok))
    if d0 != d1:
        x = torch.empty(S, dtype=torch.uint8, device=f"cuda:{d0}")
        y = torch.empty(S, dtype=torch.uint8, device=f"cuda:{d1}")
        for _ in range(3):
            y.copy_(x)
        torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
        t0 = time.perf_counter()
        for _ in range(REPS):
            y.copy_(x)
        torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
        out["copy_engine_gbps"] = S * REPS / (time.perf_counter() - t0) / 1e9
        print("copy engine", out["copy_engine_gbps"], flush=True)
    _lib.tune("put_impl", 0)
    _lib.tune("ctas_per_sm", 2)
    a.sp.close(); b.sp.close()
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/nvlink_probe.json", "w") as fh:
    json.dump(out, fh, indent=1)
