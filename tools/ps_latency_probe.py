"""Latency-bound PS config (MLP parity set, N=1): us per iteration for each
schedule, device-timed over many iterations."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.ps import PsLayout, PsStep
from paper_1805_08430_b200.workloads import mlp_shapes

L = PsLayout(mlp_shapes(), 2, 1)
ps = PsStep(L, seed=0, op="sgd", lr=0.01)
ev = [C.c_void_p(), C.c_void_p()]
for e in ev:
    _lib.call("srf_timing_event_create", ps.stream_space.handle, C.byref(e))
it = 0


def timed(fn, n):
    global it
    fn(it + 1, 50)
    it += 50
    ps.sync()
    _lib.call("srf_event_record_on", ev[0], ps.stream)
    fn(it + 1, n)
    it += n
    _lib.call("srf_event_record_on", ev[1], ps.stream)
    ps.sync()
    ms = C.c_float()
    _lib.call("srf_event_elapsed_ms", ev[0], ev[1], C.byref(ms))
    return round(ms.value * 1e3 / n, 2)


def phases(i0, n):
    ps.use_schedule("phases")
    for k in range(n):
        ps.step(i0 + k)


def exchange(i0, n):
    ps.use_schedule("exchange")
    for k in range(n):
        ps.step(i0 + k)


res = {"phases_us": timed(phases, 2000), "exchange_us": timed(exchange, 2000),
       "exchange_x64_us": timed(lambda i0, n: ps.run_exchange(i0, n), 2000),
       "exchange_x512_us": timed(lambda i0, n: ps.run_exchange(i0, n, per_launch=512), 2000),
       "persistent_us": timed(lambda i0, n: ps.run_persistent(i0, n), 2000)}
print(json.dumps(res), flush=True)
ps.close()
