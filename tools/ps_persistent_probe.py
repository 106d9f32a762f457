"""Eager per-phase launches vs one persistent cooperative launch, per PS config (N=1)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.ps import PsLayout, PsStep
from paper_1805_08430_b200.workloads import mlp_shapes, vgg16_shapes

cfgs = {"mlp": (mlp_shapes(), 2, 1), "fcn5": ([(int(204.47e6) // 40,)] * 10, 2, 1),
        "lstm": ([(int(35.93e6) // 56,)] * 14, 7, 1), "vgg": (vgg16_shapes(), 1, 1)}
for name, (shapes, W, P) in cfgs.items():
    ps = PsStep(PsLayout(shapes, W, P), seed=0, op="sgd", lr=0.01)
    ev = [C.c_void_p(), C.c_void_p()]
    for e in ev:
        _lib.call("srf_timing_event_create", ps.stream_space.handle, C.byref(e))
    n = 200 if name == "mlp" else 20
    it = 0
    for _ in range(3):
        it += 1
        ps.step(it)
    ps.sync()
    _lib.call("srf_event_record_on", ev[0], ps.stream)
    for _ in range(n):
        it += 1
        ps.step(it)
    _lib.call("srf_event_record_on", ev[1], ps.stream)
    ps.sync()
    ms = C.c_float()
    _lib.call("srf_event_elapsed_ms", ev[0], ev[1], C.byref(ms))
    eager = n / (ms.value / 1e3)
    _lib.call("srf_event_record_on", ev[0], ps.stream)
    ps.run_persistent(it + 1, n)
    it += n
    _lib.call("srf_event_record_on", ev[1], ps.stream)
    ps.sync()
    _lib.call("srf_event_elapsed_ms", ev[0], ev[1], C.byref(ms))
    pers = n / (ms.value / 1e3)
    print(json.dumps({"config": name, "eager_it_s": round(eager, 1),
                      "persistent_it_s": round(pers, 1)}), flush=True)
    ps.close()
