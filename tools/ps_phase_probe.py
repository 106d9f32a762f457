"""Per-phase device time of the PS step on every rank (torchrun): events
between the phase launches on the rank's stream, averaged over R steps.
A phase's time includes its spins on flags other GPUs set."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.distributed import init_process_group
from paper_1805_08430_b200.ps import PsLayout, PsStep
from paper_1805_08430_b200.workloads import vgg16_shapes

rank, world, local = init_process_group("nccl")
torch.cuda.set_device(local)
balanced = os.environ.get("PROBE_PLACEMENT", "round_robin")
cfg = os.environ.get("PROBE_CFG", "vgg")
if cfg == "vgg":
    L = PsLayout(vgg16_shapes(), world, world, colocate=True, placement=balanced,
                 partition_bytes=int(os.environ["PROBE_PARTITION"])
                 if os.environ.get("PROBE_PARTITION") else None)
elif cfg == "fcn5":
    L = PsLayout([(int(204.47e6) // 10 // 4,)] * 10, 2, 1, False)
else:
    L = PsLayout([(int(35.93e6) // 14 // 4,)] * 14, 7, 1, False)
mode = os.environ.get("PROBE_MODE", "phases")
if mode != "phases":
    # whole-step wall time of the phase or exchange schedule, max over ranks
    import time
    ps = PsStep(L, rank=rank, world=world, device=local, seed=0, op="sgd", lr=0.01,
                schedule="exchange" if mode == "exchange" else "phases")
    for it in range(1, 6):
        ps.step(it)
    ps.sync()
    bench.barrier_sync()
    t0 = time.perf_counter()
    R = 40
    for it in range(6, 6 + R):
        ps.step(it)
    ps.sync()
    bench.barrier_sync()
    dt = bench.dist_max(time.perf_counter() - t0) / R
    if os.environ.get("PROBE_HOST"):
        # host issue time vs device completion, one step at a time
        ti, ts = 0.0, 0.0
        for it2 in range(6 + R, 6 + R + 10):
            bench.barrier_sync()
            a0 = time.perf_counter()
            ps.step(it2)
            a1 = time.perf_counter()
            ps.sync()
            a2 = time.perf_counter()
            ti += (a1 - a0) / 10
            ts += (a2 - a1) / 10
        print(json.dumps({"rank": rank, "cfg": cfg, "mode": mode, "issue_us": round(ti * 1e6, 1),
                          "sync_us": round(ts * 1e6, 1)}), flush=True)
        R += 10
    if mode != "phases":
        from oracle import port
        mine = [v for v in range(len(L.shapes)) if L.shard_of(v) % world == rank]
        small = [v for v in mine if L.nbytes(v) < (4 << 20)][:2]
        want = port.ps_expected_device(L.shapes, L.workers, 0, range(1, 6 + R), op="sgd",
                                       lr=0.01, only=small)
        for v in small:
            assert ps.variable(v).tobytes() == want[v].tobytes(), ("mismatch", v)
    if rank == 0:
        print(json.dumps({"mode": mode, "cfg": cfg,
                          "placement": balanced, "step_us": round(dt * 1e6, 1),
                          "knobs": {k: v for k, v in os.environ.items()
                                    if k.startswith("SRFLOW_")}}), flush=True)
    ps.close()
    sys.exit(0)
ps = PsStep(L, rank=rank, world=world, device=local, seed=0, op="sgd", lr=0.01)
sp = ps.stream_space
names = ["push", "gen", "meta", "apply"]
ev = []
for _ in range(len(names) + 1):
    e = C.c_void_p()
    _lib.call("srf_timing_event_create", sp.handle, C.byref(e))
    ev.append(e)
R = 20
acc = {n: 0.0 for n in names}
acc["step"] = 0.0
b = ps.batches
for it in range(1, R + 6):
    bench.barrier_sync()
    _lib.call("srf_event_record_on", ev[0], ps.stream)
    _lib.call("srf_batch_launch", b["push"], ps.stream, it, 0, 0) if b["push"] else None
    _lib.call("srf_event_record_on", ev[1], ps.stream)
    for g in b["gen"].values():
        _lib.call("srf_batch_launch", g, ps.stream, it, 1, 0)
    _lib.call("srf_event_record_on", ev[2], ps.stream)
    if b["meta"]:
        _lib.call("srf_batch_launch", b["meta"], ps.stream, it, 0, 0)
    _lib.call("srf_event_record_on", ev[3], ps.stream)
    for a in b["apply"].values():
        _lib.call("srf_batch_launch", a, ps.stream, it, 0, 0)
    _lib.call("srf_event_record_on", ev[4], ps.stream)
    _lib.call("srf_stream_sync", ps.stream)
    if it > 5:
        for i, n in enumerate(names):
            f = C.c_float()
            _lib.call("srf_event_elapsed_ms", ev[i], ev[i + 1], C.byref(f))
            acc[n] += f.value / R
        f = C.c_float()
        _lib.call("srf_event_elapsed_ms", ev[0], ev[4], C.byref(f))
        acc["step"] += f.value / R
out = {"rank": rank, "placement": balanced, "knobs": {k: v for k, v in os.environ.items()
                                                      if k.startswith("SRFLOW_")},
       **{k: round(v * 1000, 1) for k, v in acc.items()}}
print(json.dumps(out), flush=True)
ps.close()
