"""Does the configs[4] LSTM Session (7 workers + 1 PS, dynamic gradient
edges) reach a periodic steady state, and with which period?  Runs the
Session with SRFLOW_REPLAY_MAX_PERIOD (default here 64) and prints the
recorder's status, then times run(n) once steady."""
import os
import sys
import time

os.environ.setdefault("SRFLOW_REPLAY_MAX_PERIOD", "256")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1805_08430_b200.runtime.session import Session  # noqa: E402
from paper_1805_08430_b200.workloads import build_ps_workload, total_params  # noqa: E402

shapes = [(int(35.93e6) // 14 // 4,)] * 14
W = int(os.environ.get("PROBE_W", "7"))
model = 4 * total_params(shapes)
g, placement = build_ps_workload(model, len(shapes), 0.0, W, ps_servers=1, shapes=shapes)
arena = (W + 2) * model + (64 << 20)
sess = Session(g, placement, mode="zerocp", seed=0, capacity_bytes=arena + model + (96 << 20),
               arena_bytes=arena, watchdog_sweeps=10_000,
               devices={s: 0 for s in set(placement.values())}, apply_op="sgd", lr=0.01)
import ctypes as C  # noqa: E402
from paper_1805_08430_b200 import _lib  # noqa: E402


def diag(it):
    recs = sess._recs
    if it not in recs:
        return
    for per in range(1, 15):
        if it - per in recs:
            a, b = recs[it - per], recs[it]
            buf = C.create_string_buffer(512)
            _lib.call("srf_oplist_diff", a[0], b[0], per, buf, 512)
            dd = {k: (a[2][k], b[2][k]) for k in a[2] if a[2][k] != b[2][k]}
            rr = {k: (getattr(a[1], k), getattr(b[1], k)) for k in
                  ("bytes_sent", "payload_bytes", "payload_bytes_copied", "copy_events",
                   "serialize_bytes", "arena_peak_bytes", "polls", "sim_time_us")
                  if getattr(a[1], k) != getattr(b[1], k)}
            print(f"   p={per}: work {buf.value.decode()} | row diff {rr} | delta diff "
                  f"{str(dd)[:300]}", flush=True)


t0 = time.perf_counter()
for it in range(1, 900):
    sess.run(1)
    if it % 8 == 0 or sess.replay_steady is not None:
        print(it, round(time.perf_counter() - t0, 2), sess.replay_status, flush=True)
    if it in (40, 41):
        diag(it)
    if sess.replay_steady is not None or "given up" in sess.replay_status:
        break
if sess.replay_steady is not None:
    per = sess.replay_steady[1]
    for k in range(3):
        t0 = time.perf_counter()
        sess.run(1)
        torch.cuda.synchronize()
        print("one replayed iteration incl. its graph build", round(time.perf_counter() - t0, 4),
              "s", flush=True)
    base, p_, recs = sess._steady
    for j in list(recs)[:1] + list(recs)[-1:]:
        buf = C.create_string_buffer(256)
        nops = C.c_uint32()
        _lib.call("srf_oplist_info", recs[j][0], C.byref(nops), None, buf, 256)
        print("recording", j, "ops", nops.value, buf.value.decode(), flush=True)
    t0 = time.perf_counter()
    sess.run(per)
    torch.cuda.synchronize()
    print("first pass over the period (graph builds)", round(time.perf_counter() - t0, 2), "s",
          flush=True)
    t0 = time.perf_counter()
    sess.run(per)
    torch.cuda.synchronize()
    print("second pass", round(time.perf_counter() - t0, 3), "s", flush=True)
    t0 = time.perf_counter()
    sess.run(500)
    torch.cuda.synchronize()
    print("steady it/s", 500 / (time.perf_counter() - t0), sess.replay_status, flush=True)
