"""Replay-set instantiation/launch costs on the configs[4] LSTM Session:
once steady (period 168), build sets over 1 phase (direct nodes, then every
supported op indirect) and over all phases, and time launches of each."""
import ctypes as C
import os
import sys
import time

os.environ.setdefault("SRFLOW_REPLAY_MAX_PERIOD", "256")
os.environ.setdefault("SRFLOW_REPLAY_TIMING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1805_08430_b200 import _lib  # noqa: E402
from paper_1805_08430_b200.runtime.session import Session  # noqa: E402
from paper_1805_08430_b200.workloads import build_ps_workload, total_params  # noqa: E402

shapes = [(int(35.93e6) // 14 // 4,)] * 14
W = 7
model = 4 * total_params(shapes)
g, placement = build_ps_workload(model, len(shapes), 0.0, W, ps_servers=1, shapes=shapes)
arena = (W + 2) * model + (64 << 20)
sess = Session(g, placement, mode="zerocp", seed=0, capacity_bytes=arena + model + (96 << 20),
               arena_bytes=arena, watchdog_sweeps=10_000,
               devices={s: 0 for s in set(placement.values())}, apply_op="sgd", lr=0.01)
while sess.replay_steady is None and sess._next_iteration < 800:
    sess.run(1)
base, period, recs = sess._steady
print("steady", base, period, flush=True)
st = C.c_void_p()
_lib.call("srf_stream_create", next(iter(sess.spaces.values())).handle, C.byref(st))


first = base - period + 1
cur = [base + 1]           # next iteration to replay (state continuity across variants)


def phase_of(it):
    return (it - first) % period


def run_set(label, execs):
    os.environ["SRFLOW_REPLAY_EXECS"] = str(execs)
    phases = sorted(recs)
    lists = (C.c_void_p * len(phases))(*[recs[j][0].value for j in phases])
    iters = (C.c_int64 * len(phases))(*phases)
    h = C.c_void_p()
    t0 = time.perf_counter()
    _lib.call("srf_replay_set_create", lists, iters, len(phases), C.byref(h))
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(2 * period):
        _lib.call("srf_replay_set_launch", h, phase_of(cur[0]), cur[0], st)
        cur[0] += 1
    _lib.call("srf_stream_sync", st)
    dt = (time.perf_counter() - t0) / (2 * period)
    print(f"{label}: build {t_build:.3f} s, {dt * 1e6:.0f} us/iteration", flush=True)
    _lib.call("srf_replay_set_destroy", h)


def run_per_phase(label):
    for rnd in range(2):
        t0 = time.perf_counter()
        for _ in range(period):
            j = first + phase_of(cur[0])
            _lib.call("srf_oplist_replay", recs[j][0], cur[0] - j, 1, st)
            cur[0] += 1
        _lib.call("srf_stream_sync", st)
        print(f"{label} pass {rnd}: {(time.perf_counter() - t0) / period * 1e6:.0f} us/iteration",
              flush=True)


def device_times(label, kinds):
    """device time per iteration (events around each graph launch, synced)"""
    if kinds is None:
        os.environ.pop("SRFLOW_REPLAY_IND_KINDS", None)
    else:
        os.environ["SRFLOW_REPLAY_IND_KINDS"] = str(kinds)
    os.environ["SRFLOW_REPLAY_EXECS"] = "1"
    phases = sorted(recs)
    lists = (C.c_void_p * len(phases))(*[recs[j][0].value for j in phases])
    iters = (C.c_int64 * len(phases))(*phases)
    h = C.c_void_p()
    _lib.call("srf_replay_set_create", lists, iters, len(phases), C.byref(h))
    ev = [C.c_void_p(), C.c_void_p()]
    for e in ev:
        _lib.call("srf_timing_event_create", next(iter(sess.spaces.values())).handle, C.byref(e))
    tot, host = 0.0, 0.0
    for _ in range(period):
        _lib.call("srf_event_record_on", ev[0], st)
        t0 = time.perf_counter()
        _lib.call("srf_replay_set_launch", h, phase_of(cur[0]), cur[0], st)
        host += time.perf_counter() - t0
        _lib.call("srf_event_record_on", ev[1], st)
        _lib.call("srf_stream_sync", st)
        ms = C.c_float()
        _lib.call("srf_event_elapsed_ms", ev[0], ev[1], C.byref(ms))
        tot += ms.value
        cur[0] += 1
    print(f"{label}: device {tot / period * 1e3:.0f} us/iteration, host launch "
          f"{host / period * 1e6:.0f} us", flush=True)
    _lib.call("srf_replay_set_destroy", h)


def device_per_phase(label):
    ev = [C.c_void_p(), C.c_void_p()]
    for e in ev:
        _lib.call("srf_timing_event_create", next(iter(sess.spaces.values())).handle, C.byref(e))
    tot = 0.0
    for _ in range(period):
        j = first + phase_of(cur[0])
        _lib.call("srf_event_record_on", ev[0], st)
        _lib.call("srf_oplist_replay", recs[j][0], cur[0] - j, 1, st)
        _lib.call("srf_event_record_on", ev[1], st)
        _lib.call("srf_stream_sync", st)
        ms = C.c_float()
        _lib.call("srf_event_elapsed_ms", ev[0], ev[1], C.byref(ms))
        tot += ms.value
        cur[0] += 1
    print(f"{label}: device {tot / period * 1e3:.0f} us/iteration", flush=True)


run_set("set, 4 execs", 4)
run_set("set, 1 exec", 1)
os.environ["SRFLOW_REPLAY_EXECS"] = "4"
device_times("set, synced per launch", None)
run_per_phase("per-phase graphs")
device_per_phase("per-phase graphs (events)")
