"""Why a Session does not reach a replayable steady state: per iteration,
the recorder's status and, for periods 1-8, where the newest iteration's
device work stops repeating the one p iterations before."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.runtime.session import Session
from paper_1805_08430_b200.workloads import build_ps_workload

for name, (args, kw) in {"ps24k_dyn": ((24_000, 2, 0.0, 2), {"mechanism_override": "dynamic"}),
                         "ps7w": ((7_000, 5, 0.0, 7), {})}.items():
    g, p = build_ps_workload(*args)
    s = Session(g, p, seed=3, devices={v: 0 for v in set(p.values())}, **kw)
    for it in range(1, 17):
        rep = s.run(1)
        r = rep.rows[-1]
        print(name, it, r.polls, r.arena_peak_bytes, r.bytes_sent, r.sim_time_us, "|",
              s.replay_status, flush=True)
        if s._steady is not None:
            break
        recs = s._recs
        if it in recs:
            for per in range(1, 9):
                if it - per in recs:
                    buf = C.create_string_buffer(512)
                    _lib.call("srf_oplist_diff", recs[it - per][0], recs[it][0], per, buf, 512)
                    same_row = s._same_row(recs[it - per][1], recs[it][1])
                    same_delta = s._same_delta(recs[it - per][2], recs[it][2])
                    print(f"   p={per}: row {same_row} delta {same_delta} work {buf.value.decode()}")
    s.close()
