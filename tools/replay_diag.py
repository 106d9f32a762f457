"""Why a Session does not reach a replayable steady state: per iteration,
the recorder's status (device-work diff against the previous iteration)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200.runtime.session import Session
from paper_1805_08430_b200.workloads import build_ps_workload

for name, (args, kw) in {"ps24k_dyn": ((24_000, 2, 0.0, 2), {"mechanism_override": "dynamic"}),
                         "ps7w": ((7_000, 5, 0.0, 7), {})}.items():
    g, p = build_ps_workload(*args)
    s = Session(g, p, seed=3, devices={v: 0 for v in set(p.values())}, **kw)
    for it in range(1, 13):
        rep = s.run(1)
        r = rep.rows[-1]
        print(name, it, r.polls, r.arena_peak_bytes, r.bytes_sent, "|", s.replay_status, flush=True)
    s.close()
