import os, sys, time
sys.path.insert(0, "/root/repo")
os.environ["SRFLOW_REPLAY_MAX_PERIOD"] = "1"
from paper_1805_08430_b200.runtime.session import Session
from paper_1805_08430_b200.workloads import build_ps_workload, total_params
shapes = [(int(35.93e6) // 14 // 4,)] * 14
W = 7
model = 4 * total_params(shapes)
g, placement = build_ps_workload(model, len(shapes), 0.0, W, ps_servers=1, shapes=shapes)
arena = (W + 2) * model + (64 << 20)
sess = Session(g, placement, mode="zerocp", seed=0, capacity_bytes=arena + model + (96 << 20),
               arena_bytes=arena, watchdog_sweeps=10_000,
               devices={s: 0 for s in set(placement.values())}, apply_op="sgd", lr=0.01, replay=False)
hist = []
for it in range(1, 600):
    sess.run(1)
    st = tuple((s, tuple(a._starts), tuple(a._lens), tuple(sorted(a._live))) for s, a in sorted(sess.rdma_arenas.items()))
    hist.append(st)
    for L in range(1, len(hist)):
        if hist[-1] == hist[-1 - L]:
            print("iteration", it, "state repeats with period", L, flush=True)
            sys.exit(0)
    if it % 50 == 0:
        print(it, "no repeat yet", flush=True)
