"""K1 launch-geometry probe on one GPU: the bench loop (put with credit +
consumer flag wait) for unroll x CTAs/SM x threads; K1 time by CUDA events."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1805_08430_b200 import _lib

S = int(os.environ.get("PROBE_BYTES", 256 << 20))
ring = bench.SendRecvRing(S, 0, 1, 0)
R = 30
peak, _ = bench.measured_peaks()
for unroll, vec32 in ((8, 0), (8, 1), (4, 1)):
    for ctas in (2, 4, 8):
        for threads in (256, 512):
            _lib.tune("vec32", vec32)
            _lib.tune("unroll", unroll)
            _lib.tune("ctas_per_sm", ctas)
            _lib.tune("copy_threads", threads)
            ev = [ring.event() for _ in range(2 * R)]
            a, b = ring.event(), ring.event()
            for _ in range(3):
                ring.put(); ring.consume()
            ring.sync()
            ring.record(a)
            for i in range(R):
                ring.record(ev[2 * i]); ring.put(); ring.record(ev[2 * i + 1]); ring.consume()
            ring.record(b)
            ring.sync()
            put_ms = statistics.fmean(ring.elapsed_ms(ev[2 * i], ev[2 * i + 1]) for i in range(R))
            round_ms = ring.elapsed_ms(a, b) / R
            print(json.dumps({"unroll": unroll, "vec32": vec32, "ctas": ctas, "threads": threads,
                              "k1_us": round(put_ms * 1e3, 2),
                              "k1_hbm_frac": round((2 * S + 1) / (put_ms / 1e3) / 1e9 / peak, 4),
                              "round_us": round(round_ms * 1e3, 2),
                              "payload_gbps": round(S / (round_ms / 1e3) / 1e9, 1)}), flush=True)
print("verified", ring.verify())
