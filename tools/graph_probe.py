"""Does a CUDA graph of R (event, K1, event, K2) rounds keep per-launch event
timing, and how much launch overhead does it remove?"""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1805_08430_b200 import _lib

S = 256 << 20
ring = bench.SendRecvRing(S, 0, 1, 0)
R = 50
ev = [ring.event() for _ in range(2 * R)]
a, b = ring.event(), ring.event()
for _ in range(3):
    ring.put(); ring.consume()
ring.sync()
g = C.c_void_p()
_lib.call("srf_graph_begin", ring.stream)
for i in range(R):
    ring.record(ev[2 * i]); ring.put(); ring.record(ev[2 * i + 1]); ring.consume()
_lib.call("srf_graph_end", ring.stream, C.byref(g))
_lib.call("srf_graph_launch", g, ring.stream)
ring.sync()
ring.record(a)
_lib.call("srf_graph_launch", g, ring.stream)
ring.record(b)
ring.sync()
put = [ring.elapsed_ms(ev[2 * i], ev[2 * i + 1]) for i in range(R)]
print(json.dumps({"graph_round_us": ring.elapsed_ms(a, b) / R * 1e3,
                  "graph_k1_us": statistics.fmean(put) * 1e3,
                  "k1_min_us": min(put) * 1e3, "verified": ring.verify()}))
# same without the graph
ring.record(a)
for i in range(R):
    ring.record(ev[2 * i]); ring.put(); ring.record(ev[2 * i + 1]); ring.consume()
ring.record(b)
ring.sync()
put = [ring.elapsed_ms(ev[2 * i], ev[2 * i + 1]) for i in range(R)]
print(json.dumps({"stream_round_us": ring.elapsed_ms(a, b) / R * 1e3,
                  "stream_k1_us": statistics.fmean(put) * 1e3}))
