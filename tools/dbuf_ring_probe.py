"""Two receive blocks per static edge: does overlapping round k+1's put with
round k's consume lift mid-size NVLink rounds toward 0.8 of the link?

Ring rank r -> r+1 (torchrun, N>=2).  'single' is the bench's sweep_nvlink
static row (one block: put(k), consume(k)).  'double' alternates two
SendRecvRing edges A/B on one stream in the order put(k+1), consume(k), so a
round's handshake (credit, flag, K2) runs behind the next round's body.  Same
graph replay and max-over-ranks device timing as bench.sweep_nvlink.
"""
import ctypes as C
import json
import time
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.distributed import env_world, init_process_group

MIB = 1 << 20


def main():
    rank, world, local = env_world()
    torch.cuda.set_device(local)
    init_process_group("nccl")
    for size in (1 << 10, 1 * MIB, 4 * MIB, 16 * MIB, 64 * MIB):
        rounds = 100 if size <= 4 * MIB else 20
        a = bench.SendRecvRing(size, rank, world, local)
        b = bench.SendRecvRing(size, rank, world, local)
        b.stream = a.stream
        for _ in range(4):
            a.put()
            a.consume()
        a.sync()
        single = bench._ring_graph_us(a.stream, lambda: (a.put(), a.consume()), rounds, a.src)

        def pair():
            b.put()
            a.consume()
            a.put()
            b.consume()

        a.put()  # round 0 outstanding: every replay is steady state
        for _ in range(2):
            pair()
        a.sync()
        double = bench._ring_graph_us(a.stream, pair, rounds // 2, a.src) / 2
        a.consume()
        a.sync()
        va = a.verify()
        vb = b.verify()
        ok = va and vb
        # two edges in flight: A and B on their own streams, one graph each,
        # launched back to back; wall clock around both syncs, max over ranks
        b.stream = C.c_void_p()
        _lib.call("srf_stream_create", b.src.handle, C.byref(b.stream))
        graphs = []
        for ring in (a, b):
            g = C.c_void_p()
            _lib.call("srf_graph_begin", ring.stream)
            for _ in range(rounds):
                ring.put()
                ring.consume()
            _lib.call("srf_graph_end", ring.stream, C.byref(g))
            graphs.append(g)
        def both():
            bench.barrier_sync()
            t0 = time.perf_counter()
            for ring, g in zip((a, b), graphs):
                _lib.call("srf_graph_launch", g, ring.stream)
            for ring in (a, b):
                _lib.call("srf_stream_sync", ring.stream)
            return time.perf_counter() - t0
        both()
        two = bench.dist_max(min(both() for _ in range(3))) * 1e6 / rounds
        for g in graphs:
            _lib.call("srf_graph_destroy", g)
        va2 = a.verify()
        vb2 = b.verify()
        ok = ok and va2 and vb2
        row = {"bytes": size, "single_us": single, "double_us": round(double, 3),
               "two_streams_us_per_round_pair": round(two, 3),
               "two_streams_gbps": round(2 * size / two / 1e3, 1),
               "frac_770_two_streams": round(2 * size / two / 1e3 / 770.0, 3),
               "single_gbps": round(size / single / 1e3, 1),
               "double_gbps": round(size / double / 1e3, 1),
               "frac_770_double": round(size / double / 1e3 / 770.0, 3), "verified": ok}
        if rank == 0:
            print(json.dumps(row), flush=True)
        bench.barrier_sync()


if __name__ == "__main__":
    main()
