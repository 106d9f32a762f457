"""Pipelined static edge (srf_edge_*) throughput: rounds of S bytes over one
edge with `slots` receive regions, consumer on the receiving GPU.  One
process.  Modes: same GPU (HBM), GPU0 -> GPU1 (NVLink one direction), and
both directions at once (the N=2 ring).  Device time of each side's stream
(events), GB/s = rounds * S / time.  Usage: python tools/edge_probe.py [sizes...]"""
import ctypes as C
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace
from paper_1805_08430_b200.runtime.protocol import PipelinedStaticEdge, PulledStaticEdge

KIB, MIB = 1 << 10, 1 << 20
ndev = _lib.device_count()


def r256(n):
    return (n + 255) & ~255


class Side:
    def __init__(self, src_dev, dst_dev, S, slots, nsrc, mirror=False, pull=0):
        self.S, self.slots, self.pull = S, slots, pull
        self.src_stride, self.slot_stride = r256(S), r256(S + 1)
        self.a = MemorySpace(10 + src_dev, nsrc * self.src_stride + 4 * MIB, seed=1,
                             device=src_dev)
        self.b = MemorySpace(20 + dst_dev, slots * self.slot_stride + 4 * MIB, seed=2,
                             device=dst_dev)
        _lib.call("srf_connect", self.a.handle, self.b.handle)
        self.ra = self.a.allocate_region(nsrc * self.src_stride, register=True)
        self.credit = None
        if mirror:
            self.credit = self.a.allocate_region(4 * slots)
            self.a.write_raw(self.credit.base_addr, b"\x00" * 4 * slots)
        self.rb = self.b.allocate_region(slots * self.slot_stride, register=True)
        for i in range(slots):
            self.b.write_raw(self.rb.base_addr + i * self.slot_stride + S, b"\x00")
        self.a.sync(), self.b.sync()
        self.sa, self.sb = C.c_void_p(), C.c_void_p()
        _lib.call("srf_stream_create", self.a.handle, C.byref(self.sa))
        _lib.call("srf_stream_create", self.b.handle, C.byref(self.sb))
        if pull:
            # pull edge: the receiver's GPU runs the edge; the consumer gets
            # its own stream there; the sender only posts rounds
            self.posted = self.b.allocate_region(8)
            self.sc = C.c_void_p()
            _lib.call("srf_stream_create", self.b.handle, C.byref(self.sc))
            self.edge = PulledStaticEdge(self.a, self.ra.base_addr, self.ra.access_token, S, nsrc,
                                         self.src_stride, self.b, self.rb, slots,
                                         self.slot_stride, self.posted.base_addr, tma=pull == 2)
        else:
            self.edge = PipelinedStaticEdge(self.a, self.ra, S, nsrc, self.src_stride, self.b,
                                            self.rb.base_addr, self.rb.access_token, slots,
                                            self.slot_stride,
                                            credit_addr=self.credit.base_addr if mirror else None)
        self.ev = [C.c_void_p(), C.c_void_p()]
        for e in self.ev:
            _lib.call("srf_timing_event_create", self.b.handle if pull else self.a.handle,
                      C.byref(e))
        self.next = 0

    def consume(self, rounds):
        PipelinedStaticEdge.consume(self.b, self.rb.base_addr, self.slots, self.slot_stride,
                                    self.S, self.next, rounds,
                                    stream=self.sc if self.pull else self.sb,
                                    credit=None if self.credit is None else
                                    (self.a, self.credit.base_addr))

    def launch(self, rounds, timed=False):
        """(every side's consume() must have been queued first: a consumer
        launched after a full-GPU sender grid may not fit beside it)"""
        st = self.sb if self.pull else self.sa
        if self.pull:
            PulledStaticEdge.post(self.a, self.b, self.posted.base_addr, self.next + rounds,
                                  stream=self.sa)
        if timed:
            _lib.call("srf_event_record_on", self.ev[0], st)
        if self.pull:
            self.edge.recv(rounds, self.sb)
        else:
            self.edge.send(rounds, self.sa)
        if timed:
            _lib.call("srf_event_record_on", self.ev[1], st)
        self.next += rounds

    def sync(self):
        _lib.call("srf_stream_sync", self.sa)
        _lib.call("srf_stream_sync", self.sb)
        if self.pull:
            _lib.call("srf_stream_sync", self.sc)
        self.a.sync(), self.b.sync()

    def ms(self):
        t = C.c_float()
        _lib.call("srf_event_elapsed_ms", self.ev[0], self.ev[1], C.byref(t))
        return t.value

    def close(self):
        self.edge.close()
        for s in (self.sa, self.sb) + ((self.sc,) if self.pull else ()):
            _lib.call("srf_stream_destroy", s)
        self.a.close(), self.b.close()


def run(mode, S, slots, rounds, mirror=False, pull=0):
    pairs = {"hbm": [(0, 0)], "nvl1": [(0, 1)], "nvl2": [(0, 1), (1, 0)]}[mode]
    nsrc = max(1, min(8, (256 * MIB) // max(S, 1)))
    sides = [Side(s, d, S, slots, nsrc, mirror, pull) for s, d in pairs]
    for sd in sides:
        sd.consume(max(2, rounds // 4))
    for sd in sides:
        sd.launch(max(2, rounds // 4))
    for sd in sides:
        sd.sync()
    for sd in sides:
        sd.consume(rounds)
    for sd in sides:
        sd.launch(rounds, timed=True)
    for sd in sides:
        sd.sync()
    ms = max(sd.ms() for sd in sides)
    info = sides[0].edge.info()
    for sd in sides:
        sd.close()
    return {"mode": mode, "pull": pull, "bytes": S, "slots": slots, "rounds": rounds, "mirror": mirror,
            "us_per_round": round(ms * 1e3 / rounds, 3),
            "gbps_per_dir": round(S * rounds / (ms / 1e3) / 1e9, 1),
            "chunk": info["chunk"], "ctas": info["ctas"]}


if __name__ == "__main__":
    # PROBE_MODES (nvl1,nvl2,hbm), PROBE_CHUNKS (KiB; 0 = automatic),
    # PROBE_SLOTS, PROBE_MIRROR (0,1), PROBE_CTAS (CTAs per SM), PROBE_RELEASE
    # (flag-only consumer clears with release.sys: 0,1), PROBE_PULL (0 push,
    # 1 pull with SM loads, 2 pull with TMA bulk copies); sizes in argv
    sizes = [int(x) for x in sys.argv[1:]] or [MIB, 4 * MIB, 16 * MIB, 64 * MIB, 256 * MIB]
    env = lambda k, d: [int(x) for x in os.environ.get(k, d).split(",")]
    modes = os.environ.get("PROBE_MODES", "nvl1,nvl2,hbm").split(",")
    if ndev < 2:
        modes = [m for m in modes if m == "hbm"]
    grid = itertools.product(env("PROBE_PULL", "0"), env("PROBE_RELEASE", "0"), env("PROBE_CTAS", "2"), modes, sizes,
                             env("PROBE_CHUNKS", "0"), env("PROBE_MIRROR", "0"),
                             env("PROBE_SLOTS", "2,4,8,16"))
    for pull, rel, ctas, mode, S, chunk_kib, mirror, slots in grid:
        _lib.tune("consume_release", rel)
        # PROBE_CTAS: CTAs per SM (1..4) or, above 4, CTAs in total
        _lib.tune("edge_ctas_per_sm", ctas if ctas <= 4 else 2)
        _lib.tune("edge_ctas", ctas if ctas > 4 else 0)
        _lib.tune("edge_chunk_kib", chunk_kib)
        # enough rounds that every slot is reused many times
        rounds = max(16 * slots, min(400, int(4e9 // S)))
        row = run(mode, S, slots, rounds, bool(mirror and mode != "hbm"), pull)
        row.update(chunk_kib_knob=chunk_kib, ctas_per_sm=ctas, consume_release=rel)
        print(json.dumps(row), flush=True)
    _lib.tune("edge_chunk_kib", 0)
    _lib.tune("edge_ctas_per_sm", 2)
    _lib.tune("consume_release", 0)
    _lib.tune("edge_ctas", 0)
