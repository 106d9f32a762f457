"""EXTENSION: the pipelined dynamic edge (srf_dyn_edge_*, device_stream.cuh
k_dyn_*) - dynamic allocation with `slots` metadata blocks, on-demand
destination blocks from a device ring arena and one persistent TMA receiver.
Every round's payload as checksummed by the consumer equals the bytes the
sender's metadata announced (variable sizes, ring wrap-around, several
launches); the blocks the sender writes are byte-identical to the
reference's encode_meta; a block that fails validation (address outside the
sender's registered window) raises instead of being pulled."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1805_08430_b200 import _lib, errors
from paper_1805_08430_b200.memspace import MemorySpace
from paper_1805_08430_b200.runtime.protocol import PipelinedDynamicEdge
from paper_1805_08430_b200.wire import ElemType, encode_meta

pytestmark = pytest.mark.gpu


def _checksum(b: np.ndarray) -> int:
    w = (np.arange(b.size, dtype=np.uint64) % 251 + 1)
    return int((b.astype(np.uint64) * w).sum())


def _r256(n):
    return (n + 255) & ~255


class Rig:
    def __init__(self, max_elems, nsrc, slots, rounds, ring_rounds=3, rank=1):
        two = _lib.device_count() > 1
        self.max_bytes = 4 * max_elems
        self.nsrc, self.slots, self.rounds, self.rank = nsrc, slots, rounds, rank
        self.stride = _r256(self.max_bytes)
        self.meta_stride = PipelinedDynamicEdge.meta_stride(rank)
        self.ring_cap = ring_rounds * _r256(self.max_bytes)
        self.a = MemorySpace(0, nsrc * self.stride + (4 << 20), seed=1, device=0)
        self.b = MemorySpace(1, self.ring_cap + slots * self.meta_stride + 8 * rounds + (4 << 20),
                             seed=2, device=1 if two else 0)
        _lib.call("srf_connect", self.a.handle, self.b.handle)
        self.src = self.a.allocate_region(nsrc * self.stride, register=True)
        self.ring = self.b.allocate_region(self.ring_cap, register=True)
        self.meta = self.b.allocate_region(slots * self.meta_stride, register=True)
        self.sums = self.b.allocate_region(8 * rounds)
        rng = np.random.default_rng(max_elems + slots)
        self.payloads = [rng.integers(0, 256, self.max_bytes, dtype=np.uint8) for _ in range(nsrc)]
        for i, p in enumerate(self.payloads):
            self.a.write_raw(self.src.base_addr + i * self.stride, p)
        self.a.sync(), self.b.sync()
        self.st = {k: C.c_void_p() for k in ("snd", "pull", "cons")}
        for k, sp in (("snd", self.a), ("pull", self.b), ("cons", self.b)):
            _lib.call("srf_stream_create", sp.handle, C.byref(self.st[k]))

    def edge(self, lo=None, hi=None):
        lo = self.src.base_addr if lo is None else lo
        hi = self.src.base_addr + self.src.length if hi is None else hi
        return PipelinedDynamicEdge(self.a, lo, hi, self.src.access_token, self.max_bytes,
                                    self.rank, self.b, self.meta.base_addr, self.meta_stride,
                                    self.slots, self.ring.base_addr, self.ring_cap)

    def send(self, dims, first, rounds):
        PipelinedDynamicEdge.send(self.a, self.b, self.meta.base_addr, self.meta_stride,
                                  self.slots, dims, ElemType.F32, self.src.base_addr,
                                  self.stride, self.nsrc, self.src.access_token, first, rounds,
                                  stream=self.st["snd"])

    def sync(self):
        for s in self.st.values():
            _lib.call("srf_stream_sync", s)
        self.a.sync(), self.b.sync()

    def close(self):
        for s in self.st.values():
            _lib.call("srf_stream_destroy", s)
        self.a.close(), self.b.close()


@pytest.mark.parametrize("max_elems,nsrc,slots,ring_rounds", [
    (1 << 20, 3, 4, 3), (300_001, 2, 8, 2), (1024, 5, 2, 1), ((4 << 20) + 3, 2, 3, 2)])
def test_dynamic_rounds_bit_exact(max_elems, nsrc, slots, ring_rounds):
    R1, R2 = 13, 11
    r = Rig(max_elems, nsrc, slots, R1 + R2, ring_rounds)
    e = r.edge()
    try:
        small = max(1, max_elems // 3 + 7)
        e.consume(0, R1 + R2, checksums_addr=r.sums.base_addr, stream=r.st["cons"])
        r.send((max_elems,), 0, R1)                 # full-size rounds
        r.send((small,), R1, R2)                    # then smaller ones: the ring wraps
        half = (R1 + R2) // 2
        e.recv(half, r.st["pull"])                  # two receiver launches
        e.recv(R1 + R2 - half, r.st["pull"])
        r.sync()
        got = [int(x) for x in np.frombuffer(r.b.read_raw(r.sums.base_addr, 8 * (R1 + R2)),
                                             np.uint64)]
        want = [_checksum(r.payloads[j % nsrc][:4 * (max_elems if j < R1 else small)])
                for j in range(R1 + R2)]
        assert got == want
        # every metadata block: encode_meta of its last round, flag consumed
        for s in range(slots):
            j = max(k for k in range(R1 + R2) if k % slots == s)
            n = max_elems if j < R1 else small
            blk = encode_meta((n,), ElemType.F32, r.src.base_addr + (j % nsrc) * r.stride,
                              r.src.access_token)
            raw = r.b.read_raw(r.meta.base_addr + s * r.meta_stride, len(blk))
            assert raw[:-1] == blk[:-1] and raw[-1] == 0
    finally:
        e.close()
        r.close()


def test_block_outside_the_senders_window_is_rejected():
    """The receiver validates like check_remote_access: the sender announces
    its second payload, the receiver's window covers only the first."""
    r = Rig(4096, 2, 2, 2)
    _lib.tune("put_timeout_ms", 200)
    e = r.edge(hi=r.src.base_addr + r.stride)
    try:
        r.send((4096,), 0, 2)                       # round 1 announces payload 1
        e.recv(2, r.st["pull"])
        _lib.call("srf_stream_sync", r.st["pull"])
        with pytest.raises(errors.RdmaFlowError):
            r.b.sync()
    finally:
        _lib.tune("put_timeout_ms", 5000)
        e.close()
        r.close()


def test_dynamic_edge_rejects_bad_geometry():
    r = Rig(4096, 1, 2, 1)
    try:
        with pytest.raises(errors.InvalidConfig):        # ring smaller than one round
            PipelinedDynamicEdge(r.a, r.src.base_addr, r.src.base_addr + r.src.length,
                                 r.src.access_token, 1 << 30, 1, r.b, r.meta.base_addr,
                                 r.meta_stride, 2, r.ring.base_addr, r.ring_cap)
        with pytest.raises(errors.BadToken):
            PipelinedDynamicEdge(r.a, r.src.base_addr, r.src.base_addr + r.src.length,
                                 r.src.access_token ^ 1, 4 * 4096, 1, r.b, r.meta.base_addr,
                                 r.meta_stride, 2, r.ring.base_addr, r.ring_cap)
    finally:
        r.close()
