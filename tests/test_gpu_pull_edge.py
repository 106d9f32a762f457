"""EXTENSION: the pull edge (srf_edge_create_pull / srf_edge_recv /
srf_edge_post, device_stream.cuh k_pull_stream) - the pipelined static edge
driven by the receiver's GPU, which pulls each posted round from the
sender's source straight into its pre-placed slot and releases the slot's
flag last.  Same checks as the push edge (tests/test_gpu_edge.py): the
consumer's per-round checksum taken when it acquires the flag equals the
payload that round carried, final slots are bit-exact, round numbering
continues across launches; plus the sender-side protocol (posting, the
pulled-use counts, waiting for a source to be pulled before reposting) and
a round that is never posted timing out without touching the slot."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1805_08430_b200 import _lib, errors
from paper_1805_08430_b200.memspace import MemorySpace
from paper_1805_08430_b200.runtime.protocol import PipelinedStaticEdge, PulledStaticEdge

pytestmark = pytest.mark.gpu


def _checksum(b: np.ndarray) -> int:
    w = (np.arange(b.size, dtype=np.uint64) % 251 + 1)
    return int((b.astype(np.uint64) * w).sum())


def _r256(n):
    return (n + 255) & ~255


class Rig:
    def __init__(self, nbytes, slots, nsrc, rounds, src_stride=None, seed=0):
        two = _lib.device_count() > 1
        self.nbytes, self.slots, self.nsrc, self.rounds = nbytes, slots, nsrc, rounds
        self.src_stride = src_stride or _r256(nbytes)
        self.slot_stride = _r256(nbytes + 1)
        self.a = MemorySpace(0, nsrc * self.src_stride + (4 << 20), seed=1, device=0)
        self.b = MemorySpace(1, slots * self.slot_stride + 8 * rounds + (4 << 20), seed=2,
                             device=1 if two else 0)
        _lib.call("srf_connect", self.a.handle, self.b.handle)
        self.ra = self.a.allocate_region(nsrc * self.src_stride, register=True)
        self.pulled = self.a.allocate_region(4 * nsrc)
        self.a.write_raw(self.pulled.base_addr, b"\x00" * 4 * nsrc)
        self.rb = self.b.allocate_region(slots * self.slot_stride, register=True)
        self.posted = self.b.allocate_region(8)
        self.sums = self.b.allocate_region(8 * rounds)
        rng = np.random.default_rng(nbytes * 7 + slots + seed)
        self.payloads = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(nsrc)]
        for i, p in enumerate(self.payloads):
            self.a.write_raw(self.ra.base_addr + i * self.src_stride, p)
        for i in range(slots):
            self.b.write_raw(self.rb.base_addr + i * self.slot_stride + nbytes, b"\x00")
        self.a.sync(), self.b.sync()
        self.st = {k: C.c_void_p() for k in ("snd", "pull", "cons")}
        for k, sp in (("snd", self.a), ("pull", self.b), ("cons", self.b)):
            _lib.call("srf_stream_create", sp.handle, C.byref(self.st[k]))
        self.edge = None

    def make(self, tma):
        self.edge = PulledStaticEdge(self.a, self.ra.base_addr, self.ra.access_token,
                                     self.nbytes, self.nsrc, self.src_stride, self.b, self.rb,
                                     self.slots, self.slot_stride, self.posted.base_addr,
                                     pulled_addr=self.pulled.base_addr, tma=tma)
        return self.edge

    def consume(self, first, rounds):
        PipelinedStaticEdge.consume(self.b, self.rb.base_addr, self.slots, self.slot_stride,
                                    self.nbytes, first, rounds,
                                    checksums_addr=self.sums.base_addr + 8 * first,
                                    stream=self.st["cons"])

    def post(self, count, wait=None):
        PulledStaticEdge.post(self.a, self.b, self.posted.base_addr, count, wait=wait,
                              stream=self.st["snd"])

    def sync(self):
        for s in self.st.values():
            _lib.call("srf_stream_sync", s)
        self.a.sync(), self.b.sync()

    def check(self, rounds):
        got = np.frombuffer(self.b.read_raw(self.sums.base_addr, 8 * rounds), np.uint64)
        want = [_checksum(self.payloads[j % self.nsrc]) for j in range(rounds)]
        assert [int(x) for x in got] == want
        for j in range(max(0, rounds - self.slots), rounds):
            raw = self.b.read_raw(self.rb.base_addr + (j % self.slots) * self.slot_stride,
                                  self.nbytes + 1)
            assert raw[:self.nbytes] == self.payloads[j % self.nsrc].tobytes()
            assert raw[self.nbytes] == 0

    def close(self):
        if self.edge is not None:
            self.edge.close()
        for s in self.st.values():
            _lib.call("srf_stream_destroy", s)
        self.a.close(), self.b.close()


@pytest.mark.parametrize("nbytes,slots,nsrc,rounds", [
    (1, 1, 1, 9), (4097, 2, 3, 17), ((1 << 20) + 3, 4, 5, 23), (4 << 20, 3, 2, 12),
    (300_000, 8, 8, 40), (16 << 20, 4, 2, 9)])
@pytest.mark.parametrize("tma", [True, False])
def test_pulled_rounds_bit_exact(nbytes, slots, nsrc, rounds, tma):
    r = Rig(nbytes, slots, nsrc, rounds)
    try:
        e = r.make(tma)
        half = rounds // 2
        r.consume(0, rounds)          # the consumer CTA first (resident beside the pull grid)
        r.post(half)
        e.recv(half, r.st["pull"])
        r.post(rounds)
        e.recv(rounds - half, r.st["pull"])   # round numbering continues
        r.sync()
        r.check(rounds)
        assert e.info()["next_round"] == rounds
        # every source's pulled-use count reached its number of uses
        pulled = np.frombuffer(r.a.read_raw(r.pulled.base_addr, 4 * nsrc), np.uint32)
        assert [int(x) for x in pulled] == [len(range(i, rounds, nsrc)) for i in range(nsrc)]
    finally:
        r.close()


@pytest.mark.parametrize("tma", [True, False])
def test_unaligned_source_stride_takes_the_load_path(tma):
    """A source stride that breaks 16-B alignment still delivers bit-exact
    (the TMA request falls back to coherent SM loads)."""
    r = Rig(100_003, 3, 3, 11, src_stride=100_003 + 8)
    try:
        e = r.make(tma)
        r.consume(0, 11)
        r.post(11)
        e.recv(11, r.st["pull"])
        r.sync()
        r.check(11)
    finally:
        r.close()


def test_sender_reuses_a_source_only_after_it_was_pulled():
    """One source, rewritten before every round: the sender's post of round
    j waits until round j-1 was fully pulled (pulled count >= j); every
    round's checksum is that round's own payload."""
    nbytes, rounds = (2 << 20) + 5, 6
    r = Rig(nbytes, 2, 1, rounds)
    try:
        e = r.make(True)
        rng = np.random.default_rng(5)
        pays = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(rounds)]
        r.consume(0, rounds)
        for j in range(rounds):
            # a host rewrite of the source must wait for the device licence
            if j:
                r.post(j, wait=(r.pulled.base_addr, j))
                _lib.call("srf_stream_sync", r.st["snd"])
                r.a.sync()
            r.a.write_raw(r.ra.base_addr, pays[j])
            r.a.sync()
            r.post(j + 1)
            e.recv(1, r.st["pull"])
        r.sync()
        got = np.frombuffer(r.b.read_raw(r.sums.base_addr, 8 * rounds), np.uint64)
        assert [int(x) for x in got] == [_checksum(p) for p in pays]
    finally:
        r.close()


def test_unposted_round_times_out_and_leaves_the_slot_untouched():
    nbytes = (1 << 20) + 16
    r = Rig(nbytes, 2, 1, 2)
    _lib.tune("put_timeout_ms", 50)
    try:
        e = r.make(True)
        before = r.b.read_raw(r.rb.base_addr, nbytes + 1)
        e.recv(1, r.st["pull"])          # nothing posted
        _lib.call("srf_stream_sync", r.st["pull"])
        with pytest.raises(errors.Timeout):
            r.b.sync()
        assert r.b.read_raw(r.rb.base_addr, nbytes + 1) == before
    finally:
        _lib.tune("put_timeout_ms", 5000)
        r.close()


def test_pull_edge_rejects_bad_token_bounds_and_misuse():
    a = MemorySpace(0, 8 << 20, seed=1, device=0)
    b = MemorySpace(1, 8 << 20, seed=2, device=0)
    ra = a.allocate_region(1 << 20, register=True)
    rb = b.allocate_region(1 << 20, register=True)
    posted = b.allocate_region(8)
    try:
        with pytest.raises(errors.BadToken):
            PulledStaticEdge(a, ra.base_addr, ra.access_token ^ 1, 4096, 1, 4096, b, rb, 2, 4352,
                             posted.base_addr)
        with pytest.raises(errors.RemoteOutOfBounds):
            PulledStaticEdge(a, ra.base_addr, ra.access_token, 4096, 300, 4096, b, rb, 2, 4352,
                             posted.base_addr)
        with pytest.raises(errors.InvalidConfig):
            PulledStaticEdge(a, ra.base_addr, ra.access_token, 4096, 1, 4096, b, rb, 2, 4096,
                             posted.base_addr)
        with pytest.raises(errors.InvalidConfig):   # posted word misaligned
            PulledStaticEdge(a, ra.base_addr, ra.access_token, 4096, 1, 4096, b, rb, 2, 4352,
                             posted.base_addr + 4)
        e = PulledStaticEdge(a, ra.base_addr, ra.access_token, 4096, 1, 4096, b, rb, 2, 4352,
                             posted.base_addr)
        with pytest.raises(errors.InvalidConfig):   # a pull edge is driven by the receiver
            _lib.call("srf_edge_send", e._h, 1, None, a.handle)
        e.close()
    finally:
        a.close(), b.close()
