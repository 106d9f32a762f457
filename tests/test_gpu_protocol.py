"""Send/Recv endpoints on the GPU path vs the reference's own vectors and
semantics (reference tests/test_protocol.py, minus the simulated chunk-prefix
case that has no GPU meaning - replaced by the release/acquire stress test in
test_gpu_kernels.py)."""
from __future__ import annotations

import pytest

from paper_1805_08430_b200 import _lib, errors
from paper_1805_08430_b200.analyzer import AllocSite, TraceState
from paper_1805_08430_b200.runtime.protocol import (FRAG_PAYLOAD_BYTES, DynReceiver,
                                                    DynSender, RpcReceiver, RpcSender,
                                                    StaticReceiver, StaticSender,
                                                    ZeroCopyViolation)
from paper_1805_08430_b200.wire import ElemType, Mechanism, meta_block_size

from gpu_rig import Rig

pytestmark = pytest.mark.gpu


def static_pair(rig, dims):
    entry = rig.entry(dims, Mechanism.STATIC)
    return (entry, StaticSender(entry, rig.spaces[0], rig.arenas[0], rig.fwd[1], rig.flags[0]),
            StaticReceiver(entry, rig.spaces[1]))


def dyn_pair(rig, dims):
    entry = rig.entry(dims, Mechanism.DYNAMIC)
    return (entry, DynSender(entry, rig.spaces[0], rig.arenas[0], rig.fwd[1]),
            DynReceiver(entry, rig.spaces[1], rig.arenas[1], rig.back[1]))


class TestStatic:
    def test_reference_vectors(self, golden):
        doc, arr = golden
        for r in [x for x in doc["rig"] if x["mech"] == "static"]:
            rig = Rig()
            launches = _lib.launch_count()
            entry, snd, rcv = static_pair(rig, r["dims"])
            t = rig.tensor(r["dims"])
            buf = entry.recv_buffer
            assert (buf.base_addr, buf.access_token, buf.length) == \
                (r["recv_addr"], r["recv_token"], r["recv_len"])
            assert t.buffer.handle.base_addr == r["payload_addr"]
            assert rcv.poll() is None
            snd.send(t, stage_copy=False)
            assert _lib.launch_count() == launches + 1  # one K1 launch per send
            region = rig.spaces[1].read_at(buf, 0, buf.length)
            assert region == arr[r["key"] + "/after_send"].tobytes()
            got = rcv.poll()
            assert got is not None and got.nbytes == r["got_nbytes"]
            assert rig.spaces[1].read_at(buf, 0, buf.length) == \
                arr[r["key"] + "/after_poll"].tobytes()
            assert rcv.poll() is None
            assert rig.fabric.wire_bytes == r["wire_bytes"]
            rig.close()

    def test_roundtrip_view_is_zero_copy(self):
        rig = Rig()
        entry, snd, rcv = static_pair(rig, (64, 64))
        t = rig.tensor((64, 64))
        snd.send(t, stage_copy=False)
        got = rcv.poll()
        assert got.buffer.handle.base_addr == entry.recv_buffer.base_addr
        dev = got.array(rig.spaces[1])
        assert dev.device.index == rig.spaces[1].device
        assert dev.cpu().numpy().tobytes() == rig.spaces[0].read_at(t.buffer.handle, 0, t.nbytes)

    @pytest.mark.parametrize("ce_kib", [0, 1])
    def test_large_send_through_doorbell_both_engines(self, ce_kib):
        """A 2 MiB static send between two GPUs with the body moved by SM
        stores or by the copy engine: the receiver's host doorbell sees the
        flag only with the whole body in place, three sends in a row."""
        _lib.tune("peer_ce_kib", ce_kib)
        try:
            rig = Rig(capacity=1 << 25)
            entry, snd, rcv = static_pair(rig, (1024, 512))
            for k in range(3):
                t = rig.tensor((1024, 512), seed=100 + k)
                snd.send(t, stage_copy=False)
                got = None
                while got is None:
                    got = rcv.poll()
                assert rig.spaces[1].read_at(entry.recv_buffer, 0, t.nbytes) == \
                    rig.spaces[0].read_at(t.buffer.handle, 0, t.nbytes)
                t.buffer.release()
            rig.close()
        finally:
            _lib.tune("peer_ce_kib", 0)

    def test_size_mismatch(self):
        rig = Rig()
        _, snd, _ = static_pair(rig, (3, 4))
        with pytest.raises(errors.SizeMismatch):
            snd.send(rig.tensor((3, 5)), stage_copy=False)

    def test_copy_accounting(self):
        rig = Rig()
        _, snd, rcv = static_pair(rig, (4, 4))
        t = rig.tensor((4, 4))
        snd.send(t, stage_copy=False)
        assert rig.spaces[0].counters.payload_bytes_copied == 0
        rcv.poll()
        snd.send(t, stage_copy=True)
        assert rig.spaces[0].counters.payload_bytes_copied == 64
        assert rig.spaces[0].counters.payload_copy_events == 1
        got = rcv.poll()
        assert rig.spaces[1].read_at(got.buffer.handle, 0, 64) == \
            rig.spaces[0].read_at(t.buffer.handle, 0, 64)

    def test_zero_copy_violation(self):
        rig = Rig()
        _, snd, _ = static_pair(rig, (2, 2))
        with pytest.raises(ZeroCopyViolation):
            snd.send(rig.tensor((2, 2), arena=False), stage_copy=False)

    def test_barrier_violation(self):
        rig = Rig()
        _, snd, _ = static_pair(rig, (2,))
        t = rig.tensor((2,))
        snd.send(t, stage_copy=False)
        with pytest.raises(errors.ProtocolError):
            snd.send(t, stage_copy=False)

    def test_empty_tensor_is_flag_only(self):
        rig = Rig()
        _, snd, rcv = static_pair(rig, (0, 4))
        snd.send(rig.tensor((0, 4)), stage_copy=False)
        got = rcv.poll()
        assert got is not None and got.nbytes == 0

    def test_trace_records_site(self):
        rig = Rig()
        _, snd, _ = static_pair(rig, (2, 2))
        t = rig.tensor((2, 2))
        trace = TraceState()
        trace.record_alloc(t.buffer.handle.base_addr, AllocSite(3, 0))
        snd.send(t, stage_copy=True, trace=trace)
        assert trace.transfer_sites == {AllocSite(3, 0)}

    def test_remote_checks(self):
        rig = Rig()
        entry, _, _ = static_pair(rig, (8,))
        src = rig.tensor((8,))
        ch = rig.fwd[1]
        with pytest.raises(errors.BadToken):
            ch.one_sided_write(src.buffer.handle, entry.remote_addr, entry.remote_token ^ 1)
        with pytest.raises(errors.RemoteOutOfBounds):
            ch.one_sided_write(src.buffer.handle, (1 << 22) - 4, entry.remote_token)
        unreg = rig.spaces[0].allocate_region(64)
        with pytest.raises(errors.NotRegistered):
            ch.one_sided_write(unreg, entry.remote_addr, entry.remote_token)
        with pytest.raises(errors.InvalidLength):
            ch.one_sided_write([], entry.remote_addr, entry.remote_token)


class TestDynamic:
    def test_reference_vectors(self, golden):
        doc, arr = golden
        for r in [x for x in doc["rig"] if x["mech"] == "dynamic"]:
            rig = Rig()
            entry, snd, rcv = dyn_pair(rig, r["dims"])
            t = rig.tensor(r["dims"])
            assert entry.recv_buffer.base_addr == r["recv_addr"]
            assert t.buffer.handle.base_addr == r["payload_addr"]
            assert rcv.poll() is None
            snd.send(t, stage_copy=False)
            buf = entry.recv_buffer
            # byte-identical metadata block (addresses and token included)
            assert rig.spaces[1].read_at(buf, 0, buf.length) == arr[r["key"] + "/meta"].tobytes()
            meta = rcv.poll()
            assert meta.dims == tuple(r["dims"])
            got = rcv.fetch(meta)
            pulled = rig.spaces[1].read_at(got.buffer.handle, 0, got.nbytes) if got.nbytes else b""
            assert pulled == arr[r["key"] + "/sent"].tobytes()
            if got.nbytes:
                assert got.buffer.handle.base_addr == r["pulled_addr"]
            assert rig.spaces[0].counters.serialize_bytes == r["serialize_bytes"]
            assert rig.fabric.verbs_posted == r["verbs"]
            assert rig.fabric.wire_bytes == r["wire_bytes"]

    def test_shape_change_reuses_meta_block(self):
        rig = Rig()
        entry, snd, rcv = dyn_pair(rig, (5, 8))
        snd.send(rig.tensor((5, 8)), stage_copy=False)
        rcv.fetch(rcv.poll())
        snd.send(rig.tensor((7, 8)), stage_copy=False)
        meta = rcv.poll()
        assert meta.dims == (7, 8)
        assert entry.recv_buffer.base_addr == entry.remote_addr

    def test_rank_change_rejected(self):
        rig = Rig()
        _, snd, _ = dyn_pair(rig, (5, 8))
        with pytest.raises(errors.RankChanged):
            snd.send(rig.tensor((5, 8, 1)), stage_copy=False)

    def test_empty_payload_skips_read(self):
        rig = Rig()
        _, snd, rcv = dyn_pair(rig, (0, 8))
        before = rig.fabric.verbs_posted
        snd.send(rig.tensor((0, 8)), stage_copy=False)
        got = rcv.fetch(rcv.poll())
        assert got.nbytes == 0 and rig.fabric.verbs_posted == before + 1

    def test_arena_returns_and_sender_retains(self):
        rig = Rig()
        _, snd, rcv = dyn_pair(rig, (16, 16))
        base1 = rig.arenas[1].current_resident
        res0 = rig.arenas[0].current_resident
        t1 = rig.tensor((16, 16))
        snd.send(t1, stage_copy=False)
        got = rcv.fetch(rcv.poll())
        assert rig.arenas[1].current_resident == base1 + got.nbytes
        got.buffer.release()
        assert rig.arenas[1].current_resident == base1
        t1.buffer.release()
        assert rig.arenas[0].current_resident == res0 + 1024  # still held by the sender
        snd.close()
        assert rig.arenas[0].current_resident == res0

    def test_staged_send_copies_once(self):
        rig = Rig()
        _, snd, rcv = dyn_pair(rig, (4, 4))
        t = rig.tensor((4, 4), arena=False)
        snd.send(t, stage_copy=True)
        assert rig.spaces[0].counters.payload_bytes_copied == 64
        got = rcv.fetch(rcv.poll())
        assert rig.spaces[1].read_at(got.buffer.handle, 0, 64) == \
            rig.spaces[0].read_at(t.buffer.handle, 0, 64)

    def test_meta_serialisation_counted(self):
        rig = Rig()
        _, snd, _ = dyn_pair(rig, (5, 8))
        snd.send(rig.tensor((5, 8)), stage_copy=False)
        assert rig.spaces[0].counters.serialize_bytes == meta_block_size(2) == 49


class TestRpcBaseline:
    def pump(self, snd, rcv, rounds=20_000):
        got = None
        for _ in range(rounds):
            done = snd.pump()
            r = rcv.poll()
            got = r if r is not None else got
            if done and not snd.busy and got is not None:
                return got
        raise AssertionError("transfer did not finish")

    def test_fragments_copies_and_backpressure(self):
        rig = Rig(qps=2)
        snd = RpcSender(0, 1, rig.spaces[0], rig.arenas[0], rig.fwd[1])
        rcv = RpcReceiver(0, 1, rig.spaces[1], rig.arenas[1], rig.arenas[1], rig.back[1])
        nbytes = 20 * FRAG_PAYLOAD_BYTES
        t = rig.tensor((nbytes // 4,))
        snd.start(t)
        assert snd.pump() is False  # ring full before the message ended
        got = self.pump(snd, rcv)
        assert rig.spaces[1].read_at(got.buffer.handle, 0, nbytes) == \
            rig.spaces[0].read_at(t.buffer.handle, 0, nbytes)
        copied = (rig.spaces[0].counters.payload_bytes_copied +
                  rig.spaces[1].counters.payload_bytes_copied)
        assert copied == 2 * nbytes + meta_block_size(1)


class TestRpcDevice:
    @pytest.mark.parametrize("dims", [(0, 7), (1,), (1020,), (2560, 1), (40 * 1020,), (1 << 20,)])
    def test_fragment_ring_on_device(self, dims):
        from paper_1805_08430_b200.runtime.protocol import RpcDeviceLink
        rig = Rig(capacity=1 << 24)
        link = RpcDeviceLink(len(dims), rig.spaces[0], rig.arenas[0], rig.spaces[1],
                             rig.arenas[1], rig.arenas[1])
        t = rig.tensor(dims)
        got = link.transfer(t)
        n = t.nbytes
        if n:
            assert rig.spaces[1].read_at(got.buffer.handle, 0, n) == \
                rig.spaces[0].read_at(t.buffer.handle, 0, n)
        meta = rig.spaces[1].read_at(link.meta_out, 0, meta_block_size(len(dims)))
        from paper_1805_08430_b200.wire import encode_meta
        assert meta == encode_meta(dims, ElemType.F32, 0, 0)
        copied = (rig.spaces[0].counters.payload_bytes_copied +
                  rig.spaces[1].counters.payload_bytes_copied)
        assert copied == 2 * n + meta_block_size(len(dims))
        # every ring slot re-posted
        assert rig.spaces[1].read_at(link.ring_flags, 0, 16) == bytes(16)
        # a second message through the same ring
        got.buffer.release()
        got2 = link.transfer(t)
        if n:
            assert rig.spaces[1].read_at(got2.buffer.handle, 0, n) == \
                rig.spaces[0].read_at(t.buffer.handle, 0, n)
