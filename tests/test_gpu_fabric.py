"""Verbs layer on the GPU path: the reference's fabric contracts
(reference tests/test_fabric.py) except the chunk-schedule cases, which
describe the simulator's ascending delivery (replaced by the K1 flag-last
stress test in test_gpu_kernels.py)."""
from __future__ import annotations

import threading

import pytest

from paper_1805_08430_b200 import _lib, errors
from paper_1805_08430_b200.fabric import CostModel, Fabric, FaultConfig, MemRange
from paper_1805_08430_b200.memspace import MemorySpace

pytestmark = pytest.mark.gpu


def pair(num_cqs=1, qps=1, faults=None, capacity=1 << 20):
    fab = Fabric(seed=5, faults=faults)
    sp = [MemorySpace(i, capacity, seed=i) for i in range(2)]
    a = fab.create_device(sp[0], num_cqs=num_cqs, qps_per_peer=qps)
    b = fab.create_device(sp[1], num_cqs=num_cqs, qps_per_peer=qps)
    return fab, sp, a, b, a.connect(b.endpoint)


def test_cq_round_robin_within_and_across_peers():
    _, _, _, _, chans = pair(num_cqs=2, qps=4)
    assert [c.qp.cq_index for c in chans] == [0, 1, 0, 1]
    fab = Fabric()
    sp = [MemorySpace(i, 4096) for i in range(3)]
    d = [fab.create_device(s, num_cqs=3, qps_per_peer=2) for s in sp]
    assert [c.qp.cq_index for c in d[0].connect(d[1].endpoint)] == [0, 1]
    assert [c.qp.cq_index for c in d[0].connect(d[2].endpoint)] == [2, 0]


def test_connect_errors_and_pairing():
    fab = Fabric()
    a = fab.create_device(MemorySpace(0, 4096))
    with pytest.raises(errors.PeerUnreachable):
        a.connect((99, 1))
    b = fab.create_device(MemorySpace(1, 4096), listening=False)
    with pytest.raises(errors.PeerUnreachable):
        a.connect(b.endpoint)
    _, _, a, b, chans = pair(qps=2)
    back = b.channels_to(a.endpoint)
    assert len(back) == 2
    for mine, theirs in zip(chans, back):
        assert mine.qp.peer_qp is theirs.qp and theirs.qp.peer_qp is mine.qp


def test_one_byte_write_one_completion():
    fab, sp, a, b, chans = pair()
    src = sp[0].allocate_region(1, register=True)
    dst = sp[1].allocate_region(1, register=True)
    sp[0].write_at(src, 0, b"\xab")
    before = _lib.launch_count()
    verb = chans[0].one_sided_write(src, dst.base_addr, dst.access_token, tag="t")
    assert _lib.launch_count() == before + 1
    ev = a.poll_cq(0)
    assert ev.verb_id == verb and ev.tag == "t" and ev.nbytes == 1
    assert a.poll_cq(0) is None
    ev.wait()
    assert sp[1].read_at(dst, 0, 1) == b"\xab"


def test_access_errors_do_not_mutate():
    fab, sp, a, b, chans = pair()
    src = sp[0].allocate_region(16, register=True)
    dst = sp[1].allocate_region(16, register=True)
    small = sp[1].allocate_region(8, register=True)
    plain = sp[0].allocate_region(16, register=False)
    sp[0].write_at(src, 0, b"x" * 16)
    with pytest.raises(errors.BadToken):
        chans[0].one_sided_write(src, dst.base_addr, dst.access_token ^ 5)
    assert sp[1].read_at(dst, 0, 16) == bytes(16)
    with pytest.raises(errors.RemoteOutOfBounds):
        chans[0].one_sided_write(src, small.base_addr, small.access_token)
    with pytest.raises(errors.NotRegistered):
        chans[0].one_sided_write(plain, dst.base_addr, dst.access_token)
    with pytest.raises(errors.InvalidLength):
        chans[0].one_sided_write(MemRange(src, 0, 0), dst.base_addr, dst.access_token)
    with pytest.raises(errors.InvalidLength):
        chans[0].one_sided_read(0, 0, MemRange(src, 0, 0))
    assert fab.verbs_posted == 0


def test_gather_list_concatenates():
    fab, sp, a, b, chans = pair()
    s1 = sp[0].allocate_region(8, register=True)
    s2 = sp[0].allocate_region(8, register=True)
    dst = sp[1].allocate_region(16, register=True)
    sp[0].write_at(s1, 0, b"AAAAAAAA")
    sp[0].write_at(s2, 0, b"BBBBBBBB")
    chans[0].take_completion(chans[0].one_sided_write([s1, s2], dst.base_addr,
                                                       dst.access_token))
    assert sp[1].read_at(dst, 0, 16) == b"AAAAAAAA" + b"BBBBBBBB"


def test_cost_model_clock():
    cost = CostModel()
    fab = Fabric(cost)
    sp = [MemorySpace(i, 1 << 20) for i in range(2)]
    a, b = fab.create_device(sp[0]), fab.create_device(sp[1])
    ch = a.connect(b.endpoint)[0]
    src = sp[0].allocate_region(4096, register=True)
    dst = sp[1].allocate_region(4096, register=True)
    stamps = [fab.clock.now()]
    for _ in range(5):
        ch.take_completion(ch.one_sided_write(src, dst.base_addr, dst.access_token))
        stamps.append(fab.clock.now())
    assert all(x < y for x, y in zip(stamps, stamps[1:]))
    assert stamps[1] - stamps[0] == pytest.approx(cost.alpha_s + cost.beta_s_per_byte * 4096,
                                                  rel=1e-12)


def test_read_roundtrip_and_completion_goes_to_reader():
    fab, sp, a, b, chans = pair()
    src = sp[0].allocate_region(64, register=True)
    remote = sp[1].allocate_region(64, register=True)
    local = sp[0].allocate_region(64, register=True)
    sp[0].write_at(src, 0, bytes(range(64)))
    chans[0].take_completion(chans[0].one_sided_write(src, remote.base_addr,
                                                       remote.access_token))
    verb = chans[0].one_sided_read(remote.base_addr, remote.access_token, MemRange(local),
                                   tag="r")
    ev = a.poll_cq(0)
    assert ev.verb_id == verb and ev.kind == "read" and b.poll_cq(0) is None
    ev.wait()
    assert sp[0].read_at(local, 0, 64) == bytes(range(64))


def test_concurrent_reads_on_two_qps():
    for trial in range(4):
        fab, sp, a, b, chans = pair(qps=2)
        remote = sp[1].allocate_region(1 << 16, register=True)
        sp[1].write_at(remote, 0, bytes(i % 251 for i in range(1 << 16)))
        locs = [sp[0].allocate_region(1 << 16, register=True) for _ in range(2)]
        verbs = [None, None]

        def go(i):
            verbs[i] = chans[i].one_sided_read(remote.base_addr, remote.access_token,
                                               MemRange(locs[i]))

        ts = [threading.Thread(target=go, args=(i,)) for i in ((0, 1) if trial % 2 else (1, 0))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        evs = [chans[i].take_completion(verbs[i]) for i in range(2)]
        assert evs[0].qp_id != evs[1].qp_id
        for lh in locs:
            assert sp[0].read_at(lh, 0, 1 << 16) == bytes(i % 251 for i in range(1 << 16))


def test_take_completion_routes_other_qps_to_their_stash():
    fab, sp, a, b, chans = pair(num_cqs=1, qps=2)
    src = sp[0].allocate_region(8, register=True)
    dst = sp[1].allocate_region(8, register=True)
    v0 = chans[0].one_sided_write(src, dst.base_addr, dst.access_token)
    v1 = chans[1].one_sided_write(src, dst.base_addr, dst.access_token)
    assert chans[1].take_completion(v1).verb_id == v1   # v0 stashed on qp 0
    assert chans[0].take_completion(v0).verb_id == v0
    with pytest.raises(errors.Timeout):
        chans[0].take_completion(12345)


def test_send_recv_messaging():
    fab, sp, a, b, chans = pair(capacity=1 << 22)
    buf = sp[1].allocate_region(16, register=True)
    back = b.channels_to(a.endpoint)[0]
    back.post_recv(MemRange(buf), tag="rx")
    assert chans[0].post_send(b"0123456789abcdef", tag="tx") is not None
    s_ev, r_ev = a.poll_cq(0), b.poll_cq(0)
    assert s_ev.kind == "send" and r_ev.kind == "recv" and r_ev.nbytes == 16
    assert sp[1].read_at(buf, 0, 16) == b"0123456789abcdef"
    back.post_recv(MemRange(buf))
    with pytest.raises(errors.RecvBufferTooSmall):
        chans[0].post_send(b"x" * 32)
    assert chans[0].post_send(b"y" * 16) is not None
    with pytest.raises(errors.NoPostedReceive):
        chans[0].post_send(b"hello", timeout=0.05)
    assert chans[0].post_send(b"hello", block=False) is None
    bufs = [sp[1].allocate_region(8, register=True) for _ in range(50)]

    def post():
        for bb in bufs:
            back.post_recv(MemRange(bb))

    def send():
        for i in range(50):
            chans[0].post_send(i.to_bytes(8, "little"))

    ts = [threading.Thread(target=post), threading.Thread(target=send)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i, bb in enumerate(bufs):
        assert int.from_bytes(sp[1].read_at(bb, 0, 8), "little") == i


def test_post_order_and_exactly_once_completions():
    fab, sp, a, b, chans = pair()
    src = sp[0].allocate_region(8, register=True)
    dst = sp[1].allocate_region(8, register=True)
    for i in range(10):
        chans[0].one_sided_write(src, dst.base_addr, dst.access_token, tag=i)
    tags = []
    while (ev := a.poll_cq(0)) is not None:
        tags.append(ev.tag)
        ev.wait()
    assert tags == list(range(10))
    back = b.channels_to(a.endpoint)[0]
    back.post_recv(MemRange(dst))
    chans[0].post_send(b"12345678")
    assert fab.completions_posted == fab.verbs_posted - fab.outstanding_recvs()
    assert fab.outstanding_recvs() == 0


def test_rpc_control_plane():
    faults = FaultConfig(drop_rpc_calls=1)
    fab, sp, a, b, chans = pair(faults=faults)
    with pytest.raises(errors.HandlerMissing):
        chans[0].rpc_call(b"x")
    b.register_rpc_handler(lambda req: req)
    with pytest.raises(errors.Timeout):
        chans[0].rpc_call(b"x")
    assert chans[0].rpc_call(b"\xde\xad") == b"\xde\xad"
