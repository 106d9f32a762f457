"""EXTENSION: the pipelined static edge (srf_edge_*, device_stream.cuh) -
many rounds of one static edge in one persistent launch over `slots`
pre-placed receive regions.  Every round's payload, as observed by the
device consumer when it acquires the slot's flag (weighted byte checksum),
equals the payload that round sent; the final slot contents are bit-exact;
on two GPUs the rounds cross NVLink."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1805_08430_b200 import _lib, errors
from paper_1805_08430_b200.memspace import MemorySpace
from paper_1805_08430_b200.runtime.protocol import PipelinedStaticEdge

pytestmark = pytest.mark.gpu


def _checksum(b: np.ndarray) -> int:
    w = (np.arange(b.size, dtype=np.uint64) % 251 + 1)
    return int((b.astype(np.uint64) * w).sum())


def _r256(n):
    return (n + 255) & ~255


@pytest.mark.parametrize("nbytes,slots,nsrc,rounds", [
    (1, 1, 1, 9), (4097, 2, 3, 17), ((1 << 20) + 3, 4, 5, 23), (4 << 20, 3, 2, 12),
    (300_000, 8, 8, 40)])
@pytest.mark.parametrize("sys_path", [0, 1])
@pytest.mark.parametrize("mirror", [False, True])
def test_rounds_delivered_in_order_bit_exact(nbytes, slots, nsrc, rounds, sys_path, mirror):
    two = _lib.device_count() > 1
    if sys_path and two:
        pytest.skip("two GPUs: the peer path is taken anyway")
    src_stride, slot_stride = _r256(nbytes), _r256(nbytes + 1)
    a = MemorySpace(0, nsrc * src_stride + (4 << 20), seed=1, device=0)
    b = MemorySpace(1, slots * slot_stride + 8 * rounds + (4 << 20), seed=2,
                    device=1 if two else 0)
    _lib.call("srf_connect", a.handle, b.handle)
    ra = a.allocate_region(nsrc * src_stride, register=True)
    credit = a.allocate_region(4 * slots) if mirror else None
    if mirror:
        a.write_raw(credit.base_addr, b"\x00" * 4 * slots)
    rb = b.allocate_region(slots * slot_stride, register=True)
    sums = b.allocate_region(8 * rounds)
    rng = np.random.default_rng(nbytes + slots)
    payloads = [rng.integers(0, 256, nbytes, dtype=np.uint8) for _ in range(nsrc)]
    for i, p in enumerate(payloads):
        a.write_raw(ra.base_addr + i * src_stride, p)
    for i in range(slots):
        b.write_raw(rb.base_addr + i * slot_stride + nbytes, b"\x00")
    a.sync(), b.sync()
    _lib.tune("force_sys", sys_path)
    st_a, st_b = C.c_void_p(), C.c_void_p()
    _lib.call("srf_stream_create", a.handle, C.byref(st_a))
    _lib.call("srf_stream_create", b.handle, C.byref(st_b))
    edge = PipelinedStaticEdge(a, ra, nbytes, nsrc, src_stride, b, rb.base_addr,
                               rb.access_token, slots, slot_stride,
                               credit_addr=credit.base_addr if mirror else None)
    try:
        half = rounds // 2
        # the consumer (one CTA) first, so it is resident beside the sender grid
        PipelinedStaticEdge.consume(b, rb.base_addr, slots, slot_stride, nbytes, 0, rounds,
                                    checksums_addr=sums.base_addr,
                                    credit=(a, credit.base_addr) if mirror else None,
                                    stream=st_b)
        edge.send(half, st_a)            # two launches: round numbering continues
        edge.send(rounds - half, st_a)
        _lib.call("srf_stream_sync", st_a)
        _lib.call("srf_stream_sync", st_b)
        a.sync(), b.sync()
        got = np.frombuffer(b.read_raw(sums.base_addr, 8 * rounds), np.uint64)
        want = [_checksum(payloads[j % nsrc]) for j in range(rounds)]
        assert [int(x) for x in got] == want
        for j in range(max(0, rounds - slots), rounds):
            s = j % slots
            raw = b.read_raw(rb.base_addr + s * slot_stride, nbytes + 1)
            assert raw[:nbytes] == payloads[j % nsrc].tobytes()
            assert raw[nbytes] == 0          # consumed
        assert edge.info()["next_round"] == rounds
    finally:
        edge.close()
        _lib.tune("force_sys", 0)
        _lib.call("srf_stream_destroy", st_a)
        _lib.call("srf_stream_destroy", st_b)
        a.close(), b.close()


def test_edge_rejects_bad_token_and_bounds():
    a = MemorySpace(0, 8 << 20, seed=1, device=0)
    b = MemorySpace(1, 8 << 20, seed=2, device=0)
    ra = a.allocate_region(1 << 20, register=True)
    rb = b.allocate_region(1 << 20, register=True)
    with pytest.raises(errors.BadToken):
        PipelinedStaticEdge(a, ra, 4096, 1, 4096, b, rb.base_addr, rb.access_token ^ 1, 2, 4352)
    with pytest.raises(errors.RemoteOutOfBounds):
        PipelinedStaticEdge(a, ra, 4096, 1, 4096, b, rb.base_addr, rb.access_token, 300, 4352)
    with pytest.raises(errors.InvalidConfig):
        PipelinedStaticEdge(a, ra, 4096, 1, 4096, b, rb.base_addr, rb.access_token, 2, 4096)
    with pytest.raises(errors.OutOfBounds):
        PipelinedStaticEdge(a, ra, 4096, 1, 4096, b, rb.base_addr, rb.access_token, 2, 4352,
                            credit_addr=(8 << 20) - 4)
    a.close(), b.close()
