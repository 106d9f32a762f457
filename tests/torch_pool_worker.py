"""Subprocess body of tests/test_gpu_torch_pool.py: torch's allocator must be
replaced before the process's first CUDA allocation."""
from __future__ import annotations

import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> int:
    from paper_1805_08430_b200 import _lib
    from paper_1805_08430_b200.memspace import MemorySpace
    from paper_1805_08430_b200.torch_pool import TorchPool
    pool = TorchPool(256 << 20, device=0)
    pool.install()
    import torch
    torch.manual_seed(0)
    # ordinary torch work lands in the registered pool
    a = torch.randn(512, 512, device="cuda")
    b = torch.randn(512, 512, device="cuda")
    c = a @ b + 1.0
    ref = (a.cpu() @ b.cpu()) + 1.0
    assert torch.allclose(c.cpu(), ref, rtol=1e-3, atol=1e-3)
    addr, n, tok = pool.locate(c)
    assert n == c.numel() * 4
    # zero-copy one-sided write of the torch tensor into another server's pool
    peer = MemorySpace(1, 8 << 20, device=torch.cuda.device_count() - 1)
    _lib.call("srf_connect", pool.space.handle, peer.handle)
    dst = peer.allocate_region(4 << 20, register=True)
    u = _lib.u64_array
    ev = C.c_void_p()
    torch.cuda.synchronize()
    _lib.call("srf_put", pool.space.handle, u([addr]), u([n]), u([tok]), 1, peer.handle,
              dst.base_addr, dst.access_token, 0, None, C.byref(ev))
    _lib.Event(ev).wait()
    got = peer.read_raw(dst.base_addr, n)
    assert got == c.cpu().numpy().tobytes()
    # the reference endpoints send a torch-produced tensor zero-copy: the
    # static put reads the pool directly, the dynamic edge announces its
    # address and the receiver pulls it; no payload copy is counted
    from paper_1805_08430_b200.analyzer import PlanEntry
    from paper_1805_08430_b200.fabric import Fabric
    from paper_1805_08430_b200.graph import shape_of
    from paper_1805_08430_b200.memspace import ArenaAllocator
    from paper_1805_08430_b200.runtime.protocol import (DynReceiver, DynSender,
                                                        StaticReceiver, StaticSender)
    from paper_1805_08430_b200.wire import ElemType, Mechanism, meta_block_size
    d = (torch.sigmoid(c) * 3).contiguous()
    t = pool.as_tensor(d)
    assert t.nbytes == d.numel() * 4 and t.elem_type is ElemType.F32
    fab = Fabric(seed=0)
    ar_s = ArenaAllocator(pool.space, pool.space.allocate_region(1 << 16, register=True))
    rcv = MemorySpace(2, 16 << 20, device=torch.cuda.device_count() - 1)
    _lib.call("srf_connect", pool.space.handle, rcv.handle)
    ar_r = ArenaAllocator(rcv, rcv.allocate_region(8 << 20, register=True))
    dv_s = fab.create_device(pool.space, qps_per_peer=2)
    dv_r = fab.create_device(rcv, qps_per_peer=2)
    fwd = dv_s.connect(dv_r.endpoint)
    back = dv_r.channels_to(dv_s.endpoint)
    flag = ar_s.alloc(1)
    pool.space.write_at(flag, 0, b"\x01")
    torch.cuda.synchronize()
    e = PlanEntry(0, 0, 1, Mechanism.STATIC, shape_of(*d.shape), ElemType.F32, 2)
    rb = ar_r.alloc(t.nbytes + 1)
    rcv.write_at(rb, t.nbytes, b"\x00")
    e.recv_buffer = rb
    e.remote_addr, e.remote_token, e.remote_len = rb.base_addr, rb.access_token, rb.length
    copied0 = pool.space.counters.payload_bytes_copied
    StaticSender(e, pool.space, ar_s, fwd[1], flag).send(t, stage_copy=False)
    assert StaticReceiver(e, rcv).poll() is not None
    assert rcv.read_at(rb, 0, t.nbytes) == d.cpu().numpy().tobytes()
    de = PlanEntry(1, 0, 1, Mechanism.DYNAMIC, shape_of(*d.shape), ElemType.F32, 2)
    mb = ar_r.alloc(meta_block_size(2))
    rcv.write_at(mb, mb.length - 1, b"\x00")
    de.recv_buffer = mb
    de.remote_addr, de.remote_token, de.remote_len = mb.base_addr, mb.access_token, mb.length
    snd = DynSender(de, pool.space, ar_s, fwd[1])
    dr = DynReceiver(de, rcv, ar_r, back[1])
    snd.send(t, stage_copy=False)
    meta = None
    while meta is None:
        meta = dr.poll()
    assert meta.remote_addr == t.buffer.handle.base_addr   # the pool address itself
    pulled = dr.fetch(meta)
    rcv.sync()
    assert rcv.read_at(pulled.buffer.handle, 0, t.nbytes) == d.cpu().numpy().tobytes()
    assert pool.space.counters.payload_bytes_copied == copied0   # zero-copy both ways
    snd.close()
    rcv.close()
    # churn: allocations are reused after frees, never overlap while live
    live = []
    for i in range(400):
        t = torch.empty((i * 997) % 200_000 + 1, dtype=torch.float32, device="cuda")
        t.fill_(float(i))
        live.append(t)
        if len(live) > 24:
            live.pop(i % len(live))
    spans = sorted((t.data_ptr(), t.data_ptr() + t.numel() * 4, t.numel()) for t in live)
    for (s0, e0, n0), (s1, e1, n1) in zip(spans, spans[1:]):
        assert e0 <= s1, f"overlapping live tensors {s0:#x}+{n0 * 4} / {s1:#x}+{n1 * 4}"
    for t in live:
        pool.locate(t)
    # a GPU without a pool still works (plain memory, not registered)
    if torch.cuda.device_count() > 1:
        other = torch.arange(1000, device="cuda:1", dtype=torch.float32) * 2
        assert float(other.sum()) == 999000.0
        try:
            pool.locate(other)
            return 1
        except Exception:
            pass
    torch.cuda.synchronize()
    st = pool.stats()
    assert 0 < st["in_use"] <= st["peak"] <= st["capacity"]
    del live, t
    # larger than the pool: ordinary device memory, refused as a zero-copy source
    from paper_1805_08430_b200 import errors
    big = torch.ones(1 << 28, dtype=torch.float32, device="cuda")
    assert float(big[-1]) == 1.0
    try:
        pool.locate(big)
        return 1
    except errors.NotRegistered:
        pass
    del big
    print("torch-pool OK", st, flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
