"""One rank of the cross-process pipelined-edge check (launched by
tests/test_gpu_multiprocess.py under torchrun): rank 0 is the sender, rank 1
the receiver of ONE edge, pools IPC-mapped (or VMM fds) like the bench's
configs[1] one-way sweep.

* push (PipelinedStaticEdge): rank 0's k_put_stream stores into rank 1's
  slots through its mapping of rank 1's pool; rank 1 consumes on its GPU.
* pull (PulledStaticEdge): rank 1's k_pull_stream reads rank 0's payloads
  through its mapping of rank 0's pool; rank 0 only posts rounds (one store
  into rank 1's pool) and, for a rewritten source, waits for its pulled count.
* dyn (PipelinedDynamicEdge): rank 0 writes encode_meta blocks into rank 1's
  metadata slots; rank 1 validates each, allocates from its ring arena and
  pulls the announced payload from rank 0's pool.

Every round's payload, as checksummed by the consumer when it acquires the
slot's flag, must equal what the sender had in that round's source.

SRFLOW_MP_ONE_GPU=1: both ranks on GPU 0.  Kernels of two processes on one
device do not run side by side (no MPS), so the sender's work is complete
before the receiver's starts (push: at most `slots` rounds, no credit
waits; pull: every round posted up front) - the mapping, the system-scope
flags and the posted word still cross processes.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_08430_b200 import _lib  # noqa: E402
from paper_1805_08430_b200.distributed import (all_gather_objects, exchange_spaces,  # noqa: E402
                                               init_process_group)
from paper_1805_08430_b200.memspace import MemorySpace  # noqa: E402
from paper_1805_08430_b200.runtime.protocol import (PipelinedDynamicEdge,  # noqa: E402
                                                    PipelinedStaticEdge, PulledStaticEdge)
from paper_1805_08430_b200.wire import ElemType  # noqa: E402


def checksum(b: np.ndarray) -> int:
    w = (np.arange(b.size, dtype=np.uint64) % 251 + 1)
    return int((b.astype(np.uint64) * w).sum())


def r256(n):
    return (n + 255) & ~255


def main() -> int:
    one_gpu = os.environ.get("SRFLOW_MP_ONE_GPU") == "1"
    rank, world, local = init_process_group("gloo" if one_gpu else "nccl")
    dev = 0 if one_gpu else local
    torch.cuda.set_device(dev)
    barrier = torch.distributed.barrier
    S, nsrc, slots = (3 << 20) + 5, 3, 4
    rounds = slots if one_gpu else 23
    src_stride, slot_stride = r256(S), r256(S + 1)
    rng = np.random.default_rng(11)
    payloads = [rng.integers(0, 256, S, dtype=np.uint8) for _ in range(nsrc)]
    meta_stride = PipelinedDynamicEdge.meta_stride(1)
    ring_cap = 3 * r256(S)
    size = (nsrc * src_stride if rank == 0 else
            slots * slot_stride + 8 * rounds + ring_cap + slots * meta_stride + 4096)
    sp = MemorySpace(rank, size + (4 << 20), seed=rank, device=dev)
    coords = {}
    if rank == 0:
        src = sp.allocate_region(nsrc * src_stride, register=True)
        for i, p in enumerate(payloads):
            sp.write_raw(src.base_addr + i * src_stride, p)
        coords = {"addr": src.base_addr, "token": src.access_token}
    else:
        ring = sp.allocate_region(ring_cap, register=True)   # first: 256-B aligned
        dst = sp.allocate_region(slots * slot_stride, register=True)
        posted = sp.allocate_region(8)
        sums = sp.allocate_region(8 * rounds)
        meta = sp.allocate_region(slots * meta_stride, register=True)
        coords = {"addr": dst.base_addr, "token": dst.access_token, "posted": posted.base_addr,
                  "meta": meta.base_addr}
    sp.sync()
    peer = all_gather_objects(coords)[1 - rank]
    proxies = exchange_spaces(sp, peers=[1 - rank])
    st = [C.c_void_p(), C.c_void_p()]
    for h in st:
        _lib.call("srf_stream_create", sp.handle, C.byref(h))
    # the dynamic edge announces S // 4 float32 elements: the payload's first
    # 4 * (S // 4) bytes
    n_dyn = 4 * (S // 4)
    ok = True
    for mode in ("push", "pull", "dyn"):
        want = [checksum(payloads[j % nsrc][:n_dyn if mode == "dyn" else S])
                for j in range(rounds)]
        if rank == 1:
            for i in range(slots):
                sp.write_raw(dst.base_addr + i * slot_stride + S, b"\x00")
            sp.write_raw(sums.base_addr, b"\x00" * 8 * rounds)
            sp.sync()
        barrier()
        edge = None
        if mode == "push" and rank == 0:
            edge = PipelinedStaticEdge(sp, src, S, nsrc, src_stride, proxies[1], peer["addr"],
                                       peer["token"], slots, slot_stride)
        if mode == "pull" and rank == 1:
            edge = PulledStaticEdge(proxies[0], peer["addr"], peer["token"], S, nsrc, src_stride,
                                    sp, dst, slots, slot_stride, posted.base_addr)
        if mode == "dyn" and rank == 1:
            edge = PipelinedDynamicEdge(proxies[0], peer["addr"], peer["addr"] + nsrc * src_stride,
                                        peer["token"], S, 1, sp, meta.base_addr, meta_stride,
                                        slots, ring.base_addr, ring_cap)
        barrier()
        consume = lambda: PipelinedStaticEdge.consume(  # noqa: E731
            sp, dst.base_addr, slots, slot_stride, S, 0, rounds,
            checksums_addr=sums.base_addr, stream=st[1])
        if mode == "push":
            if rank == 1 and not one_gpu:
                consume()
            barrier()
            if rank == 0:
                edge.send(rounds, st[0])
                _lib.call("srf_stream_sync", st[0])
            barrier()
            if rank == 1 and one_gpu:
                consume()
        elif mode == "pull":
            if rank == 0:
                PulledStaticEdge.post(sp, proxies[1], peer["posted"], rounds, stream=st[0])
                _lib.call("srf_stream_sync", st[0])
            barrier()
            if rank == 1:
                consume()
                edge.recv(rounds, st[0])
        else:
            if rank == 1 and not one_gpu:
                edge.consume(0, rounds, checksums_addr=sums.base_addr, stream=st[1])
            barrier()
            if rank == 0:
                PipelinedDynamicEdge.send(sp, proxies[1], peer["meta"], meta_stride, slots,
                                          (S // 4,), ElemType.F32, src.base_addr, src_stride,
                                          nsrc, src.access_token, 0, rounds, stream=st[0])
                if one_gpu:   # the sender finishes before the receiver starts
                    _lib.call("srf_stream_sync", st[0])
            barrier()
            if rank == 1:
                if one_gpu:
                    edge.consume(0, rounds, checksums_addr=sums.base_addr, stream=st[1])
                edge.recv(rounds, st[0])
        for h in st:
            _lib.call("srf_stream_sync", h)
        sp.sync()
        if rank == 1:
            got = [int(x) for x in np.frombuffer(sp.read_raw(sums.base_addr, 8 * rounds),
                                                 np.uint64)]
            if got != want:
                print(f"rank 1: {mode} checksums differ", flush=True)
                ok = False
            for j in range(max(0, rounds - slots), rounds) if mode != "dyn" else ():
                raw = sp.read_raw(dst.base_addr + (j % slots) * slot_stride, S + 1)
                if raw[:S] != payloads[j % nsrc].tobytes() or raw[S] != 0:
                    print(f"rank 1: {mode} slot of round {j} differs", flush=True)
                    ok = False
        barrier()
        if edge is not None:
            edge.close()
        barrier()
    for h in st:
        _lib.call("srf_stream_destroy", h)
    for p in proxies.values():
        p.close()
    barrier()
    sp.close()
    print(f"rank {rank}: {'OK' if ok else 'FAILED'}", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
