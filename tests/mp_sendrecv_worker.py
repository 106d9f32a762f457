"""One rank of the cross-process Send/Recv check (launched by
tests/test_gpu_multiprocess.py under torchrun).

Rank r is server r; its pool is exported (CUDA IPC handle, or a VMM fd with
SRFLOW_ALLOC_VMM=1) and mapped by the peer as a proxy space
(MemorySpace.import_remote); receive-buffer coordinates travel as the
reference's 33-byte AddrExchangeMsg (analyzer.py:166-220, wire.py:145-171).
Every rank then sends to the next through the reference endpoints
(runtime/protocol.py:49-254): StaticSender -> its K1 put writes straight into
the peer's pool, StaticReceiver.poll reads the flag from the device (an
exported space has no host doorbell), DynSender writes the metadata block,
DynReceiver.fetch pulls the payload (K4) from the peer's pool.  Payloads are
the reference's synthesize_values streams; the received bytes must equal them.

SRFLOW_MP_ONE_GPU=1: both ranks on GPU 0 with a gloo control plane (CUDA IPC
between two processes of one device), so a one-GPU box covers the
cross-process code: IPC/VMM export and import, proxy spaces, system-scope
release/acquire on imported pools and the doorbell's device-read fallback.
"""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_08430_b200.analyzer import PlanEntry  # noqa: E402
from paper_1805_08430_b200.distributed import (exchange_spaces, init_process_group,  # noqa: E402
                                               lookup, publish_addresses)
from paper_1805_08430_b200.fabric import Fabric  # noqa: E402
from paper_1805_08430_b200.graph import Tensor, node_rng, shape_of, synthesize_values  # noqa: E402
from paper_1805_08430_b200.memspace import ArenaAllocator, BufferRef, MemorySpace  # noqa: E402
from paper_1805_08430_b200.runtime.protocol import (DynReceiver, DynSender,  # noqa: E402
                                                    StaticReceiver, StaticSender)
from paper_1805_08430_b200.wire import (AddrExchangeMsg, ElemType, Mechanism,  # noqa: E402
                                        meta_block_size)


def poll_until(fn, what, timeout=20.0):
    t0 = time.time()
    while True:
        got = fn()
        if got is not None:
            return got
        if time.time() - t0 > timeout:
            raise TimeoutError(what)
        time.sleep(1e-4)


def main() -> int:
    one_gpu = os.environ.get("SRFLOW_MP_ONE_GPU") == "1"
    rank, world, local = init_process_group("gloo" if one_gpu else "nccl")
    dev = 0 if one_gpu else local
    torch.cuda.set_device(dev)
    barrier = torch.distributed.barrier
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    bad = 0
    for S in (4, 4096 + 12, (3 << 20) + 4):
        n = S // 4
        space = MemorySpace(rank, 3 * S + (8 << 20), seed=rank, device=dev)
        arena = ArenaAllocator(space, space.allocate_region(3 * S + (4 << 20), register=True))
        recv = arena.alloc(S + 1)                     # static receive region (payload || flag)
        space.write_at(recv, S, b"\x00")
        mblk = arena.alloc(meta_block_size(1))        # dynamic metadata slot
        space.write_at(mblk, mblk.length - 1, b"\x00")
        flag = arena.alloc(1)
        space.write_at(flag, 0, b"\x01")
        payload = arena.alloc(S)
        space.sync()
        proxies = exchange_spaces(space, peers=[nxt] if nxt == prv else [nxt, prv])
        pub = publish_addresses([
            AddrExchangeMsg(2 * rank, recv.base_addr, recv.access_token, recv.length,
                            Mechanism.STATIC),
            AddrExchangeMsg(2 * rank + 1, mblk.base_addr, mblk.access_token, mblk.length,
                            Mechanism.DYNAMIC)])
        fab = Fabric(seed=rank)
        me = fab.create_device(space, qps_per_peer=1)
        peer_dev = {p: fab.create_device(proxies[p], qps_per_peer=1) for p in proxies}
        to_next = me.connect(peer_dev[nxt].endpoint)[0]
        to_prev = to_next if prv == nxt else me.connect(peer_dev[prv].endpoint)[0]
        shape = shape_of(n)
        # producer side of my outgoing edges (receiver = next rank)
        m_s = lookup(pub, nxt, 2 * nxt, Mechanism.STATIC)
        out_s = PlanEntry(2 * nxt, rank, nxt, Mechanism.STATIC, shape, ElemType.F32, 1,
                          remote_addr=m_s.base_addr, remote_token=m_s.token,
                          remote_len=m_s.region_len)
        m_d = lookup(pub, nxt, 2 * nxt + 1, Mechanism.DYNAMIC)
        out_d = PlanEntry(2 * nxt + 1, rank, nxt, Mechanism.DYNAMIC, shape, ElemType.F32, 1,
                          remote_addr=m_d.base_addr, remote_token=m_d.token,
                          remote_len=m_d.region_len)
        # consumer side of my incoming edges (producer = previous rank)
        in_s = PlanEntry(2 * rank, prv, rank, Mechanism.STATIC, shape, ElemType.F32, 1,
                         recv_buffer=recv)
        in_d = PlanEntry(2 * rank + 1, prv, rank, Mechanism.DYNAMIC, shape, ElemType.F32, 1,
                         recv_buffer=mblk)
        ssend = StaticSender(out_s, space, arena, to_next, flag)
        srecv = StaticReceiver(in_s, space)
        dsend = DynSender(out_d, space, arena, to_next)
        drecv = DynReceiver(in_d, space, arena, to_prev)
        barrier()
        for it in (1, 2, 3):
            vals = synthesize_values((n,), ElemType.F32, node_rng(rank, 7, it))
            want = synthesize_values((n,), ElemType.F32, node_rng(prv, 7, it)).tobytes()
            space.write_at(payload, 0, vals)
            space.sync()
            t = Tensor((n,), ElemType.F32, BufferRef(payload), rank)
            ssend.send(t, stage_copy=(it == 2))
            got = poll_until(srecv.poll, f"static S={S} it={it}")
            if space.read_at(got.buffer.handle, 0, S) != want:
                print(f"rank {rank}: static S={S} it={it} differs", flush=True)
                bad += 1
            barrier()   # every receiver consumed (flag clear) before the next send
            dsend.send(t, stage_copy=False)
            meta = poll_until(drecv.poll, f"dynamic S={S} it={it}")
            pulled = drecv.fetch(meta)
            if space.read_at(pulled.buffer.handle, 0, S) != want:
                print(f"rank {rank}: dynamic S={S} it={it} differs", flush=True)
                bad += 1
            pulled.buffer.release()
            barrier()   # the pull finished before the sender releases its payload
        dsend.close()
        barrier()
        for p in proxies.values():
            p.close()
        barrier()
        space.close()
    print(f"rank {rank}: {'OK' if bad == 0 else 'FAIL'}", flush=True)
    torch.distributed.destroy_process_group()
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
