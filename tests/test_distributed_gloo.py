"""N>1 host logic on CPU: world_size-2 gloo process group exercising the
control plane of the multi-process path (paper_1805_08430_b200.distributed):
descriptor gathering, the 33-byte address exchange, and that every rank
derives the same peer coordinates from the PS layout as the peer publishes."""
from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                          RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
        from paper_1805_08430_b200 import distributed as D
        from paper_1805_08430_b200 import errors
        from paper_1805_08430_b200.ps import PsLayout
        from paper_1805_08430_b200.wire import AddrExchangeMsg, Mechanism
        from paper_1805_08430_b200.workloads import vgg16_shapes

        r, w, local = D.init_process_group("gloo")
        assert (r, w) == (rank, world)
        # 1. pool descriptors: one per server, duplicates rejected
        desc = {"server_id": rank, "capacity": 1 << 20, "ipc": bytes(64),
                "regions": [(0, 0, 4096, True, 1000 + rank)]}
        table = D.gather_descriptors(desc)
        assert sorted(table) == list(range(world))
        assert table[1 - rank]["regions"][0][4] == 1000 + (1 - rank)
        # 2. address exchange with the reference wire encoding
        L = PsLayout(vgg16_shapes(), world, world, colocate=True)
        mine = []
        for v in range(32):
            if L.shard_of(v) != rank:
                off = L.blocks[rank][("wbuf", v)]
                mine.append(AddrExchangeMsg(v, off, 1000 + rank, L.nbytes(v) + 1,
                                            Mechanism.STATIC))
        pub = D.publish_addresses(mine)
        peer = 1 - rank
        for v in range(32):
            if L.shard_of(v) == rank:  # I push v to the peer: its published slot
                msg = D.lookup(pub, peer, v, Mechanism.STATIC)
                assert msg.base_addr == L.blocks[peer][("wbuf", v)]
                assert msg.token == 1000 + peer and msg.region_len == L.nbytes(v) + 1
        with pytest.raises(errors.ProtocolError):
            D.lookup(pub, peer, next(v for v in range(32) if L.shard_of(v) == rank),
                     Mechanism.DYNAMIC)
        with pytest.raises(errors.UnknownAddress):
            D.lookup(pub, peer, 999, Mechanism.STATIC)
        # 3. traffic symmetry: what one rank sends the other receives
        t = [L.traffic(s) for s in range(world)]
        assert t[0]["link_out"] == t[1]["link_in"] and t[1]["link_out"] == t[0]["link_in"]
        # 4. every rank derives the same layouts - peers' block coordinates are
        # computed, not exchanged - including the labelled extensions
        import hashlib
        import json
        digests = []
        for kw in ({}, {"placement": "bytes"},
                   {"placement": "bytes", "partition_bytes": 16 << 20},
                   {"slice_bytes": 8 << 20}, {"grad_mechanism": "static"}):
            Lx = PsLayout(vgg16_shapes(), world, world, colocate=True, **kw)
            blob = json.dumps([[sorted((str(k), o) for k, o in Lx.blocks[s].items())
                                for s in range(Lx.nservers)], Lx.units, Lx.sizes],
                              sort_keys=True).encode()
            digests.append(hashlib.sha256(blob).hexdigest())
        got = D.all_gather_objects(digests)
        assert all(g == got[0] for g in got)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # report to the parent
        errq.put(f"rank {rank}: {type(exc).__name__}: {exc}")
        raise


def test_two_rank_control_plane():
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)


def _worker8(rank: int, world: int, port: int, errq):
    """The bench's N=8 placements (SCALE run): every rank derives identical
    layouts for each PS line; C5 (7 workers + 1 PS) and C3 (2 workers + 1 PS)
    put server s on GPU s mod 8; NVLink bytes balance (sum out = sum in)."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                          RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
        import hashlib
        import json
        from paper_1805_08430_b200 import distributed as D
        from paper_1805_08430_b200.ps import PsLayout, link_traffic
        from paper_1805_08430_b200.workloads import vgg16_shapes
        r, w, _local = D.init_process_group("gloo")
        assert (r, w) == (rank, world)
        layouts = {
            "vgg": PsLayout(vgg16_shapes(), world, world, colocate=True),
            "vgg_sliced_static": PsLayout(vgg16_shapes(), world, world, colocate=True,
                                          slice_bytes=8 << 20, grad_mechanism="static"),
            "vgg_sliced_dynamic": PsLayout(vgg16_shapes(), world, world, colocate=True,
                                           slice_bytes=16 << 20),
            "vgg_partitioned": PsLayout(vgg16_shapes(), world, world, colocate=True,
                                        placement="bytes", partition_bytes=16 << 20,
                                        slice_bytes=4 << 20),
            "fcn5": PsLayout([(int(204.47e6) // 10 // 4,)] * 10, 2, 1, False),
            "lstm": PsLayout([(int(35.93e6) // 14 // 4,)] * 14, 7, 1, False),
        }
        assert layouts["lstm"].nservers == 8          # C5: one server per GPU at N=8
        assert layouts["fcn5"].nservers == 3          # C3: GPUs 0-2, the rest idle
        digests = {}
        for name, L in layouts.items():
            blob = json.dumps([[sorted((str(k), o) for k, o in L.blocks[s].items())
                                for s in range(L.nservers)], L.units, L.sizes],
                              sort_keys=True).encode()
            digests[name] = hashlib.sha256(blob).hexdigest()
            t = link_traffic(L, world)
            assert sum(x["link_out"] for x in t.values()) == sum(x["link_in"] for x in t.values())
        got = D.all_gather_objects(digests)
        assert all(g == got[0] for g in got)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:
        errq.put(f"rank {rank}: {type(exc).__name__}: {exc}")
        raise


def test_eight_rank_placements():
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker8, args=(r, 8, port, errq)) for r in range(8)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
