"""One process per GPU: pool export/import and address exchange.

The reference runs every server in one process and distributes receiver
buffer coordinates with an in-fabric RPC (analyzer.py:166-220, wire.py:145-171).
Across processes the control plane is ``torch.distributed`` (NCCL on the GPU
box, gloo in CPU tests); the data plane stays one-sided: each process maps its
peers' HBM pools through CUDA IPC (``MemorySpace.import_remote``) and the
kernels store/load peer memory over NVLink directly.  The exchanged address
records are the reference's 33-byte ``AddrExchangeMsg`` encodings.
"""
from __future__ import annotations

import os
from typing import Optional

from . import errors
from .wire import AddrExchangeMsg, Mechanism


def env_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_process_group(backend: Optional[str] = None) -> tuple[int, int, int]:
    """Initialise torch.distributed when launched with WORLD_SIZE > 1."""
    import torch
    import torch.distributed as dist
    rank, world, local = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def all_gather_objects(obj) -> list:
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def gather_descriptors(desc: dict) -> dict[int, dict]:
    """server id -> exported pool descriptor, from every rank."""
    got = all_gather_objects(desc)
    table: dict[int, dict] = {}
    for d in got:
        if d["server_id"] in table:
            raise errors.InvalidConfig(f"server {d['server_id']} exported twice")
        table[d["server_id"]] = d
    return table


def exchange_spaces(local_space, peers: Optional[list[int]] = None) -> dict:
    """Map the pools of ``peers`` (default: every other rank's server) into this
    process as remote space proxies on this process's GPU."""
    from .memspace import MemorySpace
    table = gather_descriptors(local_space.export())
    wanted = [s for s in sorted(table) if s != local_space.server_id] if peers is None else peers
    return {s: MemorySpace.import_remote(table[s], local_space.device) for s in wanted}


def publish_addresses(records: list[AddrExchangeMsg]) -> dict[int, list[AddrExchangeMsg]]:
    """Every rank publishes the coordinates of the buffers it receives into;
    returns rank -> records (decoded from their 33-byte wire encoding)."""
    got = all_gather_objects([r.encode() for r in records])
    return {rank: [AddrExchangeMsg.decode(b) for b in blobs] for rank, blobs in enumerate(got)}


def lookup(published: dict[int, list[AddrExchangeMsg]], rank: int, edge_id: int,
           mechanism: Mechanism) -> AddrExchangeMsg:
    for msg in published[rank]:
        if msg.edge_id == edge_id:
            if msg.mechanism != mechanism:
                raise errors.ProtocolError(f"address exchange mismatch on edge {edge_id}")
            return msg
    raise errors.UnknownAddress(f"rank {rank} published no buffer for edge {edge_id}")
