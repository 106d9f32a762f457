"""GPU twin of the reference protocol-test rig (tests/test_protocol.py:15-71):
two servers (GPU 0 and GPU 1 when two are visible, else both on GPU 0) with
registered arenas, connected devices and flag cells."""
from __future__ import annotations

import math

import numpy as np

from paper_1805_08430_b200.analyzer import PlanEntry
from paper_1805_08430_b200.fabric import Fabric
from paper_1805_08430_b200.graph import Tensor, TensorShape
from paper_1805_08430_b200.memspace import ArenaAllocator, BufferRef, MemorySpace
from paper_1805_08430_b200.wire import (ElemType, Mechanism, meta_block_size,
                                        static_region_size)


class Rig:
    def __init__(self, faults=None, capacity=1 << 22, qps=2, seed=5):
        self.fabric = Fabric(seed=seed, faults=faults)
        self.spaces = {s: MemorySpace(s, capacity, seed=s) for s in (0, 1)}
        self.arenas = {}
        for s, space in self.spaces.items():
            self.arenas[s] = ArenaAllocator(space, space.allocate_region(capacity // 2,
                                                                         register=True))
        self.devices = {s: self.fabric.create_device(self.spaces[s], qps_per_peer=qps)
                        for s in (0, 1)}
        self.fwd = self.devices[0].connect(self.devices[1].endpoint)
        self.back = self.devices[1].channels_to(self.devices[0].endpoint)
        self.flags = {}
        for s in (0, 1):
            cell = self.arenas[s].alloc(1)
            self.spaces[s].write_at(cell, 0, b"\x01")
            self.flags[s] = cell

    def entry(self, dims, mechanism, elem=ElemType.F32, edge_id=0, producer=0, consumer=1):
        shape = TensorShape(tuple(dims))
        entry = PlanEntry(edge_id, producer, consumer, mechanism, shape, elem, shape.rank)
        size = (static_region_size(shape.static_dims(), elem) if mechanism is Mechanism.STATIC
                else meta_block_size(shape.rank))
        buf = self.arenas[consumer].alloc(size)
        self.spaces[consumer].write_at(buf, size - 1, b"\x00")
        entry.recv_buffer = buf
        entry.remote_addr, entry.remote_token, entry.remote_len = \
            buf.base_addr, buf.access_token, buf.length
        return entry

    def tensor(self, dims, elem=ElemType.F32, server=0, arena=True, data=None, seed=42):
        dims = tuple(dims)
        nbytes = math.prod(dims) * elem.size
        if data is None:
            data = np.random.default_rng(seed).integers(0, 256, nbytes, dtype=np.uint8).tobytes()
        space = self.spaces[server]
        if arena:
            h = self.arenas[server].alloc(max(nbytes, 1))
            ref = BufferRef(h, self.arenas[server])
        else:
            h = space.allocate_region(max(nbytes, 1))
            ref = BufferRef(h)
        if nbytes:
            space.write_at(h, 0, data[:nbytes])
        return Tensor(dims, elem, ref, server)

    def close(self):
        for sp in self.spaces.values():
            sp.close()
