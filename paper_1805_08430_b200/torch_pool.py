"""Torch tensors born in registered memory.

The reference makes a tensor zero-copy sendable by tracing its allocation site
and moving the producer's allocation into the RDMA arena
(``analyzer.py:226-272``, ``runtime/session.py:91-122``); only the graph's own
producers get that treatment.  Here torch's CUDA allocator itself is replaced
(``torch.cuda.memory.CUDAPluggableAllocator`` over ``srf_torch_malloc`` /
``srf_torch_free`` in libsrflow) by a first-fit allocator over ONE registered
region of a :class:`MemorySpace`, so every tensor torch creates on that GPU is
already inside a registered region: :meth:`TorchPool.locate` gives the
``(addr, length, token)`` a one-sided verb takes, with no staging copy.

The allocator must be installed before torch makes its first CUDA allocation
in the process (a torch restriction).  Freed blocks are reused only after the
stream that freed them has passed them (an event per free), like the caching
allocator's stream-ordered reuse.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from . import _lib, errors
from .memspace import MemorySpace


class TorchPool:
    """A registered pool on one GPU behind torch's allocator."""

    def __init__(self, capacity: int, device: int = 0, server_id: Optional[int] = None,
                 seed: int = 0):
        if capacity < 1 << 20:
            raise errors.InvalidConfig("torch pool needs at least 1 MiB")
        self.device = device
        self.space = MemorySpace(900 + device if server_id is None else server_id,
                                 capacity + (1 << 20), seed=seed, device=device)
        self.region = self.space.allocate_region(capacity, register=True)
        _lib.call("srf_torch_pool_attach", self.space.handle, self.region.base_addr,
                  self.region.length)
        self._installed = False

    def install(self) -> None:
        """Route torch's CUDA allocations through the pool (before any tensor
        is allocated on a GPU in this process)."""
        import torch
        alloc = torch.cuda.memory.CUDAPluggableAllocator(_lib.LIB_PATH,
                                                         "srf_torch_malloc", "srf_torch_free")
        torch.cuda.memory.change_current_allocator(alloc)
        self._installed = True

    def locate(self, tensor) -> tuple[int, int, int]:
        """(space-relative address, byte length, access token) of a tensor's
        bytes; raises NotRegistered if they are not inside the pool."""
        ptr = tensor.data_ptr()
        n = tensor.numel() * tensor.element_size()
        addr = ptr - self.space.device_base
        r = self.region
        if not (tensor.is_contiguous() and r.base_addr <= addr and addr + n <= r.base_addr + r.length):
            raise errors.NotRegistered(
                f"tensor at {ptr:#x} (+{n}) is not contiguous inside the torch pool")
        return addr, n, r.access_token

    def as_tensor(self, tensor):
        """The torch tensor as a runtime :class:`~paper_1805_08430_b200.graph.Tensor`
        of this pool's space: a non-owned view of its bytes inside the
        registered region, so the reference endpoints send it zero-copy
        (``StaticSender.send(..., stage_copy=False)`` puts straight from it,
        ``DynSender.send`` announces its address for the receiver's pull) -
        the sender-side zero-copy the reference reaches by tracing allocation
        sites (``analyzer.py:226-272``), here for any tensor torch produced."""
        from .graph import Tensor
        from .memspace import BufferRef, RegionHandle
        from .wire import ElemType
        import torch
        kinds = {torch.float32: ElemType.F32, torch.float64: ElemType.F64,
                 torch.int32: ElemType.I32, torch.int64: ElemType.I64,
                 torch.uint8: ElemType.U8}
        if tensor.dtype not in kinds:
            raise errors.InvalidConfig(f"no wire element type for {tensor.dtype}")
        addr, n, tok = self.locate(tensor)
        view = BufferRef(RegionHandle(self.region.region_id, addr, n, tok))
        return Tensor(tuple(int(d) for d in tensor.shape), kinds[tensor.dtype], view,
                      self.space.server_id)

    def stats(self) -> dict:
        used, peak, cap = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _lib.call("srf_torch_pool_stats", self.device, C.byref(used), C.byref(peak),
                  C.byref(cap))
        return {"in_use": used.value, "peak": peak.value, "capacity": cap.value}
