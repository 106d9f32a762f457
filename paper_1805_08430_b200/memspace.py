"""Per-server memory: one HBM pool per server, regions, tokens, arenas.

B200 restatement of the reference memory layer (rdmaflow ``memspace.py``):

* ``MemorySpace`` (memspace.py:89-236) owns one ``cudaMalloc(capacity)`` pool
  on the server's GPU (zero-filled like ``np.zeros``).  The region table, the
  8-byte bump pointer and the token/bounds gates live in libsrflow
  (``srf_region_alloc``/``srf_check_*``), so every verb is checked in C right
  before its kernel launch.  Addresses stay space-relative offsets.
* Tokens are drawn host-side from the same seeded stream as the reference
  (memspace.py:113, :128), so region coordinates and exchanged tokens match
  the reference bit for bit.
* ``ArenaAllocator`` (memspace.py:239-308) and ``BufferRef`` (:315-365) are
  host bookkeeping over the pool - they never touch bytes.
* ``copy_bytes`` (memspace.py:223-236) is the counted D2D copy K5.

Byte IO (``read_at``/``write_at``/``*_raw``) is synchronous host<->device
copying; it exists for setup, tests and the oracle comparison, never for
moving payloads between servers.
"""
from __future__ import annotations

import bisect
import ctypes as C
import os
import random
import threading
from dataclasses import dataclass, replace
from typing import Callable, Optional

import numpy as np

from . import _lib, errors

DEFAULT_CAPACITY = 256 * 1024 * 1024
DEFAULT_ARENA_BYTES = 64 * 1024 * 1024
DEFAULT_MAX_REGIONS = 1024

ALIGN = 8


def align_up(n: int, a: int = ALIGN) -> int:
    return -(-n // a) * a


@dataclass(frozen=True)
class RegionHandle:
    """(region id, base, length, token) of a byte range in one space.

    Arena blocks carry their backing region's id and token, as sub-ranges of
    one registered region do (memspace.py:39-54).
    """

    region_id: int
    base_addr: int
    length: int
    access_token: int

    @property
    def end(self) -> int:
        return self.base_addr + self.length


@dataclass
class CopyCounters:
    """Monotone copy counters of one space (memspace.py:57-71)."""

    payload_bytes_copied: int = 0
    payload_copy_events: int = 0
    serialize_bytes: int = 0

    def snapshot(self) -> "CopyCounters":
        return replace(self)

    def reset(self) -> None:
        self.payload_bytes_copied = self.payload_copy_events = self.serialize_bytes = 0


def token_stream(server_id: int, seed: int) -> random.Random:
    """Token RNG of a space, seeded as in memspace.py:113."""
    return random.Random(((seed & 0xFFFFFFFF) << 20) ^ (server_id * 0x9E3779B1) ^ 0x5EED)


_device_map: dict[int, int] = {}


def set_device_map(mapping: dict[int, int]) -> None:
    """Pin servers to GPUs (server id -> CUDA device) for spaces made later."""
    _device_map.update({int(k): int(v) for k, v in mapping.items()})


def default_device(server_id: int) -> int:
    """GPU of a server: explicit map, else $SRFLOW_DEVICES, else round-robin."""
    if server_id in _device_map:
        return _device_map[server_id]
    env = os.environ.get("SRFLOW_DEVICES")
    if env:
        devs = [int(x) for x in env.split(",") if x.strip()]
        return devs[server_id % len(devs)]
    n = _lib.device_count()
    if n < 1:
        raise errors.DeviceError("no CUDA device visible; the transfer path runs on B200 only")
    return server_id % n


def _fetch_fd(pid: int, fd: int) -> int:
    """Duplicate file descriptor ``fd`` of process ``pid`` into this process
    (pidfd_getfd, Linux >= 5.6)."""
    libc = C.CDLL(None, use_errno=True)
    pidfd = os.pidfd_open(pid)
    try:
        got = libc.syscall(438, pidfd, fd, 0)  # SYS_pidfd_getfd on x86_64
        if got < 0:
            err = C.get_errno()
            raise errors.PeerUnreachable(f"pidfd_getfd({pid}, {fd}): {os.strerror(err)}")
        return got
    finally:
        os.close(pidfd)


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter for zero-copy torch views."""

    __slots__ = ("__cuda_array_interface__",)

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {
            "data": (ptr, False), "shape": shape, "typestr": typestr,
            "strides": None, "version": 3, "stream": None,
        }


def device_view(ptr: int, nbytes: int, device: int, dtype=None, shape=None):
    """torch tensor aliasing ``nbytes`` of device memory at ``ptr``."""
    import torch
    if nbytes == 0:
        t = torch.empty(0, dtype=torch.uint8, device=f"cuda:{device}")
    else:
        t = torch.as_tensor(_CudaArray(ptr, (nbytes,), "|u1"), device=f"cuda:{device}")
    if dtype is not None and dtype != torch.uint8:
        t = t.view(dtype)
    if shape is not None:
        t = t.reshape(shape)
    return t


class MemorySpace:
    """HBM pool of one server.  Same constructor as memspace.py:98-99 plus
    ``device`` (CUDA ordinal; default from :func:`default_device`)."""

    def __init__(self, server_id: int, capacity: int = DEFAULT_CAPACITY, *,
                 max_regions: int = DEFAULT_MAX_REGIONS, seed: int = 0,
                 device: Optional[int] = None):
        self.server_id = server_id
        self.capacity = capacity
        self.max_regions = max_regions
        self.counters = CopyCounters()
        #: hook called as on_copy(nbytes) after each counted copy
        self.on_copy: Optional[Callable[[int], None]] = None
        self.device = default_device(server_id) if device is None else device
        self._rng = token_stream(server_id, seed)
        self._lock = threading.RLock()
        self._torch_stream = None
        #: (region_id, base, length, registered, token) - exported to peers
        self.regions: list[tuple[int, int, int, bool, int]] = []
        self.remote = False
        self._inflight: dict = {}    # receive flag -> event of a write in flight
        self._pulls: dict = {}       # payload addr -> event of a peer's pull
        h = C.c_void_p()
        _lib.call("srf_space_create", server_id, self.device, capacity, max_regions,
                  C.byref(h))
        self._h = h
        base = C.c_void_p()
        _lib.call("srf_space_info", self._h, None, None, None, C.byref(base))
        self.device_base = base.value or 0

    # -- multi-process: export / import (one process per GPU) -------------------

    def export(self) -> dict:
        """Descriptor a peer process needs to map this pool over NVLink: the
        CUDA IPC handle (cudaMalloc pools) or (pid, fd) of the VMM allocation
        (SRFLOW_ALLOC_VMM=1 pools), plus the region table for identical checks."""
        desc = {"server_id": self.server_id, "capacity": self.capacity,
                "regions": list(self.regions)}
        buf = (C.c_uint8 * 64)()
        try:
            _lib.call("srf_space_export", self._h, buf)
            desc["ipc"] = bytes(buf)
        except errors.InvalidConfig:
            fd = C.c_int()
            _lib.call("srf_space_export_fd", self._h, C.byref(fd))
            desc["pid"], desc["fd"] = os.getpid(), fd.value
        return desc

    @classmethod
    def import_remote(cls, desc: dict, local_device: int) -> "MemorySpace":
        """Proxy for a peer process's pool, mapped into this process on
        ``local_device`` (cudaIpcOpenMemHandle).  Verbs may target it; it
        cannot allocate."""
        self = cls.__new__(cls)
        self.server_id = desc["server_id"]
        self.capacity = desc["capacity"]
        self.max_regions = 1 << 30
        self.counters = CopyCounters()
        self.on_copy = None
        self.device = local_device
        self._rng = None
        self._lock = threading.RLock()
        self._torch_stream = None
        self.regions = list(desc["regions"])
        self.remote = True
        self._inflight, self._pulls = {}, {}
        h = C.c_void_p()
        if "ipc" in desc:
            ipc = (C.c_uint8 * 64).from_buffer_copy(desc["ipc"])
            _lib.call("srf_space_import", ipc, self.server_id, local_device, self.capacity,
                      C.byref(h))
        else:
            fd = _fetch_fd(desc["pid"], desc["fd"])
            try:
                _lib.call("srf_space_import_fd", fd, self.server_id, local_device,
                          self.capacity, C.byref(h))
            finally:
                os.close(fd)
        self._h = h
        for rid, base, length, reg, token in self.regions:
            _lib.call("srf_region_import", h, rid, base, length, int(reg), token)
        base = C.c_void_p()
        _lib.call("srf_space_info", h, None, None, None, C.byref(base))
        self.device_base = base.value or 0
        return self

    # -- plumbing -------------------------------------------------------------

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def cuda_stream(self) -> int:
        return _lib.load().srf_space_cuda_stream(self._h) or 0

    def torch_stream(self):
        """The space's default CUDA stream as a torch stream."""
        if self._torch_stream is None:
            import torch
            self._torch_stream = torch.cuda.ExternalStream(
                self.cuda_stream, device=f"cuda:{self.device}")
        return self._torch_stream

    def sync(self) -> None:
        """Wait for all work queued on this space's stream."""
        _lib.call("srf_space_sync", self._h)

    def fence(self) -> "_lib.Event":
        """An event after all work queued so far on this space's stream."""
        h = C.c_void_p()
        _lib.call("srf_event_record", self._h, None, C.byref(h))
        return _lib.Event(h)

    def close(self) -> None:
        for table in (getattr(self, "_inflight", {}), getattr(self, "_pulls", {})):
            for ev in table.values():
                ev.free()
            table.clear()
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().srf_space_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def next_addr(self) -> int:
        v = C.c_uint64()
        _lib.call("srf_next_addr", self._h, C.byref(v))
        return v.value

    # -- regions (memspace.py:116-167) ------------------------------------------

    def allocate_region(self, length: int, register: bool = False) -> RegionHandle:
        if self.remote:
            raise errors.InvalidConfig("cannot allocate in a remote space proxy")
        if length < 1:
            raise errors.ZeroLength(f"region length must be >= 1, got {length}")
        with self._lock:
            # draw the token only for an allocation that will succeed, so the
            # token stream advances exactly like the reference's
            if self.region_count() >= self.max_regions:
                raise errors.OutOfMemory(
                    f"server {self.server_id}: region table full ({self.max_regions})")
            base = align_up(self.next_addr)
            if base + length > self.capacity:
                raise errors.OutOfMemory(
                    f"server {self.server_id}: need {length} bytes at {base}, "
                    f"capacity {self.capacity}")
            token = self._rng.getrandbits(64) if register else 0
            rid, addr = C.c_int64(), C.c_uint64()
            _lib.call("srf_region_alloc", self._h, length, int(register), token,
                      C.byref(rid), C.byref(addr))
            self.regions.append((rid.value, addr.value, length, bool(register), token))
            return RegionHandle(rid.value, addr.value, length, token)

    def region_count(self) -> int:
        n = C.c_uint32()
        _lib.call("srf_region_count", self._h, C.byref(n))
        return n.value

    def check_remote_access(self, addr: int, length: int, token: int) -> None:
        _lib.call("srf_check_remote", self._h, addr, length, token)

    def check_registered(self, handle: RegionHandle, offset: int = 0,
                         length: Optional[int] = None) -> None:
        if length is None:
            length = handle.length - offset
        _lib.call("srf_check_registered", self._h, handle.base_addr + offset,
                  length, handle.access_token)

    # -- byte IO (memspace.py:171-219) -----------------------------------------

    def _handle_range(self, handle: RegionHandle, offset: int, length: int) -> int:
        if offset < 0 or length < 0 or offset + length > handle.length:
            raise errors.OutOfBounds(
                f"range [{offset}, {offset + length}) escapes handle of {handle.length} bytes")
        addr = handle.base_addr + offset
        if addr < 0 or addr + length > self.capacity:
            raise errors.OutOfBounds(f"address range [{addr}, {addr + length}) escapes space")
        return addr

    def _raw_range(self, addr: int, length: int, what: str) -> None:
        if addr < 0 or length < 0 or addr + length > self.capacity:
            raise errors.OutOfBounds(f"raw {what} [{addr}, {addr + length})")

    def _d2h(self, addr: int, length: int) -> bytes:
        if length == 0:
            return b""
        out = np.empty(length, dtype=np.uint8)
        _lib.call("srf_read", self._h, addr, length, out.ctypes.data)
        return out.tobytes()

    def _h2d(self, addr: int, data) -> None:
        arr = np.ascontiguousarray(
            np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray)
            else data.reshape(-1).view(np.uint8))
        if arr.size:
            _lib.call("srf_write", self._h, addr, arr.size, arr.ctypes.data)

    def read_at(self, handle: RegionHandle, offset: int, length: int) -> bytes:
        return self._d2h(self._handle_range(handle, offset, length), length)

    def write_at(self, handle: RegionHandle, offset: int, data) -> None:
        n = len(data) if not isinstance(data, np.ndarray) else data.nbytes
        self._h2d(self._handle_range(handle, offset, n), data)

    def view(self, handle: RegionHandle, offset: int = 0,
             length: Optional[int] = None):
        """Writable uint8 device view (a torch tensor aliasing the pool).

        Work torch issues on the view runs on torch's stream, which is not
        ordered with this space's stream: synchronise it (e.g.
        ``torch.cuda.current_stream(dev).synchronize()``) before a verb reads
        or writes the same bytes."""
        if length is None:
            length = handle.length - offset
        addr = self._handle_range(handle, offset, length)
        return device_view(self.device_base + addr, length, self.device)

    def read_raw(self, addr: int, length: int) -> bytes:
        self._raw_range(addr, length, "read")
        return self._d2h(addr, length)

    def view_raw(self, addr: int, length: int):
        self._raw_range(addr, length, "view")
        return device_view(self.device_base + addr, length, self.device)

    def write_raw(self, addr: int, data) -> None:
        n = len(data) if not isinstance(data, np.ndarray) else data.nbytes
        self._raw_range(addr, n, "write")
        self._h2d(addr, data)

    def device_ptr(self, addr: int) -> int:
        return self.device_base + addr

    def write_async(self, handle: RegionHandle, offset: int, pinned, length: int) -> None:
        """H2D from a pinned staging buffer, ordered on the space's stream (the
        verbs this space issues next see the bytes; no host wait)."""
        addr = self._handle_range(handle, offset, length)
        _lib.call("srf_write_async", self._h, addr, length, pinned.ptr, None)

    # -- receive flags (host doorbells) ------------------------------

    def bind_doorbell(self, handle: RegionHandle, mirror: bool = False) -> None:
        """Give a receive region a host-visible shadow that this process's
        one-sided writes keep current (flag only, or the whole block)."""
        if self.remote:
            return
        _lib.call("srf_doorbell_bind", self._h, handle.base_addr, handle.length, int(mirror))

    # -- asynchronous dynamic verbs within one process --------------------------
    # A DynSender's metadata write and a DynReceiver's pull complete on the
    # device after the call returns; these tables keep the reference's
    # observable order: a poll of a receive flag with a write in flight waits
    # for that write (so `polls` counts stay the reference's), and a payload
    # that a peer is still pulling is not reused before the pull finished.

    def note_inflight_write(self, tail_addr: int, ev: "_lib.Event") -> None:
        old = self._inflight.pop(tail_addr, None)
        if old is not None:
            old.free()
        self._inflight[tail_addr] = ev

    def settle_inflight_write(self, tail_addr: int) -> None:
        ev = self._inflight.pop(tail_addr, None)
        if ev is not None:
            ev.wait_free()

    def note_pull(self, addr: int, ev: "_lib.Event") -> None:
        old = self._pulls.pop(addr, None)
        if old is not None:
            old.free()
        self._pulls[addr] = ev

    def order_after_pull(self, addr: int) -> None:
        """Order this space's stream after a peer's pull of ``addr`` (no host
        wait)."""
        ev = self._pulls.pop(addr, None)
        if ev is not None:
            _lib.call("srf_space_wait_event", self._h, ev._h)
            ev.free()

    def flag_read(self, tail_addr: int, length: int = 1) -> bytes:
        """The ``length`` bytes ending at ``tail_addr`` (inclusive): from the
        doorbell shadow when possible, else from the device."""
        out = (C.c_uint8 * length)()
        _lib.call("srf_flag_read", self._h, tail_addr, length, out)
        return bytes(out)

    def flag_clear(self, tail_addr: int) -> None:
        _lib.call("srf_flag_clear", self._h, tail_addr)

    # -- counted copy (memspace.py:223-236): kernel K5 ---------------------------

    def copy_bytes(self, src: RegionHandle, src_off: int,
                   dst: RegionHandle, dst_off: int, length: int) -> None:
        if length == 0:
            return
        s = self._handle_range(src, src_off, length)
        d = self._handle_range(dst, dst_off, length)
        _lib.call("srf_copy", self._h, s, d, length, None, None)
        with self._lock:
            self.counters.payload_bytes_copied += length
            self.counters.payload_copy_events += 1
        if self.on_copy is not None:
            self.on_copy(length)


class ArenaAllocator:
    """First-fit sub-allocator over one backing region (memspace.py:239-308).

    Blocks reserve ``align_up(len, 8)`` bytes; residency is counted in the
    requested bytes; freed blocks merge with both neighbours.  Pure host
    bookkeeping: the bytes live in the space's HBM pool.
    """

    def __init__(self, space: MemorySpace, backing: RegionHandle):
        self.space = space
        self.backing = backing
        self.current_resident = 0
        self.peak_resident = 0
        usable = backing.length & ~(ALIGN - 1)
        # sorted by offset: parallel lists of starts and lengths
        self._starts: list[int] = [0] if usable else []
        self._lens: list[int] = [usable] if usable else []
        self._live: dict[int, tuple[int, int]] = {}
        self._lock = threading.Lock()
        # (offset, reserved, Event) of blocks freed while device work could
        # still touch them (BufferRef.release): the bookkeeping free is
        # immediate - first-fit addresses stay the reference's - and a later
        # allocation that reuses any of those bytes orders the space's stream
        # after the fence
        self._fences: list[tuple[int, int, "_lib.Event"]] = []

    def _wait_fences(self, off: int, need: int) -> None:
        keep = []
        for f_off, f_len, ev in self._fences:
            if f_off < off + need and off < f_off + f_len:
                if not ev.query():
                    _lib.call("srf_space_wait_event", self.space.handle, ev._h)
                ev.free()
            elif ev.query():
                ev.free()
            else:
                keep.append((f_off, f_len, ev))
        self._fences = keep

    def alloc(self, length: int) -> RegionHandle:
        if length < 1:
            raise errors.ZeroLength(f"arena allocation must be >= 1 byte, got {length}")
        need = align_up(length)
        with self._lock:
            for i, size in enumerate(self._lens):
                if size < need:
                    continue
                off = self._starts[i]
                if size == need:
                    del self._starts[i], self._lens[i]
                else:
                    self._starts[i] = off + need
                    self._lens[i] = size - need
                addr = self.backing.base_addr + off
                if self._fences:
                    self._wait_fences(off, need)
                self._live[addr] = (length, need)
                self.current_resident += length
                self.peak_resident = max(self.peak_resident, self.current_resident)
                return RegionHandle(self.backing.region_id, addr, length,
                                    self.backing.access_token)
        raise errors.ArenaExhausted(
            f"server {self.space.server_id}: no free block of {length} bytes "
            f"(resident {self.current_resident}/{self.backing.length})")

    def free(self, handle: RegionHandle, fence: Optional["_lib.Event"] = None) -> None:
        """Return a block (memspace.py:279-290).  ``fence``: an event after
        the last device work that may use the block; reusing its bytes waits
        for it."""
        with self._lock:
            entry = self._live.pop(handle.base_addr, None)
            if entry is None:
                if fence is not None:
                    fence.free()
                raise ValueError(f"not a live arena block: addr {handle.base_addr}")
            requested, reserved = entry
            off = handle.base_addr - self.backing.base_addr
            self._give_back(off, reserved)
            self.current_resident -= requested
            if fence is not None:
                self._fences.append((off, reserved, fence))

    def _give_back(self, off: int, length: int) -> None:
        i = bisect.bisect_left(self._starts, off)
        if i > 0 and self._starts[i - 1] + self._lens[i - 1] == off:
            i -= 1
            off = self._starts[i]
            length += self._lens[i]
            del self._starts[i], self._lens[i]
        if i < len(self._starts) and off + length == self._starts[i]:
            length += self._lens[i]
            del self._starts[i], self._lens[i]
        self._starts.insert(i, off)
        self._lens.insert(i, length)

    def live_blocks(self) -> list[tuple[int, int]]:
        """Sorted (offset, reserved length) of live blocks."""
        with self._lock:
            return sorted((addr - self.backing.base_addr, res)
                          for addr, (_req, res) in self._live.items())


class BufferRef:
    """Refcounted hold on an arena block, or a non-owned view when
    ``arena is None`` (memspace.py:315-357)."""

    __slots__ = ("handle", "arena", "_refs", "_lock")

    def __init__(self, handle: RegionHandle, arena: Optional[ArenaAllocator] = None,
                 refs: int = 1):
        self.handle = handle
        self.arena = arena
        self._refs = refs
        self._lock = threading.Lock()

    @property
    def nbytes(self) -> int:
        return self.handle.length

    @property
    def refs(self) -> int:
        return self._refs

    def retain(self, n: int = 1) -> "BufferRef":
        with self._lock:
            self._refs += n
        return self

    def release(self, n: int = 1) -> None:
        with self._lock:
            self._refs -= n
            if self._refs < 0:
                raise AssertionError("buffer over-released")
            owned_and_dead = self._refs == 0 and self.arena is not None
        if owned_and_dead:
            # event-guarded: device work queued on the space's stream before
            # this release may still read or write the block, and so may a
            # peer's pull of it (a DynReceiver in this process)
            space = self.arena.space
            if getattr(space, "_pulls", None):
                space.order_after_pull(self.handle.base_addr)
            fence = getattr(space, "fence", None)
            self.arena.free(self.handle, fence=fence() if fence is not None else None)

    def __repr__(self) -> str:  # pragma: no cover
        kind = "owned" if self.arena is not None else "view"
        return (f"BufferRef({kind}, addr={self.handle.base_addr}, "
                f"len={self.handle.length}, refs={self._refs})")


NULL_HANDLE = RegionHandle(-1, 0, 0, 0)


def null_buffer() -> BufferRef:
    """Zero-length placeholder buffer of empty tensors."""
    return BufferRef(NULL_HANDLE, None, refs=1)
