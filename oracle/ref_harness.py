"""Timing harness around the REAL reference (TEST INFRASTRUCTURE ONLY).

Imports rdmaflow from oracle/_ref (vendored by oracle/vendor_ref.py; on this
container also straight from /root/reference/pkg/src) and drives it through
its own public API and stock code path, for bench.py's CPU arm
(``--impl reference``, ``cpu_baseline.kind = "reference"``) and
``cpu_sweep``.  Nothing in paper_1805_08430_b200 imports this module.

* Session arms (SURVEY.md 8(d) "How to time the CPU reference"):
  ``Session(build_microbench(S), mode, seed=0, capacity/arena from
  benchcli._memory_for)``, one ``run(1)`` per step after the iteration-1
  tracing warm-up - the reference's own steady ``wall_time_us``
  (runtime/session.py:606-629).
* Transfer-only arms: the reference endpoints on its test Rig layout
  (tests/test_protocol.py:15-71): StaticSender.send + StaticReceiver.poll
  (+ the ReduceMax consumer's max), DynSender.send + DynReceiver.poll/fetch,
  and the RPC fragment ring RpcSender.start/pump + RpcReceiver.poll
  (runtime/protocol.py:257-448).
"""
from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
_CANDIDATES = (os.path.join(HERE, "_ref"), "/root/reference/pkg/src")


def reference():
    """The rdmaflow package, or None when neither copy is present."""
    if "rdmaflow" in sys.modules:
        return sys.modules["rdmaflow"]
    for path in _CANDIDATES:
        if os.path.isdir(os.path.join(path, "rdmaflow")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import rdmaflow
            return rdmaflow
    return None


def source() -> str:
    mod = reference()
    return os.path.dirname(os.path.dirname(mod.__file__)) if mod else ""


MIB = 1 << 20


class SessionArm:
    """One steady Session iteration of build_microbench(S) per step()."""

    def __init__(self, nbytes: int, mode: str = "zerocp", mechanism_override=None):
        reference()
        from rdmaflow.benchcli import ScenarioConfig, _memory_for
        from rdmaflow.runtime.session import Session
        from rdmaflow.workloads import build_microbench
        graph, placement = build_microbench(nbytes)
        capacity, arena = _memory_for(nbytes, ScenarioConfig())
        self.session = Session(graph, placement, mode=mode, seed=0, capacity_bytes=capacity,
                               arena_bytes=arena, mechanism_override=mechanism_override)
        self.session.run(1)  # iteration 1: tracing warm-up, excluded

    def step(self) -> None:
        self.session.run(1)

    def close(self) -> None:
        self.session.close()


class EndpointRig:
    """Two connected reference servers and one edge of ``nbytes`` fp32
    (tests/test_protocol.py Rig layout); step() = one transfer + consume."""

    def __init__(self, nbytes: int, mechanism: str = "static", stage_copy: bool = False,
                 seed: int = 5):
        reference()
        import numpy as np
        from rdmaflow.analyzer import PlanEntry
        from rdmaflow.fabric import Fabric
        from rdmaflow.graph import Tensor, TensorShape
        from rdmaflow.memspace import ArenaAllocator, BufferRef, MemorySpace
        from rdmaflow.runtime import protocol as P
        from rdmaflow.wire import ElemType, Mechanism, meta_block_size, static_region_size
        self.np, self.P = np, P
        cap = 4 * nbytes + 4 * MIB
        self.fabric = Fabric(seed=seed)
        self.spaces = {s: MemorySpace(s, cap, seed=s) for s in (0, 1)}
        self.arenas = {s: ArenaAllocator(sp, sp.allocate_region(cap - MIB, register=True))
                       for s, sp in self.spaces.items()}
        dev = {s: self.fabric.create_device(self.spaces[s], qps_per_peer=2) for s in (0, 1)}
        fwd = dev[0].connect(dev[1].endpoint)
        back = dev[1].channels_to(dev[0].endpoint)
        flag = self.arenas[0].alloc(1)
        self.spaces[0].write_at(flag, 0, b"\x01")
        n = nbytes // 4
        shape = TensorShape((n,))
        self.mechanism, self.stage_copy, self.nbytes = mechanism, stage_copy, nbytes
        h = self.arenas[0].alloc(max(nbytes, 1))
        vals = np.random.default_rng(42).random(n, dtype=np.float32)
        self.spaces[0].write_at(h, 0, vals.tobytes())
        self.tensor = Tensor((n,), ElemType.F32, BufferRef(h, self.arenas[0]), 0)
        if mechanism == "rpc":
            self.sender = P.RpcSender(0, 1, self.spaces[0], self.arenas[0], fwd[1])
            self.receiver = P.RpcReceiver(0, 1, self.spaces[1], self.arenas[1], self.arenas[1],
                                          back[1])
            return
        mech = Mechanism.STATIC if mechanism == "static" else Mechanism.DYNAMIC
        entry = PlanEntry(0, 0, 1, mech, shape, ElemType.F32, 1)
        size = (static_region_size((n,), ElemType.F32) if mech is Mechanism.STATIC
                else meta_block_size(1))
        buf = self.arenas[1].alloc(size)
        self.spaces[1].write_at(buf, size - 1, b"\x00")
        entry.recv_buffer = buf
        entry.remote_addr, entry.remote_token, entry.remote_len = \
            buf.base_addr, buf.access_token, buf.length
        if mech is Mechanism.STATIC:
            self.sender = P.StaticSender(entry, self.spaces[0], self.arenas[0], fwd[1], flag)
            self.receiver = P.StaticReceiver(entry, self.spaces[1])
        else:
            self.sender = P.DynSender(entry, self.spaces[0], self.arenas[0], fwd[1])
            self.receiver = P.DynReceiver(entry, self.spaces[1], self.arenas[1], back[1])

    def _consume(self, t) -> float:
        # the microbench consumer is ReduceMax (workloads.py:11-28)
        raw = self.spaces[1].read_at(t.buffer.handle, 0, self.nbytes)
        return float(self.np.frombuffer(raw, self.np.float32).max())

    def step(self) -> float:
        P = self.P
        if self.mechanism == "rpc":
            self.sender.start(self.tensor)
            got = None
            while got is None or self.sender.busy:
                self.sender.pump()
                r = self.receiver.poll()
                got = got if r is None else r
            out = self._consume(got)
            got.buffer.release()
            return out
        if self.mechanism == "static":
            self.sender.send(self.tensor, stage_copy=self.stage_copy)
            got = self.receiver.poll()
            return self._consume(got)
        self.sender.send(self.tensor, stage_copy=self.stage_copy)
        got = self.receiver.fetch(self.receiver.poll())
        out = self._consume(got)
        got.buffer.release()
        return out


class PsArm:
    """Session(PS graph).run(1) per step (configs[2]-[4]): the graph of
    build_ps_workload (workloads.py:59-94) with per-variable shapes, built
    through the reference's own DataFlowGraph API in the same node order
    (variable, then per worker gen_grad + apply_grad), variables round-robin
    over the shards; ``colocate``: shard k on worker k's server.
    The reference update is XOR (graph.py:392-405)."""

    def __init__(self, shapes, workers: int, shards: int = 1, colocate: bool = False):
        reference()
        from rdmaflow.benchcli import ScenarioConfig, _memory_for
        from rdmaflow.graph import DataFlowGraph, shape_of
        from rdmaflow.runtime.session import Session
        from rdmaflow.wire import ElemType
        g = DataFlowGraph()
        placement = {}
        for v, dims in enumerate(shapes):
            shard = (v % shards) + (0 if colocate else workers)
            w_edge = g.variable(shape_of(*dims), ElemType.F32)
            placement[g.edges[w_edge].producer] = shard
            for w in range(workers):
                grad = g.gen_grad(shape_of(*dims), ElemType.F32, inputs=(w_edge,), compute_time=0.0)
                placement[g.edges[grad].producer] = w
                upd = g.apply_grad(w_edge, grad)
                placement[g.edges[upd].producer] = shard
        g.freeze()
        biggest = max(4 * _prod(d) for d in shapes)
        total = sum(4 * _prod(d) for d in shapes)
        capacity, arena = _memory_for(max(biggest * workers * 4, MIB), ScenarioConfig())
        # registered arena: every server's variables, gradients and receive
        # regions with slack; the normal arena (capacity - arena) keeps its size
        normal = capacity - arena
        arena = max(arena, 2 * total * (workers + 1) + 16 * MIB)
        capacity = arena + normal
        self.session = Session(g, placement, mode="zerocp", seed=0, capacity_bytes=capacity,
                               arena_bytes=arena, watchdog_sweeps=10_000)
        self.session.run(1)  # iteration 1: tracing warm-up, excluded

    def step(self) -> None:
        self.session.run(1)

    def close(self) -> None:
        self.session.close()


def _prod(dims) -> int:
    n = 1
    for d in dims:
        n *= int(d)
    return n


def time_steps(step, seconds: float, min_steps: int = 2, max_steps=None):
    """(steps, elapsed s) of repeated step() calls for about ``seconds``."""
    n, t0 = 0, time.perf_counter()
    while True:
        step()
        n += 1
        dt = time.perf_counter() - t0
        if (max_steps is not None and n >= max_steps) or (dt >= seconds and n >= min_steps):
            return n, dt
