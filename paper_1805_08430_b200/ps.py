"""Parameter-server training step on B200, fully device-driven.

This is the hot loop of BASELINE.json configs[2..4]: the reference's
``Session.run`` over ``build_ps_workload`` (workloads.py:59-94,
runtime/session.py:606-629), where per iteration every variable is pushed
shard -> workers with static placement (the weight edge, analyzer.py:105-128
makes it STATIC), every worker returns a gradient with dynamic allocation
(meta write + receiver pull, the Variable-feeding rule makes it DYNAMIC), and
the shard applies the workers' gradients in ascending node order
(graph.py:507-535) in place.

On B200 the whole iteration is four kernel launches per GPU, with no host
round trip between phases (``srf_batch_*`` in include/srflow.h):

1. put batch   K1 - weight pushes, payload + tail flag, credit-gated;
2. gen batch       - each worker acquires/clears its weight flags (the
                     StaticReceiver poll) and produces its gradient (device
                     RNG stand-in for GenGrad, or host-uploaded PCG64 values in
                     parity mode);
3. put batch   K3 - the 8D+33-byte metadata blocks, byte-identical to
                     ``encode_meta``, into the shards' fixed slots;
4. apply batch K4+K6 - the shard decodes each meta block on the device,
                     validates token/bounds/length, and folds every worker's
                     gradient straight from the peer pool (XOR = the
                     reference's bit-exact update, or SGD) - the pull and the
                     update fused, so no gradient copy lands in shard HBM.

Servers follow the reference placement: workers ``0..W-1``; shard k is server
``W + k`` or, with ``colocate``, server k (the paper's deployment).  A server
lives on rank ``server % world``; all of a rank's servers share its GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib, errors
from .graph import node_rng, synthesize_values
from .memspace import ArenaAllocator, MemorySpace
from .wire import ElemType, encode_meta, meta_block_size
from .workloads import ps_node_ids

_NONE = (1 << 64) - 1


#: block alignment (power of two >= 32; SRFLOW_PS_ALIGN for experiments).
#: 256 B keeps every warp's 32-B vectors inside whole 128-B lines of a peer's
#: pool: the fused pull + apply went 643 -> 748 GB/s over NVLink at N=2 vs 32 B
#: (profiles/r1_ps_phase_probe.jsonl)
_BLOCK_ALIGN = int(os.environ.get("SRFLOW_PS_ALIGN", "256"))


def _r16(n: int) -> int:
    """Block size rounded to the block alignment (>= 32 B, so blocks stay
    co-aligned for 32-B vectors)."""
    return (n + _BLOCK_ALIGN - 1) & ~(_BLOCK_ALIGN - 1)


@dataclass
class PsLayout:
    """Deterministic per-server memory layout (pure host logic).

    Every block is a 256-B aligned slice of the server's one registered arena,
    allocated in a fixed order, so every rank can derive every peer's
    coordinates; the exchanged region tables (tokens) validate them.
    """

    shapes: list[tuple[int, ...]]
    workers: int
    shards: int
    colocate: bool = False
    elem: ElemType = ElemType.F32
    #: "round_robin" = the reference placement v % shards (workloads.py:84);
    #: "bytes" = extension: largest variable first onto the least-loaded shard
    placement: str = "round_robin"
    #: EXTENSION (partitioned variables, as MXNet's kvstore splits big arrays
    #: over servers): a variable larger than this many bytes is cut into
    #: ``shards`` contiguous slices, each its own transfer unit on its own
    #: shard.  Updates are elementwise and gradients are generated per global
    #: element index, so the model's values are bit-identical to unpartitioned.
    partition_bytes: Optional[int] = None
    #: EXTENSION (pipelined transfers): a unit larger than this many bytes is
    #: cut into consecutive slices of about this size that all stay on the
    #: unit's shard (the placement is unchanged), each with its own flag,
    #: metadata block and apply, so slice j's pull and update overlap slice
    #: j+1's push instead of waiting for the whole tensor.  Values are
    #: bit-identical (elementwise update, per-element gradient streams).
    slice_bytes: Optional[int] = None
    #: gradient edges' transfer mechanism: "dynamic" is what the reference's
    #: analyzer picks (metadata block + one-sided pull, analyzer.py); "static"
    #: is its ``mechanism_override="static"`` (runtime/session.py:368): the
    #: worker puts the gradient + flag into a preallocated receive region on
    #: the shard (K1), and the apply reads it there.  Same values either way.
    grad_mechanism: str = "dynamic"
    blocks: dict[int, dict] = field(default_factory=dict)
    sizes: dict[int, int] = field(default_factory=dict)

    def __post_init__(self):
        self.model_shapes = [tuple(int(d) for d in s) for s in self.shapes]
        if self.colocate and self.shards > self.workers:
            raise errors.InvalidConfig("colocate needs shards <= workers")
        if self.workers > _lib.MAX_WORKERS:
            raise errors.InvalidConfig(f"at most {_lib.MAX_WORKERS} workers")
        if self.grad_mechanism not in ("dynamic", "static"):
            raise errors.InvalidConfig(f"unknown gradient mechanism {self.grad_mechanism!r}")
        # transfer units: (model variable, first element, elements, slice index)
        units = []
        esz = self.elem.size
        for v, dims in enumerate(self.model_shapes):
            n = math.prod(dims)
            if self.partition_bytes is not None and n * esz > self.partition_bytes \
                    and self.shards > 1:
                step = -(-n // self.shards)
                step = (step + 63) // 64 * 64          # 256-B slices
                for j, off in enumerate(range(0, n, step)):
                    units.append((v, off, min(step, n - off), j))
            else:
                units.append((v, 0, n, -1))
        if self.placement == "round_robin":
            # slice j of variable v on shard (v + j) % shards
            shard = [(v + max(j, 0)) % self.shards for v, _o, _c, j in units]
        elif self.placement == "bytes":
            load = [0] * self.shards
            shard = [0] * len(units)
            for u in sorted(range(len(units)), key=lambda u: (-units[u][2], u)):
                k = min(range(self.shards), key=lambda k: (load[k], k))
                shard[u] = k
                load[k] += units[u][2] * esz
        else:
            raise errors.InvalidConfig(f"unknown placement {self.placement!r}")
        # transfer units: (model variable, first element, elements, slice index)
        self.units, self._shard = [], []
        for (v, off, n, j), k in zip(units, shard):
            if self.slice_bytes is not None and n * esz > self.slice_bytes:
                step = max(64, self.slice_bytes // esz // 64 * 64)   # 256-B multiples
                for i, o in enumerate(range(off, off + n, step)):
                    self.units.append((v, o, min(step, off + n - o), max(j, 0) * 1024 + i))
                    self._shard.append(k)
            else:
                self.units.append((v, off, n, j))
                self._shard.append(k)
        self.shapes = [self.model_shapes[v] if j < 0 else (cnt,)
                       for v, _off, cnt, j in self.units]
        for s in range(self.nservers):
            self._lay_out(s)

    @property
    def nservers(self) -> int:
        return self.workers if self.colocate else self.workers + self.shards

    def nbytes(self, v: int) -> int:
        return math.prod(self.shapes[v]) * self.elem.size

    def parent(self, u: int) -> tuple[int, int, int]:
        """(model variable, first element, elements) of transfer unit u."""
        v, off, n, _j = self.units[u]
        return v, off, n

    def node_ids(self, u: int, w: int) -> tuple[int, int, int]:
        """Reference node ids (variable, GenGrad, ApplyGrad) of unit u's model
        variable for worker w (workloads.py:81-93)."""
        return ps_node_ids(len(self.model_shapes), self.workers, self.units[u][0], w)

    def shard_of(self, v: int) -> int:
        return self._shard[v] + (0 if self.colocate else self.workers)

    def is_worker(self, s: int) -> bool:
        return s < self.workers

    def _lay_out(self, s: int) -> None:
        off = 0
        b: dict = {}

        def take(key, n):
            nonlocal off
            b[key] = off
            off += _r16(n)

        take("flag", 1)
        for v in range(len(self.shapes)):
            if self.shard_of(v) == s:
                take(("var", v), self.nbytes(v))
                if self.is_worker(s):  # co-located: the in-place gradient's ready byte
                    take(("ready", v), 1)
        static = self.grad_mechanism == "static"
        if self.is_worker(s):
            for v in range(len(self.shapes)):
                take(("grad", v), self.nbytes(v))
                if self.shard_of(v) != s:
                    take(("wbuf", v), self.nbytes(v) + 1)
                    if static:   # gradient complete / copied out (gen <-> push)
                        take(("ready", v), 1)
                    else:
                        take(("mstage", v), meta_block_size(len(self.shapes[v])))
        for v in range(len(self.shapes)):
            if self.shard_of(v) == s:
                for w in range(self.workers):
                    if w != s:
                        if static:   # the static gradient receive region (payload || flag)
                            take(("grecv", v, w), self.nbytes(v) + 1)
                        else:
                            take(("mslot", v, w), meta_block_size(len(self.shapes[v])))
        self.blocks[s] = b
        self.sizes[s] = off

    def grad_signal_bytes(self, v: int) -> int:
        """Bytes besides the payload a gradient edge moves: the metadata block
        (dynamic) or the tail flag (static)."""
        return 1 if self.grad_mechanism == "static" else meta_block_size(len(self.shapes[v]))

    def traffic(self, s: int) -> dict:
        """Algorithmic bytes per iteration at server s.

        ``link_out``/``link_in``: bytes leaving/entering s over NVLink - weight
        pushes out of a shard, gradient reads a shard makes from worker pools
        (they leave the worker), metadata blocks.  ``hbm``: local bytes of the
        update (variable read + write, co-located gradient) and gradient
        production."""
        out = {"push_out": 0, "meta_out": 0, "pull_in": 0, "link_out": 0, "link_in": 0,
               "hbm": 0}
        for v in range(len(self.shapes)):
            S = self.nbytes(v)
            meta = self.grad_signal_bytes(v)
            sh = self.shard_of(v)
            if sh == s:
                remote = [w for w in range(self.workers) if w != s]
                out["push_out"] += len(remote) * (S + 1)
                out["pull_in"] += len(remote) * S
                out["link_out"] += len(remote) * (S + 1)
                out["link_in"] += len(remote) * (S + meta)
                out["hbm"] += 2 * S + (self.workers - len(remote)) * S
            if self.is_worker(s):
                out["hbm"] += S  # gradient produced
                if sh != s:
                    out["meta_out"] += meta
                    out["link_out"] += meta + S   # meta written, gradient read by the shard
                    out["link_in"] += S + 1       # weight pushed in
        return out


def link_traffic(L: "PsLayout", world: int) -> dict[int, dict]:
    """NVLink bytes per iteration per GPU (server s on GPU s % world); traffic
    between servers on the same GPU stays in HBM and is not counted."""
    out = {g: {"link_out": 0, "link_in": 0} for g in range(world)}
    for v in range(len(L.shapes)):
        S = L.nbytes(v)
        meta = L.grad_signal_bytes(v)
        s = L.shard_of(v)
        for w in range(L.workers):
            if w == s or w % world == s % world:
                continue
            gs, gw = s % world, w % world
            out[gs]["link_out"] += S + 1          # weight push
            out[gw]["link_in"] += S + 1
            out[gw]["link_out"] += meta + S       # metadata write + gradient read
            out[gs]["link_in"] += meta + S
    return out


class PsStep:
    """The device-resident PS exchange of one rank (see module docstring)."""

    def __init__(self, layout: PsLayout, *, rank: int = 0, world: int = 1, device: int = 0,
                 seed: int = 0, op: str = "xor", lr: float = 0.01,
                 schedule: str = "phases",
                 exchange_lag: Optional[int] = None, exchange_order: Optional[str] = None,
                 fuse_push: bool = False):
        self.L = layout
        self.rank, self.world, self.device = rank, world, device
        self.seed = seed
        self.op = {"xor": _lib.APPLY_XOR, "sgd": _lib.APPLY_SGD}[op]
        self.lr = float(lr)
        self.static_grads = layout.grad_mechanism == "static"
        self.local = [s for s in range(layout.nservers) if s % world == rank]
        self.spaces: dict[int, MemorySpace] = {}
        self.regions = {}
        for s in self.local:
            size = layout.sizes[s]
            sp = MemorySpace(s, size + (1 << 20), seed=seed, device=device)
            reg = sp.allocate_region(size, register=True)
            arena = ArenaAllocator(sp, reg)
            # allocate the layout's blocks in order: first fit == bump here
            for key, off in sorted(layout.blocks[s].items(), key=lambda kv: kv[1]):
                h = arena.alloc(_r16(self._block_len(s, key)))
                if h.base_addr != reg.base_addr + off:
                    raise AssertionError(f"layout drift at {key}")
            self.spaces[s] = sp
            self.regions[s] = reg
        self.peers: dict[int, MemorySpace] = {}
        if world > 1:
            table = gather_descriptors_all(self.spaces)
            for s, desc in table.items():
                if s not in self.spaces:
                    proxy = MemorySpace.import_remote(desc, device)
                    self.peers[s] = proxy
                    rid, base, length, reg_, tok = desc["regions"][0]
                    self.regions[s] = _Reg(base, length, tok)
        for a in self.spaces.values():
            for b in list(self.spaces.values()) + list(self.peers.values()):
                _lib.call("srf_connect", a.handle, b.handle)
        self._init_memory()
        if world > 1:
            # no peer may write into this rank's pools before they are set up
            import torch.distributed as dist
            dist.barrier()
        # a rank hosting no server of this layout still joins the collectives;
        # it gets a 1 MiB scratch pool only to own a stream
        self.stream_space = (self.spaces[self.local[0]] if self.local else
                             MemorySpace(-1 - rank, 1 << 20, seed=seed, device=device))
        self.stream = C.c_void_p()
        _lib.call("srf_stream_create", self.stream_space.handle, C.byref(self.stream))
        # device iteration counter for graph-replayed steps
        self._counter = self.stream_space.allocate_region(64)
        self._exchange_push = None
        self.batches = self._build_batches()
        for g in self.batches["gen"].values():
            _lib.call("srf_batch_set_iteration_source", g, self.stream_space.handle,
                      self._counter.base_addr)
        self._exchange = None
        self._exchange_built = None
        self._exchange_nopush = None
        self._exchange_gpush = None
        self._exchange_cfg = (
            int(os.environ.get("SRFLOW_PS_EXCHANGE_LAG", 3) if exchange_lag is None
                else exchange_lag),
            (os.environ.get("SRFLOW_PS_EXCHANGE_ORDER", "size") if exchange_order is None
             else exchange_order))
        self.schedule = "phases"
        #: EXTENSION (fused weight push, phase schedule): the apply of
        #: iteration k also stores the updated variable into every remote
        #: worker's weight receive region and releases its flag - the weight
        #: Send of iteration k+1 without re-reading the variable.  Toggle
        #: between steps; while a forwarded push is outstanding the next
        #: step skips its push batch.
        self.fuse_push = bool(fuse_push)
        self._pushed_ahead = False
        self._set_forward()
        self.use_schedule(schedule)

    # -- layout helpers -------------------------------------------------------------

    def _block_len(self, s: int, key) -> int:
        kind = key if isinstance(key, str) else key[0]
        if kind in ("flag", "ready"):
            return 1
        v = key[1]
        if kind in ("var", "grad"):
            return self.L.nbytes(v)
        if kind in ("wbuf", "grecv"):
            return self.L.nbytes(v) + 1
        return meta_block_size(len(self.L.shapes[v]))

    def space(self, s: int) -> MemorySpace:
        return self.spaces.get(s) or self.peers[s]

    def addr(self, s: int, key) -> int:
        return self.regions[s].base_addr + self.L.blocks[s][key]

    def token(self, s: int) -> int:
        return self.regions[s].access_token

    # -- initial state ------------------------------------------------------------------

    def _init_memory(self) -> None:
        L = self.L
        for s, sp in self.spaces.items():
            sp.write_raw(self.addr(s, "flag"), b"\x01")
            for v in range(len(L.shapes)):
                if L.shard_of(v) == s:
                    sp.write_raw(self.addr(s, ("var", v)), self._model_slice(v, 0, 0))
                    for w in range(L.workers):
                        if w != s and self.static_grads:
                            sp.write_raw(self.addr(s, ("grecv", v, w)) + L.nbytes(v), b"\x00")
                        elif w != s:
                            mk = ("mslot", v, w)
                            sp.write_raw(self.addr(s, mk) + meta_block_size(len(L.shapes[v])) - 1,
                                         b"\x00")
                if L.is_worker(s) and L.shard_of(v) != s:
                    sp.write_raw(self.addr(s, ("wbuf", v)) + L.nbytes(v), b"\x00")
                    if self.static_grads:
                        sp.write_raw(self.addr(s, ("ready", v)), b"\x00")
                        continue
                    meta = encode_meta(L.shapes[v], L.elem, self.addr(s, ("grad", v)), self.token(s))
                    sp.write_raw(self.addr(s, ("mstage", v)), meta)
            sp.sync()

    def _model_slice(self, u: int, kind: int, iteration: int) -> np.ndarray:
        """Unit u's slice of its model variable's initial value (kind 0) or of
        worker w=kind-1's reference PCG64 gradient (graph.py:333-350)."""
        L = self.L
        v, off, n = L.parent(u)
        node = (L.node_ids(u, 0)[0] if kind == 0 else L.node_ids(u, kind - 1)[1])
        key = (v, node, iteration)
        cache = self.__dict__.setdefault("_slice_cache", {})
        if key not in cache:
            cache.clear()
            cache[key] = synthesize_values(L.model_shapes[v], L.elem,
                                           node_rng(self.seed, node, iteration)).reshape(-1)
        return cache[key][off:off + n].reshape(L.shapes[u])

    def _build_batches(self) -> dict:
        L = self.L
        P, u64 = C.c_void_p, _lib.u64_array
        out = {}
        # variable of every edge, per batch (exchange keys)
        self._rows = {"push": [], "gen": [], "meta": [], "apply": {}}
        # 1. weight pushes (K1), credit-gated
        rows = []
        for s in self.local:
            for v in range(len(L.shapes)):
                if L.shard_of(v) != s:
                    continue
                for w in range(L.workers):
                    if w == s:
                        continue
                    rows.append((s, self.addr(s, ("var", v)), L.nbytes(v), self.token(s),
                                 self.addr(s, "flag"), w, self.addr(w, ("wbuf", v)), self.token(w)))
                    self._rows["push"].append(v)
        out["push"] = self._put_batch(rows, _lib.PUT_WAIT_EMPTY)
        # 2. worker gen batch
        g_rows = []
        for w in self.local:
            if not L.is_worker(w):
                continue
            for v in range(len(L.shapes)):
                sh = L.shard_of(v)
                remote = sh != w
                mlen = meta_block_size(len(L.shapes[v]))
                g_rows.append((self.addr(w, ("grad", v)), L.nbytes(v),
                               self.addr(w, ("wbuf", v)) + L.nbytes(v) if remote else _NONE,
                               self.space(sh).handle.value if remote and not self.static_grads
                               else None,
                               self.addr(sh, ("mslot", v, w)) + mlen - 1
                               if remote and not self.static_grads else _NONE,
                               L.node_ids(v, w)[1], w))
                self._rows["gen"].append((w, v))
        out["gen"] = {}
        if g_rows:
            b = C.c_void_p()
            n = len(g_rows)
            _lib.call("srf_batch_gen_create", n,
                      (P * n)(*[self.spaces[r[-1]].handle.value for r in g_rows]),
                      u64(r[0] for r in g_rows), u64(r[1] for r in g_rows),
                      u64(r[2] for r in g_rows), (P * n)(*[r[3] for r in g_rows]),
                      u64(r[4] for r in g_rows), u64(r[5] for r in g_rows), self.seed,
                      C.byref(b))
            ready = [self.addr(w, ("ready", v)) if L.shard_of(v) == w or self.static_grads
                     else _NONE for w, v in self._rows["gen"]]
            if any(r != _NONE for r in ready):
                _lib.call("srf_batch_gen_set_ready", b,
                          (P * n)(*[self.spaces[w].handle.value for w, _v in self._rows["gen"]]),
                          u64(ready))
            offs = [L.parent(v)[1] for _w, v in self._rows["gen"]]
            if any(offs):  # partitioned variables: slices keep global element indices
                _lib.call("srf_batch_gen_set_offsets", b, u64(offs))
            out["gen"]["all"] = b
        self._push_rows = rows_push = rows
        # 3. metadata writes (K3), or the static gradient pushes (K1)
        rows = []
        self._rows["gpush"] = []
        for w in self.local:
            if not L.is_worker(w):
                continue
            for v in range(len(L.shapes)):
                sh = L.shard_of(v)
                if sh == w:
                    continue
                if self.static_grads:
                    rows.append((w, self.addr(w, ("grad", v)), L.nbytes(v), self.token(w),
                                 self.addr(w, "flag"), sh, self.addr(sh, ("grecv", v, w)),
                                 self.token(sh)))
                    self._rows["gpush"].append((w, v))
                    continue
                mlen = meta_block_size(len(L.shapes[v]))
                rows.append((w, self.addr(w, ("mstage", v)), mlen - 1, self.token(w),
                             self.addr(w, ("mstage", v)) + mlen - 1, sh,
                             self.addr(sh, ("mslot", v, w)), self.token(sh)))
                self._rows["meta"].append((w, v))
        out["gpush"] = None
        self._gpush_rows = rows
        if self.static_grads:
            out["meta"] = None
            out["gpush"] = self._put_batch(rows, _lib.PUT_WAIT_EMPTY)
            if rows:
                self._set_src_ready(out["gpush"], self._rows["gpush"])
        else:
            out["meta"] = self._put_batch(rows, 0)
        del rows_push
        # 4. fused pull + apply per shard
        out["apply"] = {}
        for s in self.local:
            vs = [v for v in range(len(L.shapes)) if L.shard_of(v) == s]
            if not vs:
                continue
            self._rows["apply"][s] = vs
            out["apply"][s] = self._make_apply(s, [(v, list(range(L.workers))) for v in vs])
        return out

    def _set_forward(self) -> None:
        """Forward destinations of every apply descriptor: the weight receive
        regions the variable's push rows write (same workers, same order)."""
        L = self.L
        for s, a in self.batches["apply"].items():
            nfwd, sp, ad, tok = [], [], [], []
            for v in self._rows["apply"][s]:
                ws = [w for w in range(L.workers) if w != s and L.shard_of(v) == s]
                nfwd.append(len(ws))
                for w in ws:
                    sp.append(self.space(w).handle.value)
                    ad.append(self.addr(w, ("wbuf", v)))
                    tok.append(self.token(w))
            if not any(nfwd):
                continue
            n = len(nfwd)
            _lib.call("srf_batch_apply_set_forward", a, (C.c_int * n)(*nfwd),
                      (C.c_void_p * len(sp))(*sp), _lib.u64_array(ad), _lib.u64_array(tok),
                      self.spaces[s].handle, self.addr(s, "flag"))

    def _check_unfused(self, what: str) -> None:
        if self._pushed_ahead:
            raise errors.InvalidConfig(
                f"{what}: a fused weight push is outstanding; run one step with "
                f"fuse_push=False first")

    def _make_apply(self, s: int, groups) -> C.c_void_p:
        """One apply batch on shard s: a descriptor per (variable, workers)
        group, the workers' gradients applied in the listed (ascending) order."""
        L = self.L
        P, u64 = C.c_void_p, _lib.u64_array
        srcsp, srcad, ismeta, peersp, lo, hi, tok, ready = [], [], [], [], [], [], [], []
        for v, ws in groups:
            for w in ws:
                if w == s:
                    srcsp.append(self.spaces[s].handle.value)
                    srcad.append(self.addr(s, ("grad", v)))
                    ismeta.append(0)
                    peersp.append(self.spaces[s].handle.value)
                    lo.append(0), hi.append(0), tok.append(0)
                    ready.append(self.addr(s, ("ready", v)) if L.is_worker(s) else _NONE)
                elif self.static_grads:
                    # StaticReceiver: the gradient landed in s's receive region;
                    # its tail flag is the apply's ready byte (cleared = credit)
                    srcsp.append(self.spaces[s].handle.value)
                    srcad.append(self.addr(s, ("grecv", v, w)))
                    ismeta.append(0)
                    peersp.append(self.spaces[s].handle.value)
                    lo.append(0), hi.append(0), tok.append(0)
                    ready.append(self.addr(s, ("grecv", v, w)) + L.nbytes(v))
                else:
                    srcsp.append(self.spaces[s].handle.value)
                    srcad.append(self.addr(s, ("mslot", v, w)))
                    ismeta.append(1)
                    peersp.append(self.space(w).handle.value)
                    r = self.regions[w]
                    lo.append(r.base_addr), hi.append(r.base_addr + r.length)
                    tok.append(r.access_token)
                    ready.append(_NONE)
        n = len(groups)
        b = C.c_void_p()
        ints = C.c_int * n
        _lib.call("srf_batch_apply_create", self.spaces[s].handle, n,
                  u64(self.addr(s, ("var", v)) for v, _ws in groups),
                  u64(L.nbytes(v) for v, _ws in groups),
                  ints(*[len(ws) for _v, ws in groups]),
                  ints(*[len(L.shapes[v]) for v, _ws in groups]),
                  (P * len(srcsp))(*srcsp), u64(srcad), (C.c_int * len(ismeta))(*ismeta),
                  (P * len(peersp))(*peersp), u64(lo), u64(hi), u64(tok), self.op,
                  self.lr, C.byref(b))
        if any(r != _NONE for r in ready):
            _lib.call("srf_batch_apply_set_ready", b, self.spaces[s].handle, u64(ready))
        return b

    def _set_src_ready(self, batch, wv) -> None:
        """Put edge i waits for its gradient's ready byte (wv[i] = (worker,
        variable); None: no source gate)."""
        P = C.c_void_p
        anyw = next(x for x in wv if x is not None)[0]
        _lib.call("srf_batch_put_set_src_ready", batch,
                  (P * len(wv))(*[self.spaces[anyw if x is None else x[0]].handle.value
                                  for x in wv]),
                  _lib.u64_array(_NONE if x is None else self.addr(x[0], ("ready", x[1]))
                                 for x in wv))

    def _put_batch(self, rows, flags):
        if not rows:
            return None
        P, u64 = C.c_void_p, _lib.u64_array
        b = C.c_void_p()
        n = len(rows)
        _lib.call("srf_batch_put_create", n,
                  (P * n)(*[self.space(r[0]).handle.value for r in rows]),
                  u64(r[1] for r in rows), u64(r[2] for r in rows), u64(r[3] for r in rows),
                  u64(r[4] for r in rows), (P * n)(*[self.space(r[5]).handle.value for r in rows]),
                  u64(r[6] for r in rows), u64(r[7] for r in rows), flags, C.byref(b))
        return b

    def use_schedule(self, schedule: str) -> None:
        """Switch between the per-phase launches and the exchange launch (both
        use the same flags and credits, so they can alternate step by step)."""
        if schedule not in ("phases", "exchange"):
            raise errors.InvalidConfig(f"unknown PS schedule {schedule!r}")
        if schedule == "exchange":
            b = self.batches
            if self._exchange_built is None and (b["push"] is not None or b["gen"]
                                                 or b["apply"]):
                self._exchange_built = self._build_exchange(*self._exchange_cfg)
            # (a rank hosting no server of the layout has nothing to launch)
            self._exchange = self._exchange_built
        else:
            self._exchange = None
        self.schedule = schedule

    def set_exchange_config(self, lag: int, order: str) -> None:
        """Rebuild the exchange schedules with another apply lag / unit order
        (the next exchange launch builds them; the phase schedule is
        unaffected).  Call between steps."""
        self.sync()
        for x in (self._exchange_built, self._exchange_nopush):
            if x is not None:
                _lib.call("srf_ps_exchange_destroy", x)
        was = self.schedule
        self._exchange = self._exchange_built = self._exchange_nopush = None
        self._exchange_cfg = (int(lag), order)
        if was == "exchange":
            self.use_schedule("exchange")

    def _exchange_for_launch(self) -> tuple:
        """(exchange object, mode bits) for the next exchange launch, and
        whether this rank must first push (the fused schedule's prologue).
        With weights already forwarded (a fused step before) or fusion on,
        the exchange without weight pushes runs; the applies forward iff
        fusion is on."""
        if self._exchange is None:
            return None, 0, False
        if not (self.fuse_push or self._pushed_ahead) or self.batches["push"] is None:
            return self._exchange, 0, False
        if self._exchange_nopush is None:
            self._exchange_nopush = self._build_exchange(*self._exchange_cfg, nopush=True)
        return (self._exchange_nopush, 2 if self.fuse_push else 0,
                self.fuse_push and not self._pushed_ahead)

    def _build_exchange(self, lag: int, order: str, nopush: bool = False):
        """One queue of this GPU's units (k_ps_exchange).  Keys are a global
        order every rank derives alike: push(v) < gen(v) < apply(v), the
        apply of a variable placed ``lag`` variables later so the next
        weights are already moving while its gradients are awaited; static
        gradient puts sit between gen(v) and apply(v).  Defaults (largest
        variable first, lag 3) from profiles/r1_ps_order_probe.jsonl."""
        L, b, rows = self.L, self.batches, self._rows
        u64 = _lib.u64_array
        nv = len(L.shapes)
        if order == "index":
            seq = list(range(nv))
        elif order == "size":  # largest first: the longest push -> pull chain starts first
            seq = sorted(range(nv), key=lambda v: (-L.nbytes(v), v))
        else:
            raise errors.InvalidConfig(f"unknown exchange order {order!r}")
        pos = {v: i for i, v in enumerate(seq)}
        gen = next(iter(b["gen"].values()), None)
        if b["meta"] is not None:
            index = {wv: i for i, wv in enumerate(rows["gen"])}
            gi = (C.c_int * len(rows["meta"]))(*[index[wv] for wv in rows["meta"]])
            _lib.call("srf_batch_gen_set_meta", gen, len(rows["meta"]), gi, b["meta"])
        applies = list(b["apply"].items())
        push, push_vars = b["push"], list(rows["push"])
        push_keys = [4 * pos[v] for v in rows["push"]]
        if nopush:    # fused weight push: the applies write the weights
            push, push_vars, push_keys = None, [], []
        apply_slot = 2
        if self.static_grads and self._gpush_rows and nopush:
            push = self._exchange_gpush = self._put_batch(self._gpush_rows, _lib.PUT_WAIT_EMPTY)
            self._set_src_ready(push, rows["gpush"])
            push_keys = [4 * pos[v] + 2 for _w, v in rows["gpush"]]
            push_vars = [None] * len(rows["gpush"])
            apply_slot = 3
        elif self.static_grads and self._gpush_rows:
            # static gradients: the weight pushes and the gradient pushes (after
            # their gen, before their apply) share the exchange's one put batch
            push = self._exchange_push = self._put_batch(self._push_rows + self._gpush_rows,
                                                         _lib.PUT_WAIT_EMPTY)
            self._set_src_ready(push, [None] * len(self._push_rows) + rows["gpush"])
            push_keys += [4 * pos[v] + 2 for _w, v in rows["gpush"]]
            push_vars += [None] * len(rows["gpush"])
            apply_slot = 3
        x = C.c_void_p()
        _lib.call("srf_ps_exchange_create",
                  push, u64(push_keys) if push_keys else None,
                  gen, u64(4 * pos[v] + 1 for _w, v in rows["gen"]) if rows["gen"] else None,
                  (C.c_void_p * max(1, len(applies)))(*[a.value for _s, a in applies]),
                  len(applies),
                  u64(4 * (pos[v] + lag) + apply_slot for s, _a in applies
                      for v in rows["apply"][s])
                  if applies else None,
                  C.byref(x))
        if push_vars:
            # weight push edge -> its variable's apply descriptor (global order
            # over the apply batches), for launches of several iterations
            index, base = {}, 0
            for s_, _a in applies:
                for i, v in enumerate(rows["apply"][s_]):
                    index[v] = base + i
                base += len(rows["apply"][s_])
            link = (C.c_int * len(push_vars))(*[-1 if v is None else index.get(v, -1)
                                                for v in push_vars])
            _lib.call("srf_ps_exchange_link", x, link)
        return x

    # -- running --------------------------------------------------------------------------

    def step(self, iteration: int, regen: bool = True) -> int:
        """Queue one PS iteration; returns the number of kernel launches."""
        b, n = self.batches, 0
        mode = 1 if regen else 0
        if self._exchange is not None:
            x, bits, prologue = self._exchange_for_launch()
            if prologue:
                _lib.call("srf_batch_launch", b["push"], self.stream, iteration, 0, 0)
                n += 1
            _lib.call("srf_ps_exchange_launch", x, self.stream, iteration, mode | bits)
            self._pushed_ahead = self.fuse_push and b["push"] is not None
            return n + 1
        if b["push"] is not None and not self._pushed_ahead:
            _lib.call("srf_batch_launch", b["push"], self.stream, iteration, 0, 0)
            n += 1
        for g in b["gen"].values():
            _lib.call("srf_batch_launch", g, self.stream, iteration, mode, 0)
            n += 1
        for m in (b["meta"], b["gpush"]):
            if m is not None:
                _lib.call("srf_batch_launch", m, self.stream, iteration, 0, 0)
                n += 1
        fwd = 1 if self.fuse_push else 0
        for a in b["apply"].values():
            _lib.call("srf_batch_launch", a, self.stream, iteration, fwd, 0)
            n += 1
        self._pushed_ahead = self.fuse_push and b["push"] is not None
        return n

    def launches_per_step(self) -> int:
        if self._exchange is not None:
            return 1
        b = self.batches
        return ((b["push"] is not None) + len(b["gen"]) + (b["meta"] is not None)
                + (b["gpush"] is not None) + len(b["apply"]))

    def capture(self, steps: int, regen: bool = True):
        """A CUDA graph of ``steps`` iterations on self.stream; the gen batch
        reads the iteration from the device counter, which each captured step
        advances (set the first value with :meth:`set_iteration`)."""
        if self._exchange is not None:
            raise errors.InvalidConfig("graph capture uses the one-stream phase schedule")
        none = (1 << 64) - 1
        graph = C.c_void_p()
        b = self.batches
        fwd = 1 if self.fuse_push else 0
        if fwd and b["push"] is not None and not self._pushed_ahead:
            # the fused push's prologue runs before the graph: every captured
            # step then finds its weights already forwarded
            _lib.call("srf_batch_launch", b["push"], self.stream, none, 0, 0)
            self._pushed_ahead = True
        elif not fwd:
            self._check_unfused("an unfused capture")
        _lib.call("srf_graph_begin", self.stream)
        for _ in range(steps):
            if b["push"] is not None and not fwd:
                _lib.call("srf_batch_launch", b["push"], self.stream, none, 0, 0)
            for g in b["gen"].values():
                _lib.call("srf_batch_launch", g, self.stream, none, 1 if regen else 0, 0)
            for m in (b["meta"], b["gpush"]):
                if m is not None:
                    _lib.call("srf_batch_launch", m, self.stream, none, 0, 0)
            for a in b["apply"].values():
                _lib.call("srf_batch_launch", a, self.stream, none, fwd, 0)
            _lib.call("srf_counter_add", self.stream_space.handle, self._counter.base_addr, 1,
                      self.stream)
        _lib.call("srf_graph_end", self.stream, C.byref(graph))
        return graph

    def run_exchange(self, first_iteration: int, iterations: int, regen: bool = True,
                     per_launch: int = 64) -> int:
        """``iterations`` PS iterations as exchange launches of up to
        ``per_launch`` iterations each (the unit queue repeats inside one
        launch; a push of iteration k waits for its variable's apply of
        iteration k-1).  Returns the number of launches."""
        self.use_schedule("exchange")
        n, it = 0, first_iteration
        if self._pushed_ahead and not self.fuse_push and iterations > 0:
            n += self.step(it, regen)   # consumes the forwarded weights (no push)
            it += 1
            iterations -= 1
        while iterations > 0:
            k = min(per_launch, iterations)
            x, bits, prologue = self._exchange_for_launch()
            if prologue:
                _lib.call("srf_batch_launch", self.batches["push"], self.stream, it, 0, 0)
                n += 1
            if x is not None:
                _lib.call("srf_ps_exchange_launch_n", x, self.stream, it, k,
                          (1 if regen else 0) | bits)
                n += 1
            self._pushed_ahead = self.fuse_push and self.batches["push"] is not None
            it += k
            iterations -= k
        return n

    def run_persistent(self, first_iteration: int, iterations: int, regen: bool = True) -> None:
        """``iterations`` PS iterations in one cooperative launch (every server
        of the layout on this GPU, world == 1): phases separated by grid-wide
        barriers instead of kernel boundaries."""
        if self.world != 1:
            raise errors.InvalidConfig("the persistent PS step runs on one GPU")
        if self.fuse_push:
            raise errors.InvalidConfig("the fused weight push runs in the phase schedule")
        self._check_unfused("the persistent schedule")
        b = self.batches
        applies = list(b["apply"].values())
        gen = next(iter(b["gen"].values()), None)
        _lib.call("srf_ps_persistent", b["push"], gen,
                  b["meta"] if b["meta"] is not None else b["gpush"],
                  (C.c_void_p * max(1, len(applies)))(*[a.value for a in applies]),
                  len(applies), self.stream, first_iteration, iterations,
                  1 if regen else 0)

    def set_iteration(self, iteration: int) -> None:
        self.sync()
        self.stream_space.write_at(self._counter, 0, np.array([iteration], dtype="<u8"))

    def replay(self, graph) -> int:
        _lib.call("srf_graph_launch", graph, self.stream)
        return 0

    def fork(self) -> None:
        """(Timing helper; every schedule runs on self.stream.)"""

    def join(self) -> None:
        """(Timing helper; every schedule runs on self.stream.)"""

    def sync(self) -> None:
        _lib.call("srf_stream_sync", self.stream)
        for sp in self.spaces.values():
            sp.sync()

    def upload_gradients(self, iteration: int) -> None:
        """Parity mode: this iteration's gradients from the reference's PCG64
        stream (graph.py:333-350).  Call only after a barrier (no step in
        flight)."""
        L = self.L
        for w in self.local:
            if not L.is_worker(w):
                continue
            for v in range(len(L.shapes)):
                g = self._model_slice(v, w + 1, iteration)
                self.spaces[w].write_raw(self.addr(w, ("grad", v)), g)
            self.spaces[w].sync()

    def variable(self, v: int) -> np.ndarray:
        s = self.L.shard_of(v)
        raw = self.spaces[s].read_raw(self.addr(s, ("var", v)), self.L.nbytes(v))
        return np.frombuffer(raw, dtype=self.L.elem.np_dtype).reshape(self.L.shapes[v])

    def close(self) -> None:
        self.sync()
        for x in (self._exchange_built, self._exchange_nopush):
            if x is not None:
                _lib.call("srf_ps_exchange_destroy", x)
        self._exchange = self._exchange_built = self._exchange_nopush = None
        for b in [self.batches["push"], self.batches["meta"], self.batches["gpush"],
                  self._exchange_push, self._exchange_gpush, *self.batches["gen"].values(),
                  *self.batches["apply"].values()]:
            if b is not None:
                _lib.load().srf_batch_destroy(b)
        _lib.call("srf_stream_destroy", self.stream)
        # pools: every rank stops touching its peers' pools before any is freed
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
        for sp in self.peers.values():
            sp.close()
        if self.world > 1:
            dist.barrier()
        if self.stream_space not in self.spaces.values():
            self.stream_space.close()
        for sp in self.spaces.values():
            sp.close()


@dataclass
class _Reg:
    base_addr: int
    length: int
    access_token: int


def gather_descriptors_all(spaces: dict[int, MemorySpace]) -> dict[int, dict]:
    """Every rank's exported pools, keyed by server id."""
    from .distributed import all_gather_objects
    got = all_gather_objects([sp.export() for sp in spaces.values()])
    return {d["server_id"]: d for lst in got for d in lst}
