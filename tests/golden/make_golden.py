"""Generate golden vectors from the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports rdmaflow from /root/reference/pkg/src and writes
tests/golden/golden.json + golden.npz.  Nothing at test/bench time reads
/root/reference; the committed fixtures travel instead.  The oracle
restatement (oracle/port.py) and the GPU path are both checked against them.
"""
from __future__ import annotations

import base64
import hashlib
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from rdmaflow import wire  # noqa: E402
from rdmaflow.analyzer import PlanEntry  # noqa: E402
from rdmaflow.fabric import Fabric  # noqa: E402
from rdmaflow.graph import (DataFlowGraph, Tensor, TensorShape, node_rng,  # noqa: E402
                            shape_of, synthesize_values)
from rdmaflow.memspace import ArenaAllocator, BufferRef, MemorySpace  # noqa: E402
from rdmaflow.runtime.protocol import (DynReceiver, DynSender, StaticReceiver,  # noqa: E402
                                       StaticSender)
from rdmaflow.runtime.session import Session  # noqa: E402
from rdmaflow.wire import ElemType, Mechanism  # noqa: E402
from rdmaflow.workloads import build_microbench, build_ps_workload  # noqa: E402

ROW_FIELDS = ("iteration", "bytes_sent", "payload_bytes", "payload_bytes_copied",
              "copy_events", "serialize_bytes", "arena_peak_bytes", "polls")

arrays: dict[str, np.ndarray] = {}
doc: dict = {"generator": "tests/golden/make_golden.py", "reference": REF}


def b64(b: bytes) -> str:
    return base64.b64encode(b).decode()


# 1. wire layouts -----------------------------------------------------------------
w = {}
w["formats_meta_hex"] = wire.encode_meta((3, 4), ElemType.F32, 0x1000, 0x42).hex()
w["formats_addr_hex"] = wire.AddrExchangeMsg(7, 0x2A000, 0x1122334455667788, 49,
                                             Mechanism.DYNAMIC).encode().hex()
rng = random.Random(1234)
cases = []
for _ in range(300):
    rank = rng.randint(1, 4)
    dims = [rng.choice([0, 1, 3, 7, 1024, rng.randint(0, 1 << 20)]) for _ in range(rank)]
    elem = rng.randint(0, 4)
    addr, tok = rng.getrandbits(48), rng.getrandbits(64)
    cases.append({"dims": dims, "elem": elem, "addr": addr, "token": tok,
                  "hex": wire.encode_meta(dims, ElemType(elem), addr, tok).hex()})
w["meta_cases"] = cases
doc["wire"] = w

# 2. synthetic values ----------------------------------------------------------------
syn = []
for seed, node, it in [(0, 0, 2), (0, 0, 1), (3, 5, 7), (11, 123, 4), (0xFFFFFFFF, 9, 0)]:
    for elem in ElemType:
        v = synthesize_values((257,), elem, node_rng(seed, node, it))
        key = f"syn/{seed}_{node}_{it}_{int(elem)}"
        arrays[key] = np.ascontiguousarray(v)
        syn.append({"seed": seed, "node": node, "it": it, "elem": int(elem), "key": key})
doc["synth"] = syn
c1 = synthesize_values((262144,), ElemType.F32, node_rng(0, 0, 2))
doc["c1"] = {"first4": [float(x) for x in c1[:4]], "sum64": float(c1.astype(np.float64).sum())}

# 3. chunk plans ----------------------------------------------------------------------
plans = []
for seed in (0, 5, 77):
    fab = Fabric(seed=seed)
    for total in (1, 41, 4096, 4097, 10000, 1 << 20):
        plans.append({"seed": seed, "total": total, "plan": fab.chunk_plan(total)})
doc["chunk_plans"] = plans


# 4. Rig-level protocol vectors (the reference test rig, tests/test_protocol.py:15-71)
class Rig:
    def __init__(self, capacity=1 << 22, qps=2, seed=5):
        self.fabric = Fabric(seed=seed)
        self.spaces = {s: MemorySpace(s, capacity, seed=s) for s in (0, 1)}
        self.arenas = {}
        for s, sp in self.spaces.items():
            self.arenas[s] = ArenaAllocator(sp, sp.allocate_region(capacity // 2, register=True))
        self.devices = {s: self.fabric.create_device(self.spaces[s], qps_per_peer=qps)
                        for s in (0, 1)}
        self.fwd = self.devices[0].connect(self.devices[1].endpoint)
        self.back = self.devices[1].channels_to(self.devices[0].endpoint)
        self.flags = {}
        for s in (0, 1):
            cell = self.arenas[s].alloc(1)
            self.spaces[s].write_at(cell, 0, b"\x01")
            self.flags[s] = cell

    def entry(self, dims, mech, elem=ElemType.F32):
        shape = TensorShape(tuple(dims))
        e = PlanEntry(0, 0, 1, mech, shape, elem, shape.rank)
        size = (wire.static_region_size(shape.static_dims(), elem) if mech is Mechanism.STATIC
                else wire.meta_block_size(shape.rank))
        buf = self.arenas[1].alloc(size)
        self.spaces[1].write_at(buf, size - 1, b"\x00")
        e.recv_buffer = buf
        e.remote_addr, e.remote_token, e.remote_len = buf.base_addr, buf.access_token, buf.length
        return e

    def tensor(self, dims, elem=ElemType.F32, seed=42):
        n = int(np.prod(dims)) if dims else 1
        nbytes = n * elem.size
        data = np.random.default_rng(seed).integers(0, 256, nbytes, dtype=np.uint8).tobytes()
        h = self.arenas[0].alloc(max(nbytes, 1))
        if nbytes:
            self.spaces[0].write_at(h, 0, data)
        return Tensor(tuple(dims), elem, BufferRef(h, self.arenas[0]), 0)


rig_out = []
for dims in [(3, 4), (10,), (0, 4), (1,), (257, 3), (1 << 14,)]:
    rig = Rig()
    e = rig.entry(dims, Mechanism.STATIC)
    t = rig.tensor(dims)
    StaticSender(e, rig.spaces[0], rig.arenas[0], rig.fwd[1], rig.flags[0]).send(
        t, stage_copy=False)
    region_after_send = rig.spaces[1].read_at(e.recv_buffer, 0, e.recv_buffer.length)
    got = StaticReceiver(e, rig.spaces[1]).poll()
    region_after_poll = rig.spaces[1].read_at(e.recv_buffer, 0, e.recv_buffer.length)
    key = f"rig/static/{'x'.join(map(str, dims))}"
    arrays[key + "/sent"] = np.frombuffer(rig.spaces[0].read_at(t.buffer.handle, 0, t.nbytes)
                                          if t.nbytes else b"", np.uint8)
    arrays[key + "/after_send"] = np.frombuffer(region_after_send, np.uint8)
    arrays[key + "/after_poll"] = np.frombuffer(region_after_poll, np.uint8)
    rig_out.append({"mech": "static", "dims": list(dims), "key": key,
                    "recv_addr": e.recv_buffer.base_addr, "recv_token": e.recv_buffer.access_token,
                    "recv_len": e.recv_buffer.length, "payload_addr": t.buffer.handle.base_addr,
                    "wire_bytes": rig.fabric.wire_bytes, "got_nbytes": got.nbytes})

for dims in [(5, 8), (0, 8), (7,), (1 << 13,)]:
    rig = Rig()
    e = rig.entry(dims, Mechanism.DYNAMIC)
    snd = DynSender(e, rig.spaces[0], rig.arenas[0], rig.fwd[1])
    rcv = DynReceiver(e, rig.spaces[1], rig.arenas[1], rig.back[1])
    t = rig.tensor(dims)
    snd.send(t, stage_copy=False)
    meta_block = rig.spaces[1].read_at(e.recv_buffer, 0, e.recv_buffer.length)
    meta = rcv.poll()
    got = rcv.fetch(meta)
    key = f"rig/dynamic/{'x'.join(map(str, dims))}"
    arrays[key + "/meta"] = np.frombuffer(meta_block, np.uint8)
    pulled = rig.spaces[1].read_at(got.buffer.handle, 0, got.nbytes) if got.nbytes else b""
    arrays[key + "/sent"] = np.frombuffer(rig.spaces[0].read_at(t.buffer.handle, 0, t.nbytes)
                                          if t.nbytes else b"", np.uint8)
    assert pulled == arrays[key + "/sent"].tobytes()
    rig_out.append({"mech": "dynamic", "dims": list(dims), "key": key,
                    "recv_addr": e.recv_buffer.base_addr, "pulled_addr": got.buffer.handle.base_addr,
                    "payload_addr": t.buffer.handle.base_addr,
                    "serialize_bytes": rig.spaces[0].counters.serialize_bytes,
                    "verbs": rig.fabric.verbs_posted, "wire_bytes": rig.fabric.wire_bytes})
doc["rig"] = rig_out


# 5. sessions ---------------------------------------------------------------------------
def run_session(name, graph, placement, iters, **kw):
    s = Session(graph, placement, capture_edges=True, **kw)
    rep = s.run(iters)
    s.close()
    rows = [{f: getattr(r, f) for f in ROW_FIELDS} | {"sim_time_us": r.sim_time_us}
            for r in rep.rows]
    caps = []
    for (it, edge, srv), data in sorted(rep.captured.items()):
        k = f"cap/{name}/{it}_{edge}_{srv}"
        if len(data) <= 1024:   # small values verbatim, large ones by digest
            arrays[k] = np.frombuffer(data, np.uint8)
        caps.append([it, edge, srv, k, hashlib.sha256(data).hexdigest(), len(data)])
    return {"name": name, "rows": rows, "captured": caps, "kwargs": {
        k: v for k, v in kw.items() if isinstance(v, (int, float, str, type(None)))},
        "mechanisms": {f"{e}_{c}": int(m) for (e, c), m in s.mechanisms.items()},
        "arena_resident": {f"{it}_{srv}": v for (it, srv), v in rep.arena_resident.items()}}


def ps_graph_shapes(shapes, workers, ps_servers=1, colocate=False):
    """PS graph with per-variable shapes built with the reference API, one
    variable/gen_grad/apply_grad group per variable as workloads.py:81-93."""
    g = DataFlowGraph()
    placement = {}
    for v, dims in enumerate(shapes):
        shard = (v % ps_servers) + (0 if colocate else workers)
        weight = g.variable(shape_of(*dims))
        placement[g.edges[weight].producer] = shard
        for wk in range(workers):
            grad = g.gen_grad(shape_of(*dims), inputs=(weight,))
            placement[g.edges[grad].producer] = wk
            upd = g.apply_grad(weight, grad)
            placement[g.edges[upd].producer] = shard
    g.freeze()
    return g, placement


sessions = []
g, p = build_microbench(4096)
sessions.append(run_session("micro4k", g, p, 3, mode="zerocp", seed=0))
g, p = build_microbench(1 << 20)
sessions.append(run_session("micro1m", g, p, 3, mode="zerocp", seed=0,
                            capacity_bytes=(16 << 20) + (4 << 20) + (1 << 20),
                            arena_bytes=(4 << 20) + (1 << 20)))
g, p = build_microbench(4096)
sessions.append(run_session("micro4k_dyn", g, p, 3, mode="zerocp", seed=0,
                            mechanism_override="dynamic"))
g, p = build_microbench(4096)
sessions.append(run_session("micro4k_cp", g, p, 2, mode="cp", seed=0))
g, p = build_ps_workload(24_000, 2, 0.0, 2)
sessions.append(run_session("ps24k", g, p, 3, mode="zerocp", seed=3))
g, p = build_ps_workload(24_000, 2, 0.0, 2)
sessions.append(run_session("ps24k_dyn", g, p, 3, mode="zerocp", seed=3,
                            mechanism_override="dynamic"))
g, p = build_ps_workload(40_000, 2, 0.0, 2)
sessions.append(run_session("ps40k_cp", g, p, 2, mode="cp", seed=11))
g, p = ps_graph_shapes([(16, 12), (12, 10), (10, 4)], 2)
sessions.append(run_session("mlp_ps", g, p, 4, mode="zerocp", seed=0))
g, p = ps_graph_shapes([(3000,)] * 4, 4, ps_servers=4, colocate=True)
sessions.append(run_session("coloc4", g, p, 3, mode="zerocp", seed=1))
g, p = build_ps_workload(7_000, 5, 0.0, 7)
sessions.append(run_session("ps7w", g, p, 2, mode="zerocp", seed=2, watchdog_sweeps=10_000))
doc["sessions"] = sessions

with open(os.path.join(HERE, "golden.json"), "w") as fh:
    json.dump(doc, fh, indent=1)
np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
print(f"wrote {len(arrays)} arrays, {len(sessions)} sessions")
