"""Pin the CPU oracle (oracle/port.py) against vectors the reference produced.

CPU only.  Fixtures: tests/golden/make_golden.py (imports the reference).
"""
from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from oracle import port

RIG_CAP = 1 << 22


class OracleRig:
    """The reference protocol-test rig (tests/test_protocol.py:15-71) on the oracle."""

    def __init__(self, seed=5):
        self.fab = port.Delivery(seed)
        self.spaces = {s: port.Space(s, RIG_CAP, seed=s) for s in (0, 1)}
        self.arenas = {}
        for s, sp in self.spaces.items():
            base, tok = sp.allocate_region(RIG_CAP // 2, True)
            self.arenas[s] = port.Arena(base, RIG_CAP // 2, tok)
        self.flags = {}
        for s in (0, 1):
            cell = self.arenas[s].alloc(1)
            self.spaces[s].mem[cell] = 1
            self.flags[s] = cell

    def region(self, size):
        a = self.arenas[1].alloc(size)
        self.spaces[1].mem[a + size - 1] = 0
        return (a, size, self.arenas[1].token)

    def tensor(self, dims, elem_size=4, seed=42):
        nbytes = math.prod(dims) * elem_size
        data = np.random.default_rng(seed).integers(0, 256, nbytes, dtype=np.uint8)
        a = self.arenas[0].alloc(max(nbytes, 1))
        self.spaces[0].mem[a:a + nbytes] = data
        return a, nbytes


def test_wire_formats(golden):
    doc, _ = golden
    w = doc["wire"]
    assert port.encode_meta((3, 4), 0, 0x1000, 0x42).hex() == w["formats_meta_hex"]
    assert port.addr_msg(7, 0x2A000, 0x1122334455667788, 49, 1).hex() == w["formats_addr_hex"]
    for c in w["meta_cases"]:
        raw = port.encode_meta(c["dims"], c["elem"], c["addr"], c["token"])
        assert raw.hex() == c["hex"]
        dims, elem, addr, tok, plen = port.decode_meta(raw, len(c["dims"]))
        assert list(dims) == c["dims"] and (elem, addr, tok) == (c["elem"], c["addr"], c["token"])


def test_synthetic_streams(golden):
    doc, arr = golden
    for s in doc["synth"]:
        got = port.synthesize(257, s["elem"], port.node_rng(s["seed"], s["node"], s["it"]))
        assert got.tobytes() == arr[s["key"]].tobytes()
    c1 = port.synthesize(262144, 0, port.node_rng(0, 0, 2))
    assert [float(x) for x in c1[:4]] == doc["c1"]["first4"]
    assert float(c1.astype(np.float64).sum()) == doc["c1"]["sum64"]


def test_chunk_plans(golden):
    doc, _ = golden
    fabs = {}
    for p in doc["chunk_plans"]:
        fab = fabs.setdefault(p["seed"], port.Delivery(p["seed"]))
        plan = fab.chunk_plan(p["total"])
        assert plan == p["plan"]
        assert sum(plan) == p["total"] and all(1 <= c <= 4096 for c in plan)


def test_rig_static_vectors(golden):
    doc, arr = golden
    for r in [x for x in doc["rig"] if x["mech"] == "static"]:
        rig = OracleRig()
        dims = tuple(r["dims"])
        region = rig.region(math.prod(dims) * 4 + 1)
        payload = rig.tensor(dims)
        assert (region[0], region[1], region[2]) == (r["recv_addr"], r["recv_len"], r["recv_token"])
        assert payload[0] == r["payload_addr"]
        port.static_send(rig.fab, rig.spaces[0], payload, rig.flags[0], rig.spaces[1], region)
        a, n, _ = region
        assert rig.spaces[1].mem[a:a + n].tobytes() == arr[r["key"] + "/after_send"].tobytes()
        got = port.static_poll(rig.spaces[1], region)
        assert got is not None and got.nbytes == r["got_nbytes"]
        assert rig.spaces[1].mem[a:a + n].tobytes() == arr[r["key"] + "/after_poll"].tobytes()
        assert rig.fab.wire_bytes == r["wire_bytes"]
        with pytest.raises(AssertionError):  # second send before consumption
            rig.spaces[1].mem[a + n - 1] = 1
            port.static_send(rig.fab, rig.spaces[0], payload, rig.flags[0], rig.spaces[1], region)


def test_rig_dynamic_vectors(golden):
    doc, arr = golden
    for r in [x for x in doc["rig"] if x["mech"] == "dynamic"]:
        rig = OracleRig()
        dims = tuple(r["dims"])
        meta_region = rig.region(port.meta_block_size(len(dims)))
        payload = rig.tensor(dims)
        stage = rig.arenas[0].alloc(port.meta_block_size(len(dims)))
        # the reference DynSender allocates its meta stage at construction,
        # before the tensor: rebuild that order
        rig = OracleRig()
        meta_region = rig.region(port.meta_block_size(len(dims)))
        stage = rig.arenas[0].alloc(port.meta_block_size(len(dims)))
        payload = rig.tensor(dims)
        assert meta_region[0] == r["recv_addr"] and payload[0] == r["payload_addr"]
        port.dyn_send(rig.fab, rig.spaces[0], stage, dims, 0, payload[0],
                      rig.arenas[0].token, rig.spaces[1], meta_region)
        a, n, _ = meta_region
        assert rig.spaces[1].mem[a:a + n].tobytes() == arr[r["key"] + "/meta"].tobytes()
        local, plen, got_dims = port.dyn_poll_fetch(rig.fab, rig.spaces[1], rig.arenas[1],
                                                    meta_region, len(dims), rig.spaces[0])
        assert got_dims == dims
        sent = arr[r["key"] + "/sent"].tobytes()
        assert rig.spaces[1].mem[local:local + plen].tobytes() == sent
        if plen:
            assert local == r["pulled_addr"]
        assert rig.fab.verbs == r["verbs"] and rig.fab.wire_bytes == r["wire_bytes"]


def _session(doc, name):
    return next(s for s in doc["sessions"] if s["name"] == name)


def _final_vars(sess, shapes, workers, shard_of, steps):
    """Digests of each variable's value after ``steps`` iterations, read from
    the captured output edge of its last ApplyGrad (edge id == node id)."""
    caps = {(it, e, s): (k, h) for it, e, s, k, h, _n in sess["captured"]}
    out = []
    for v in range(len(shapes)):
        apply_last = port.ps_node_ids(v, workers - 1, workers)[2]
        out.append(caps[(steps, apply_last, shard_of(v))][1])
    return out


@pytest.mark.parametrize("name,shapes,workers,shards,coloc,seed,steps", [
    ("ps24k", [(3000,)] * 2, 2, 1, False, 3, 3),
    ("ps24k_dyn", [(3000,)] * 2, 2, 1, False, 3, 3),
    ("mlp_ps", [(16, 12), (12, 10), (10, 4)], 2, 1, False, 0, 4),
    ("coloc4", [(3000,)] * 4, 4, 4, True, 1, 3),
    ("ps7w", [(350,)] * 5, 7, 1, False, 2, 2),
])
def test_ps_xor_recipe_matches_reference(golden, name, shapes, workers, shards, coloc,
                                         seed, steps):
    doc, _ = golden
    sess = _session(doc, name)
    want = _final_vars(sess, shapes, workers,
                       lambda v: (v % shards) + (0 if coloc else workers), steps)
    got = port.ps_expected(shapes, workers, seed, steps, op="xor")
    assert [hashlib.sha256(g.tobytes()).hexdigest() for g in got] == want


def test_ps_rig_equals_recipe():
    shapes = [(1000,), (37,), (4, 9)]
    for coloc, W, P in ((False, 2, 1), (True, 3, 3), (False, 3, 2)):
        rig = port.PsRig(shapes, W, P, coloc, seed=4)
        for _ in range(3):
            rig.step()
        want = port.ps_expected(shapes, W, 4, 3)
        for v in range(len(shapes)):
            assert rig.variable(v).tobytes() == want[v].tobytes()
        rig = port.PsRig(shapes, W, P, coloc, seed=4, op="sgd", lr=0.05)
        for _ in range(2):
            rig.step()
        want = port.ps_expected(shapes, W, 4, 2, op="sgd", lr=0.05)
        for v in range(len(shapes)):
            assert rig.variable(v).tobytes() == want[v].tobytes()


def test_sgd_restatement_is_unfused_fp32():
    # var - lr*g with a separately rounded product (no FMA): check one case
    # where FMA and the two-step form differ
    v = np.array([1.0000001], np.float32)
    g = np.array([0.3333333], np.float32)
    lr = 0.1
    two_step = np.float32(v[0] - np.float32(np.float32(lr) * g[0]))
    port.apply_sgd(v, [g], lr)
    assert v[0] == two_step


def test_transfer_rigs_run():
    for mech in ("static", "dynamic"):
        rig = port.TransferRig(10_000, mech)
        for _ in range(3):
            rig.step()
    mb = port.MicrobenchRig(4096)
    val = mb.step()
    want = port.synthesize(1024, 0, port.node_rng(0, 0, 2)).max()
    assert val == float(want)


def test_rpc_port_and_cp_rig():
    rig = port.RpcRig(40 * port.FRAG_PAYLOAD + 123 * 4)
    out = rig.step()
    assert out.tobytes() == rig.src.tobytes()
    assert rig.copied == 2 * rig.n + port.meta_block_size(1)
    rig.step()
    cp = port.MicrobenchRig(1 << 16, generate=False, stage_copy=True)
    zc = port.MicrobenchRig(1 << 16, generate=False)
    assert cp.step() == zc.step()
