"""Whole sessions on the GPU path vs the reference's own runs (golden rows and
captured edge values: bit-identical), plus the reference's session-level
contracts (copy accounting, footprint, tracing, distributed == local)."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import port
from paper_1805_08430_b200 import errors
from paper_1805_08430_b200.analyzer import AllocSite
from paper_1805_08430_b200.graph import DataFlowGraph, shape_of
from paper_1805_08430_b200.runtime.session import Session
from paper_1805_08430_b200.wire import Mechanism, meta_block_size, static_region_size
from paper_1805_08430_b200.workloads import (build_layered_forward, build_microbench,
                                             build_ps_workload, mlp_shapes)

pytestmark = pytest.mark.gpu

ROW_FIELDS = ("iteration", "bytes_sent", "payload_bytes", "payload_bytes_copied",
              "copy_events", "serialize_bytes", "arena_peak_bytes", "polls")


def golden_case(name):
    if name.startswith("micro"):
        g, p = build_microbench(1 << 20 if name == "micro1m" else 4096)
    elif name in ("ps24k", "ps24k_dyn"):
        g, p = build_ps_workload(24_000, 2, 0.0, 2)
    elif name == "ps40k_cp":
        g, p = build_ps_workload(40_000, 2, 0.0, 2)
    elif name == "mlp_ps":
        g, p = build_ps_workload(0, 3, 0.0, 2, shapes=mlp_shapes())
    elif name == "coloc4":
        g, p = build_ps_workload(0, 4, 0.0, 4, ps_servers=4, shapes=[(3000,)] * 4,
                                 colocate=True)
    elif name == "ps7w":
        g, p = build_ps_workload(7_000, 5, 0.0, 7)
    else:
        raise KeyError(name)
    return g, p


@pytest.mark.parametrize("name", ["micro4k", "micro1m", "micro4k_dyn", "micro4k_cp",
                                  "ps24k", "ps24k_dyn", "ps40k_cp", "mlp_ps", "coloc4",
                                  "ps7w"])
def test_session_matches_reference_run(golden, name):
    doc, arr = golden
    ref = next(s for s in doc["sessions"] if s["name"] == name)
    g, p = golden_case(name)
    kw = dict(ref["kwargs"])
    s = Session(g, p, capture_edges=True, **kw)
    assert {f"{e}_{c}": int(m) for (e, c), m in s.mechanisms.items()} == ref["mechanisms"]
    rep = s.run(len(ref["rows"]))
    s.close()
    for got, want in zip(rep.rows, ref["rows"]):
        for f in ROW_FIELDS:
            assert getattr(got, f) == want[f], (name, got.iteration, f)
        assert got.sim_time_us == pytest.approx(want["sim_time_us"], rel=1e-12)
    assert len(rep.captured) == len(ref["captured"])
    for it, edge, srv, key, digest, n in ref["captured"]:
        data = rep.captured[(it, edge, srv)]
        assert len(data) == n and hashlib.sha256(data).hexdigest() == digest, \
            (name, it, edge, srv)
    for k, v in ref["arena_resident"].items():
        it, srv = map(int, k.split("_"))
        assert rep.arena_resident[(it, srv)] == v


def test_sgd_session_matches_restatement():
    shapes = mlp_shapes()
    g, p = build_ps_workload(0, 3, 0.0, 2, shapes=shapes)
    s = Session(g, p, seed=0, apply_op="sgd", lr=0.05)
    s.run(4)
    want = port.ps_expected(shapes, 2, 0, 4, op="sgd", lr=0.05)
    for v in range(3):
        got = np.frombuffer(s.variable_bytes(port.ps_node_ids(v, 0, 2)[0]), np.float32)
        # north-star tolerance 1e-6 relative; the kernel is in fact bit-exact
        np.testing.assert_allclose(got, want[v].reshape(-1), rtol=1e-6, atol=0)
        assert got.tobytes() == want[v].tobytes()
    s.close()


def test_zero_copy_accounting_contracts():
    g, p = build_ps_workload(40_000, 2, 0.0, 2)
    s = Session(g, p, mode="zerocp", seed=11)
    rep = s.run(4)
    n = len(s.pgraph.cross)
    assert rep.rows[0].copy_events == n
    assert all(r.payload_bytes_copied == 0 and r.copy_events == 0 for r in rep.rows[1:])
    assert sum(x.zero_copy_checks for x in s.senders.values()) == n * 3
    s.close()
    s = Session(g, p, mode="cp", seed=11)
    rep = s.run(2)
    assert all(r.copy_events == n and r.payload_bytes_copied == r.payload_bytes
               for r in rep.rows)
    s.close()


def test_rpc_mode_copies_twice_plus_meta():
    g, p = build_ps_workload(40_000, 2, 0.0, 2)
    s = Session(g, p, mode="rpc", seed=11)
    rep = s.run(2)
    meta = sum(meta_block_size(s.shapes[ce.edge_id].rank) for ce in s.pgraph.cross)
    for r in rep.rows:
        assert r.payload_bytes_copied == 2 * r.payload_bytes + meta
    s.close()


def test_ps_footprint_static_vs_dynamic():
    workers, var_bytes = 4, 40_000
    g, p = build_ps_workload(var_bytes, 1, 0.0, workers)
    ps = workers
    s = Session(g, p, seed=6, mechanism_override="static")
    assert sum(e.recv_buffer.length for e in s.plan.for_consumer(ps)) == \
        workers * static_region_size((var_bytes // 4,), s.elem_types[0])
    base = s.report.arena_baseline[ps]
    rep = s.run(3)
    assert all(rep.arena_resident[(it, ps)] == base + var_bytes for it in (1, 2, 3))
    s.close()
    s = Session(g, p, seed=6)
    assert sum(e.recv_buffer.length for e in s.plan.for_consumer(ps)) == \
        workers * meta_block_size(1)
    base = s.report.arena_baseline[ps]
    rep = s.run(3)
    assert all(rep.arena_resident[(it, ps)] == base + var_bytes for it in (1, 2, 3))
    assert s.rdma_arenas[ps].peak_resident >= base + 2 * var_bytes
    s.close()


def test_tracing_equals_oracle_instrumentation():
    g = DataFlowGraph()
    src = g.gen_grad(shape_of(64))
    fwd = g.inplace_scale(src)
    sink = g.reduce_max(fwd)
    p = {g.edges[src].producer: 0, g.edges[fwd].producer: 0, g.edges[sink].producer: 1}
    g.freeze()
    s = Session(g, p, seed=8, trace_oracle=True)
    s.run(3)
    traced = set().union(*(t.transfer_sites for t in s.traces.values()))
    assert traced == {AllocSite(g.edges[src].producer, 0)}
    assert s.oracle.sites_by_iteration[3] == traced
    s.close()


def _random_graph(seed):
    """Random small placed graph with placement-independent values."""
    rng = np.random.default_rng(seed)
    g = DataFlowGraph()
    edges = []
    for _ in range(int(rng.integers(1, 3))):
        edges.append(g.gen_grad(shape_of(int(rng.integers(1, 5)), 4)))
    for _ in range(int(rng.integers(2, 7))):
        e = edges[int(rng.integers(0, len(edges)))]
        k = int(rng.integers(0, 4))
        if k == 0:
            edges.append(g.sigmoid(e))
        elif k == 1:
            edges.append(g.reduce_max(e))
        elif k == 2:
            edges.append(g.concat_dyn([e], dyn_range=(1, 4)))
        else:
            edges.append(g.add(e, e))
    g.freeze()
    placement = {n: int(rng.integers(0, 3)) for n in g.nodes}
    return g, placement


@pytest.mark.parametrize("trial", range(8))
def test_distributed_equals_local(trial):
    g, p = _random_graph(1000 + trial)
    for override in (None, "dynamic"):
        dist = Session(g, p, seed=trial, capture_edges=True, mechanism_override=override)
        rd = dist.run(3)
        local = Session(g, {n: 0 for n in g.nodes}, seed=trial, capture_edges=True)
        rl = local.run(3)
        lv = {(it, e): v for (it, e, _s), v in rl.captured.items()}
        for (it, e, _s), v in rd.captured.items():
            assert lv[(it, e)] == v
        if override == "dynamic" and dist.mechanisms:
            assert set(dist.mechanisms.values()) == {Mechanism.DYNAMIC}
        dist.close()
        local.close()


def test_layered_forward_single_server_has_no_traffic():
    g, _, _ = build_layered_forward()
    s = Session(g, {n: 0 for n in g.nodes})
    rep = s.run(2)
    assert rep.total("bytes_sent") == 0
    s.close()


def test_mode_validation():
    g, p = build_microbench(4096)
    with pytest.raises(errors.InvalidConfig):
        Session(g, p, mode="bogus")


@pytest.mark.parametrize("mode", ["zerocp", "rpc"])
def test_threaded_sessions_match_round_robin_counters(mode):
    """One OS thread per server (reference session.py:631-649): interleavings
    differ, byte volumes / counters / simulated time agree; host doorbells are
    polled concurrently from several threads."""
    def rows(threads):
        g, p = build_ps_workload(24_000, 2, 0.0, 2)
        s = Session(g, p, mode=mode, seed=33, threads=threads)
        rep = s.run(3)
        s.close()
        return [(r.iteration, r.bytes_sent, r.payload_bytes, r.payload_bytes_copied,
                 r.copy_events, r.serialize_bytes, round(r.sim_time_us, 6)) for r in rep.rows]
    assert rows(False) == rows(True)


def test_doorbell_falls_back_to_device_reads_once_exported():
    from paper_1805_08430_b200.memspace import MemorySpace
    sp = MemorySpace(0, 1 << 20, device=0)
    r = sp.allocate_region(4096, register=True)
    sp.bind_doorbell(r)
    tail = r.base_addr + r.length - 1
    sp.write_raw(tail, b"\x01")            # a write the shadow never saw
    assert sp.flag_read(tail, 1) == b"\x00"   # in-process: the shadow is authoritative
    sp.export()                             # producers may now be other processes
    assert sp.flag_read(tail, 1) == b"\x01"   # device read
    sp.flag_clear(tail)
    assert sp.read_raw(tail, 1) == b"\x00"
