"""Host-side logic that needs no GPU: C-ABI exports, wire layouts, arena
ledger, analyzer classification, partitioning, scheduler.  CPU only."""
from __future__ import annotations

import ctypes as C
import os
import random
import re

import numpy as np
import pytest

from paper_1805_08430_b200 import _lib, errors, wire
from paper_1805_08430_b200.analyzer import classify_edges
from paper_1805_08430_b200.graph import (ExecMode, infer_shapes, in_place_control_deps,
                                         partition)
from paper_1805_08430_b200.memspace import ArenaAllocator, RegionHandle
from paper_1805_08430_b200.runtime.executor import Executor, FnHandler
from paper_1805_08430_b200.wire import ElemType, Mechanism
from paper_1805_08430_b200.workloads import (build_layered_forward, build_microbench,
                                             build_ps_workload, total_params, vgg16_shapes)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# -- the C ABI -----------------------------------------------------------------------


def header_functions() -> list[str]:
    text = open(os.path.join(ROOT, "include", "srflow.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/srflow.h but not exported"
    assert set(names) == set(_lib.SIGNATURES), "ctypes binding out of sync with the header"
    assert lib.srf_version() == 1


def test_library_is_sm100a():
    so = _lib.LIB_PATH
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    assert "sm_100a" in out, out


def test_status_codes_map_to_reference_classes():
    assert _lib._STATUS[13] is errors.NotRegistered
    assert _lib._STATUS[14] is errors.BadToken
    assert _lib._STATUS[15] is errors.RemoteOutOfBounds
    assert issubclass(errors.RemoteOutOfBounds, errors.FabricError)
    with pytest.raises(errors.BadToken):
        _lib.check(14)
    assert _lib.check(0) == 0 and _lib.check(1) == 1


# -- wire (product) vs reference-generated vectors -------------------------------------


def test_wire_matches_reference_vectors(golden):
    doc, _ = golden
    w = doc["wire"]
    assert wire.encode_meta((3, 4), ElemType.F32, 0x1000, 0x42).hex() == w["formats_meta_hex"]
    msg = wire.AddrExchangeMsg(7, 0x2A000, 0x1122334455667788, 49, Mechanism.DYNAMIC)
    assert msg.encode().hex() == w["formats_addr_hex"]
    assert wire.AddrExchangeMsg.decode(msg.encode()) == msg
    for c in w["meta_cases"]:
        raw = wire.encode_meta(c["dims"], ElemType(c["elem"]), c["addr"], c["token"])
        assert raw.hex() == c["hex"]
        m = wire.decode_meta(raw, len(c["dims"]))
        assert list(m.dims) == c["dims"] and m.remote_token == c["token"]


def test_wire_errors():
    raw = wire.encode_meta((2, 2), ElemType.F32, 0, 0)
    with pytest.raises(errors.RankMismatch):
        wire.decode_meta(raw, 3)
    with pytest.raises(errors.RankZero):
        wire.encode_meta((), ElemType.F32, 0, 0)
    bad = bytearray(raw)
    bad[0] = 9
    with pytest.raises(errors.BadElemType):
        wire.decode_meta(bytes(bad), 2)
    bad = bytearray(raw)
    bad[-1] = 0
    with pytest.raises(errors.WireError):
        wire.decode_meta(bytes(bad), 2)
    with pytest.raises(errors.LengthMismatch):
        wire.decode_meta(raw[:-1], 2)
    assert wire.static_region_size((1024, 1024), ElemType.F32) == 4_194_305
    assert wire.meta_block_size(1) == 41 and wire.meta_block_size(2) == 49


# -- arena ledger (memspace.py:239-308 semantics) ---------------------------------------


class _FakeSpace:
    server_id = 0


def test_arena_ledger_replay():
    backing = RegionHandle(0, 64, 1 << 20, 0xABC)
    arena = ArenaAllocator(_FakeSpace(), backing)
    rng = random.Random(7)
    live: dict[int, int] = {}
    for _ in range(1000):
        if live and rng.random() < 0.45:
            addr = rng.choice(sorted(live))
            arena.free(RegionHandle(0, addr, live.pop(addr), 0xABC))
        else:
            n = rng.randint(1, 5000)
            try:
                h = arena.alloc(n)
            except errors.ArenaExhausted:
                continue
            assert h.base_addr % 8 == 0 and h.access_token == 0xABC
            live[h.base_addr] = n
        assert arena.current_resident == sum(live.values())
        blocks = arena.live_blocks()
        for (o1, l1), (o2, _l2) in zip(blocks, blocks[1:]):
            assert o1 + l1 <= o2
    for addr in sorted(live):
        arena.free(RegionHandle(0, addr, live[addr], 0xABC))
    assert arena.current_resident == 0
    assert arena.alloc((1 << 20) - 8).base_addr == 64  # fully coalesced
    with pytest.raises(ValueError):
        arena.free(RegionHandle(0, 12345, 8, 0))


def test_arena_first_fit_reuse():
    arena = ArenaAllocator(_FakeSpace(), RegionHandle(0, 0, 1 << 16, 1))
    a, b, c = (arena.alloc(1024) for _ in range(3))
    arena.free(b)
    assert arena.alloc(1024).base_addr == b.base_addr
    with pytest.raises(errors.ArenaExhausted):
        arena.alloc((1 << 16) + 1)


# -- analyzer / graph ------------------------------------------------------------------


def test_ps_classification_matches_reference(golden):
    doc, _ = golden
    g, p = build_ps_workload(24_000, 2, 0.0, 2)
    mech = classify_edges(partition(g, p), infer_shapes(g))
    want = next(s for s in doc["sessions"] if s["name"] == "ps24k")["mechanisms"]
    assert {f"{e}_{c}": int(m) for (e, c), m in mech.items()} == want
    assert set(mech.values()) == {Mechanism.STATIC, Mechanism.DYNAMIC}
    assert len(partition(g, p).cross) == 2 * 2 * 2  # weight + grad per (var, worker)


def test_dynamic_cone_and_shapes():
    g, _, cone = build_layered_forward(with_concat=True)
    shapes = infer_shapes(g)
    for e, s in shapes.items():
        assert s.is_static == (e not in cone)


def test_in_place_deps_order_readers_before_writers():
    g, p = build_ps_workload(8_000, 1, 0.0, 3)
    pg = partition(g, p)
    ps = 3
    ids = pg.nodes_on(ps)
    deps = in_place_control_deps(ids, pg.node, lambda e: pg.consumers_on(e, ps))
    applies = sorted(n for n in ids if pg.node(n).kind.value == "ApplyGrad")
    for prev, nxt in zip(applies, applies[1:]):
        assert prev in deps[nxt]
    sends = [n for n in ids if pg.node(n).kind.value == "RdmaSend"]
    assert all(s in deps[applies[0]] for s in sends)


def test_vgg16_shapes():
    shapes = vgg16_shapes()
    assert len(shapes) == 32 and total_params(shapes) == 138_357_544


def test_microbench_graph():
    g, p = build_microbench(1 << 20)
    pg = partition(g, p)
    assert len(pg.cross) == 1
    assert classify_edges(pg, infer_shapes(g))[(0, 1)] is Mechanism.STATIC


# -- scheduler (runtime/executor.py semantics) ---------------------------------------------


def test_pending_poll_reenqueues_at_tail_and_fairness():
    ex = Executor(0, keep_trace=True)
    done = []
    for i in range(100):
        ex.add_node(2 * i, FnHandler(ExecMode.POLLING_ASYNC, poll=lambda: None))
        ex.add_node(2 * i + 1, FnHandler(run=lambda i=i: done.append(i)))
    ex.begin_iteration(1)
    steps = 0
    while len(done) < 100:
        ex.step()
        steps += 1
        assert steps <= 400
    polls: dict[int, int] = {}
    for _s, node, ev in ex.trace:
        if ev == "poll_pending":
            polls[node] = polls.get(node, 0) + 1
    assert max(polls.values()) <= 2


def test_watchdog_trips():
    ex = Executor(0)
    ex.add_node(0, FnHandler(ExecMode.POLLING_ASYNC, poll=lambda: None))
    ex.begin_iteration(1)
    with pytest.raises(errors.Deadlock):
        ex.run_until_done(watchdog_steps=200)


def test_ready_poll_completes_once():
    seen = []
    ex = Executor(0)
    ex.add_node(0, FnHandler(ExecMode.POLLING_ASYNC, poll=lambda: "tok",
                             complete=seen.append))
    ex.begin_iteration(1)
    ex.step()
    assert not ex.done()
    ex.step()
    assert ex.done() and seen == ["tok"]


# -- PS layout (pure host) ----------------------------------------------------------------


def test_ps_layout_blocks_and_traffic():
    from paper_1805_08430_b200.ps import PsLayout
    shapes = vgg16_shapes()
    L = PsLayout(shapes, 8, 8, colocate=True)
    assert L.nservers == 8
    for s in range(8):
        offs = sorted(L.blocks[s].values())
        assert all(o % 16 == 0 for o in offs)
        assert len(set(offs)) == len(offs)
    t = [L.traffic(s) for s in range(8)]
    # round-robin places fc6 (25088x4096, v=26) on shard 2: the hottest egress (F5)
    assert L.shard_of(26) == 2
    assert max(range(8), key=lambda s: t[s]["push_out"]) == 2
    total_vars = sum(L.nbytes(v) for v in range(32))
    assert sum(x["pull_in"] for x in t) == 7 * total_vars
    L1 = PsLayout(shapes, 1, 1)
    assert L1.nservers == 2 and L1.shard_of(5) == 1
    assert L1.traffic(1)["push_out"] == sum(L1.nbytes(v) + 1 for v in range(32))


def test_ps_byte_balanced_placement_extension():
    from paper_1805_08430_b200.ps import PsLayout
    shapes = vgg16_shapes()
    rr = PsLayout(shapes, 8, 8, colocate=True)
    bb = PsLayout(shapes, 8, 8, colocate=True, placement="bytes")
    load = lambda L: [sum(L.nbytes(v) for v in range(32) if L.shard_of(v) == k) for k in range(8)]
    assert max(load(bb)) < max(load(rr))  # fc6 still alone, but nothing piles onto it
    assert sorted(bb.shard_of(v) for v in range(32)) != [v % 8 for v in range(32)]
    assert max(load(bb)) == bb.nbytes(26)  # the 411 MB fc6 shard holds only fc6


def test_ps_link_traffic_excludes_same_gpu_servers():
    from paper_1805_08430_b200.ps import PsLayout, link_traffic
    L = PsLayout([(1000,)] * 10, 2, 1)          # workers 0,1 + PS server 2
    t = link_traffic(L, 2)                      # servers 0,2 on GPU 0; server 1 on GPU 1
    S = 4000
    assert t[0]["link_out"] == 10 * (S + 1)     # pushes to worker 1 only
    assert t[1]["link_out"] == 10 * (41 + S)    # worker 1's metadata + gradient reads
    assert link_traffic(L, 1)[0] == {"link_out": 0, "link_in": 0}


def test_partitioned_layout_units():
    from paper_1805_08430_b200.ps import PsLayout
    from paper_1805_08430_b200.workloads import vgg16_shapes
    shapes = vgg16_shapes()
    L = PsLayout(shapes, 4, 4, colocate=True, placement="bytes", partition_bytes=16 << 20)
    # every element of every model variable is covered exactly once, in order
    for v, dims in enumerate(shapes):
        parts = sorted((L.parent(u)[1], L.parent(u)[2]) for u in range(len(L.shapes))
                       if L.parent(u)[0] == v)
        n = int(np.prod(dims))
        assert parts[0][0] == 0 and sum(c for _o, c in parts) == n
        for (o1, c1), (o2, _c2) in zip(parts, parts[1:]):
            assert o1 + c1 == o2 and (o2 * 4) % 256 == 0
    big = [u for u in range(len(L.shapes)) if L.parent(u)[0] == 26]   # fc6
    assert len(big) == 4 and len({L.shard_of(u) for u in big}) == 4
    # no unit exceeds the largest slice; shard loads within one slice of each other
    load = [sum(L.nbytes(u) for u in range(len(L.shapes)) if L.shard_of(u) == k)
            for k in range(4)]
    assert max(load) - min(load) <= max(L.nbytes(u) for u in range(len(L.shapes)))
    # node ids are the model variable's
    assert L.node_ids(big[2], 1) == L.node_ids(big[0], 1)


def test_sliced_layout_units_stay_on_their_shard():
    """EXTENSION (pipelined transfers): big units are cut into consecutive
    ~slice_bytes slices; the reference placement is unchanged."""
    from paper_1805_08430_b200.ps import PsLayout
    from paper_1805_08430_b200.workloads import vgg16_shapes
    shapes = vgg16_shapes()
    ref = PsLayout(shapes, 4, 4, colocate=True)
    L = PsLayout(shapes, 4, 4, colocate=True, slice_bytes=8 << 20)
    assert len(L.shapes) > len(ref.shapes)
    for v, dims in enumerate(shapes):
        us = [u for u in range(len(L.shapes)) if L.parent(u)[0] == v]
        parts = [(L.parent(u)[1], L.parent(u)[2]) for u in us]
        assert parts[0][0] == 0 and sum(c for _o, c in parts) == int(np.prod(dims))
        for (o1, c1), (o2, _c2) in zip(parts, parts[1:]):
            assert o1 + c1 == o2 and (o2 * 4) % 256 == 0
        assert {L.shard_of(u) for u in us} == {ref.shard_of(v)}   # placement kept
        assert all(L.nbytes(u) <= 8 << 20 for u in us)
        if len(us) == 1:
            assert L.shapes[us[0]] == tuple(dims)                 # small tensors untouched
    # slices of a partitioned variable stay on their partition's shard
    P = PsLayout(shapes, 4, 4, colocate=True, placement="bytes", partition_bytes=16 << 20)
    PS = PsLayout(shapes, 4, 4, colocate=True, placement="bytes", partition_bytes=16 << 20,
                  slice_bytes=8 << 20)
    for u in range(len(PS.shapes)):
        v, off, _n = PS.parent(u)
        owner = next(p for p in range(len(P.shapes)) if P.parent(p)[0] == v
                     and P.parent(p)[1] <= off < P.parent(p)[1] + P.parent(p)[2])
        assert PS.shard_of(u) == P.shard_of(owner)


def test_static_gradient_layout_and_traffic():
    """grad_mechanism="static" (the reference's mechanism_override="static"):
    receive regions of S+1 on the shard instead of metadata slots, a ready
    byte per remote gradient on the worker; NVLink bytes drop the metadata
    block for the one flag byte."""
    from paper_1805_08430_b200.ps import PsLayout, link_traffic
    shapes = [(1000,), (37,), (4, 9)]
    d = PsLayout(shapes, 2, 1)
    s = PsLayout(shapes, 2, 1, grad_mechanism="static")
    for v in range(3):
        for w in range(2):
            assert ("grecv", v, w) in s.blocks[2] and ("mslot", v, w) not in s.blocks[2]
            assert ("ready", v) in s.blocks[w] and ("mstage", v) not in s.blocks[w]
    S = sum(d.nbytes(v) for v in range(3))
    td, ts = link_traffic(d, 3), link_traffic(s, 3)
    meta = sum(41 if len(x) == 1 else 49 for x in shapes)
    assert td[0]["link_out"] - ts[0]["link_out"] == meta - 3
    assert td[2]["link_in"] - ts[2]["link_in"] == 2 * (meta - 3)
    assert ts[0]["link_out"] == S + 3 and ts[2]["link_out"] == 2 * (S + 3)
    with pytest.raises(errors.InvalidConfig):
        PsLayout(shapes, 2, 1, grad_mechanism="bogus")


def test_missing_library_fails_loudly(monkeypatch):
    """No CPU fallback: without libsrflow.so every entry point raises."""
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libsrflow.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load()
    from paper_1805_08430_b200.memspace import MemorySpace
    with pytest.raises(ImportError):
        MemorySpace(0, 1 << 20)


def test_device_pcg_stream_on_host(tmp_path):
    """device_pcg.cuh (the device GenGrad stream) compiled for the host and
    run over simulated grids: bit-exact vs numpy's Generator(PCG64(mix))
    .random(float32) of the reference's node_rng (graph.py:333-350), for
    even/odd slice starts, 64-bit seeds and one-thread grids."""
    import shutil
    import subprocess
    from oracle import port
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "pcg_host")
    subprocess.check_call([nvcc, "-std=c++17", "-Wno-deprecated-gpu-targets", "-o", exe,
                           os.path.join(root, "tools", "pcg_host_check.cu")])
    out = str(tmp_path / "o.bin")
    for seed, node, it, n, e0, nth in [(0, 0, 2, 262144, 0, 1000), (0, 1, 2, 1003, 0, 64),
                                       (5, 123, 7, 999, 1, 13), (1, 2, 3, 50, 3, 1),
                                       (2**31 + 7, 10**12, 3, 777, 12345, 3),
                                       (0xFFFFFFFF, 2**40, 2**33, 333, 0, 5),
                                       (0, 0, 0, 17, 1, 100)]:
        subprocess.check_call([exe, str(seed), str(node), str(it), str(n), str(e0), str(nth), out])
        got = np.fromfile(out, dtype=np.float32)
        want = port.synthesize(e0 + n, 0, port.node_rng(seed, node, it))[e0:]
        assert got.tobytes() == want.tobytes(), (seed, node, it, n, e0, nth)
        assert got.tobytes() == port.reference_values(seed, node, it, e0, n).tobytes()


def test_reference_harness_times_the_real_reference():
    """oracle/ref_harness.py drives the vendored reference (oracle/_ref, or
    /root/reference here) through its own endpoints; the RPC ring moves the
    same bytes at ~0.2x the zero-copy rate, as in the reference."""
    from oracle import ref_harness as R
    if R.reference() is None:
        pytest.skip("reference not vendored")
    for mech in ("static", "dynamic", "rpc"):
        rig = R.EndpointRig(64 << 10, mech)
        a, b = rig.step(), rig.step()
        assert a == b and 0.0 <= a < 1.0     # ReduceMax of uniform [0, 1) floats
    arm = R.PsArm([(64,), (7, 3)], 2, 1)
    arm.step()


def test_ref_alias_plugin_maps_the_package():
    """tests/ref_alias.py (the reference suite's alias plugin) maps every
    rdmaflow module to this package; benchcli is the reference's own."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not os.path.isdir(os.path.join(root, "oracle", "_ref", "rdmaflow")):
        pytest.skip("reference not vendored")
    code = ("import sys; sys.path[:0] = ['tests', '.']; import ref_alias; "
            "import rdmaflow.runtime.session as s, rdmaflow.memspace as m, rdmaflow.benchcli as b; "
            "assert s.__name__ == 'paper_1805_08430_b200.runtime.session'; "
            "assert m.__name__ == 'paper_1805_08430_b200.memspace'; "
            "assert b.Session is s.Session; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
