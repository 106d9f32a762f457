"""Device-driven PS step (paper_1805_08430_b200.ps) vs the oracle: the
reference's XOR update bit-exact (pinned by the golden PS runs through
oracle.port.ps_expected) and SGD (unpinned restatement), in parity mode
(host-uploaded PCG64 gradients) and regen mode (the device generates the
reference's own PCG64 GenGrad stream, device_pcg.cuh) - both checked against
the same golden-pinned ps_expected."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import port
from paper_1805_08430_b200 import _lib, errors
from paper_1805_08430_b200.ps import PsLayout, PsStep
from paper_1805_08430_b200.workloads import mlp_shapes

pytestmark = pytest.mark.gpu

CASES = [
    # (shapes, workers, shards, colocate)
    ([(1000,), (37,), (4, 9)], 1, 1, False),             # G=1: worker + PS on one GPU
    (mlp_shapes(), 2, 1, False),                          # configs[2] parity set
    ([(3000,), (17,), (64, 64), (5,)], 4, 4, True),       # co-located shards
    ([(641,)] * 3, 7, 1, False),                          # configs[4] shape: 7 workers
]


@pytest.mark.parametrize("shapes,W,P,coloc", CASES)
@pytest.mark.parametrize("op", ["xor", "sgd"])
def test_parity_mode_matches_oracle(shapes, W, P, coloc, op):
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=3, op=op, lr=0.05)
    launches = _lib.launch_count()
    for it in (1, 2, 3):
        ps.upload_gradients(it)
        ps.step(it, regen=False)
        ps.sync()
    assert _lib.launch_count() - launches >= 3 * 3
    want = port.ps_expected(shapes, W, 3, 3, op=op, lr=0.05)
    for v in range(len(shapes)):
        got = ps.variable(v)
        if op == "sgd":
            np.testing.assert_allclose(got, want[v], rtol=1e-6, atol=0)
        assert got.tobytes() == want[v].tobytes(), (v, op)
    ps.close()


@pytest.mark.parametrize("shapes,W,P,coloc", CASES[:3])
def test_regen_mode_pipelined(shapes, W, P, coloc):
    """Back-to-back device iterations (no host sync between steps): the
    credit/flag protocol alone orders the phases."""
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=9, op="sgd", lr=0.01)
    for it in range(1, 9):
        ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 9, 8, op="sgd", lr=0.01)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes()
    ps.close()


def test_device_gradient_is_the_reference_stream():
    """GenGrad on the device = synthesize_values(F32, node_rng(seed, gen, it))."""
    L = PsLayout([(1031,)], 1, 1, False)
    ps = PsStep(L, seed=5)
    ps.step(7)
    ps.sync()
    g = np.frombuffer(ps.spaces[0].read_raw(ps.addr(0, ("grad", 0)), 1031 * 4), np.float32)
    want = port.synthesize(1031, 0, port.node_rng(5, port.ps_node_ids(0, 0, 1)[1], 7))
    assert g.tobytes() == want.tobytes()
    ps.close()


def test_meta_blocks_are_reference_bytes():
    from paper_1805_08430_b200.wire import ElemType, encode_meta
    L = PsLayout([(10, 3)], 2, 1, False)
    ps = PsStep(L, seed=1)
    ps.step(1)
    ps.sync()
    for w in (0, 1):
        stage = ps.spaces[w].read_raw(ps.addr(w, ("mstage", 0)), 49)
        assert stage == port.encode_meta((10, 3), 0, ps.addr(w, ("grad", 0)), ps.token(w))
        assert stage == encode_meta((10, 3), ElemType.F32, ps.addr(w, ("grad", 0)), ps.token(w))
    # the shard consumed and cleared every meta flag
    for w in (0, 1):
        assert ps.spaces[2].read_raw(ps.addr(2, ("mslot", 0, w)) + 48, 1) == b"\x00"
    ps.close()


def test_bad_token_in_meta_is_rejected():
    L = PsLayout([(256,)], 2, 1, False)
    ps = PsStep(L, seed=1)
    # corrupt worker 1's metadata token (offset 16 + 8*rank, wire.py layout)
    raw = bytearray(ps.spaces[1].read_raw(ps.addr(1, ("mstage", 0)), 41))
    raw[24] ^= 0xFF
    ps.spaces[1].write_raw(ps.addr(1, ("mstage", 0)), bytes(raw))
    before = ps.variable(0).copy()
    ps.step(1)
    with pytest.raises(errors.BadToken):
        ps.sync()
    assert ps.variable(0).tobytes() == before.tobytes()  # no update applied


def test_out_of_range_meta_address_is_rejected():
    L = PsLayout([(256,)], 2, 1, False)
    ps = PsStep(L, seed=1)
    raw = bytearray(ps.spaces[0].read_raw(ps.addr(0, ("mstage", 0)), 41))
    raw[16:24] = (1 << 40).to_bytes(8, "little")  # remote_addr (after dims) out of range
    ps.spaces[0].write_raw(ps.addr(0, ("mstage", 0)), bytes(raw))
    ps.step(1)
    with pytest.raises(errors.BadToken):
        ps.sync()


def test_inconsistent_meta_dims_are_rejected():
    L = PsLayout([(256,)], 2, 1, False)
    ps = PsStep(L, seed=1)
    raw = bytearray(ps.spaces[0].read_raw(ps.addr(0, ("mstage", 0)), 41))
    raw[8:16] = (255).to_bytes(8, "little")  # dims no longer match payload_len
    ps.spaces[0].write_raw(ps.addr(0, ("mstage", 0)), bytes(raw))
    ps.step(1)
    with pytest.raises(errors.BadToken):
        ps.sync()


def test_graph_replayed_steps_match_eager():
    """CUDA-graph capture of several iterations: the gen batch reads the
    iteration from the device counter the captured steps advance."""
    shapes, W, P = mlp_shapes(), 2, 1
    L = PsLayout(shapes, W, P, False)
    ps = PsStep(L, seed=4, op="sgd", lr=0.02)
    ps.step(1)
    ps.set_iteration(2)
    g = ps.capture(5)
    ps.replay(g)
    ps.sync()
    want = port.ps_expected(shapes, W, 4, 6, op="sgd", lr=0.02)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes()
    _lib.call("srf_graph_destroy", g)
    ps.close()


@pytest.mark.parametrize("shapes,W,P,coloc", CASES)
def test_persistent_step_matches_oracle(shapes, W, P, coloc):
    """All four phases of many iterations in one cooperative launch."""
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=6, op="sgd", lr=0.03)
    ps.step(1)
    ps.run_persistent(2, 6)
    ps.step(8)
    ps.sync()
    want = port.ps_expected(shapes, W, 6, 8, op="sgd", lr=0.03)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes()
    ps.close()


@pytest.mark.parametrize("shapes,W,P,coloc", CASES)
@pytest.mark.parametrize("lag,order", [(1, "index"), (0, "index"), (2, "size")])
def test_exchange_schedule_matches_oracle(shapes, W, P, coloc, lag, order):
    """One k_ps_exchange launch per iteration (dependency-ordered work queue,
    metadata puts fused into the gradient producer): same bytes as the phases."""
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=12, op="sgd", lr=0.03, schedule="exchange", exchange_lag=lag,
                exchange_order=order)
    launches = _lib.launch_count()
    for it in range(1, 7):
        assert ps.step(it) == 1
    ps.sync()
    assert _lib.launch_count() - launches == 6
    want = port.ps_expected(shapes, W, 12, 6, op="sgd", lr=0.03)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), (v, lag, order)
    # parity mode (reference PCG64 gradients uploaded), XOR
    ps.close()
    ps = PsStep(L, seed=3, op="xor", schedule="exchange", exchange_lag=lag,
                exchange_order=order)
    for it in (1, 2, 3):
        ps.upload_gradients(it)
        ps.step(it, regen=False)
        ps.sync()
    want = port.ps_expected(shapes, W, 3, 3, op="xor")
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes()
    ps.close()


def test_exchange_schedule_mixes_with_phases():
    """Phase launches and exchange launches share flags and credits: a run
    that alternates them matches the oracle."""
    shapes, W, P = mlp_shapes(), 2, 1
    L = PsLayout(shapes, W, P, False)
    ps = PsStep(L, seed=2, op="sgd", lr=0.01, schedule="exchange")
    for it in range(1, 7):
        ps.use_schedule("exchange" if it % 2 else "phases")
        ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 2, 6, op="sgd", lr=0.01)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes()
    ps.close()


@pytest.mark.parametrize("placement", ["round_robin", "bytes"])
def test_partitioned_variables_equal_the_model(placement):
    """EXTENSION: variables cut into one slice per shard; gathering the slices
    gives exactly the unpartitioned model's values (device and PCG64 grads)."""
    shapes, W, P = [(3000,), (17,), (64, 70), (5,)], 3, 3
    L = PsLayout(shapes, W, P, True, placement=placement, partition_bytes=4096)
    assert len(L.shapes) > len(shapes)
    for op, regen in (("sgd", True), ("xor", False)):
        ps = PsStep(L, seed=8, op=op, lr=0.02)
        for it in range(1, 5):
            if not regen:
                ps.upload_gradients(it)
            ps.step(it, regen=regen)
            if not regen:
                ps.sync()
        ps.sync()
        want = (port.ps_expected(shapes, W, 8, 4, op=op, lr=0.02) if regen
                else port.ps_expected(shapes, W, 8, 4, op=op))
        got = [np.zeros(int(np.prod(s)), np.float32) for s in shapes]
        for u in range(len(L.shapes)):
            v, off, n = L.parent(u)
            got[v][off:off + n] = ps.variable(u).reshape(-1)
        for v in range(len(shapes)):
            assert got[v].tobytes() == want[v].reshape(-1).tobytes(), (op, v)
        ps.close()


@pytest.mark.parametrize("schedule", ["phases", "exchange"])
def test_sliced_variables_equal_the_model(schedule):
    """EXTENSION: variables cut into slices on their own shard (pipelined
    transfers); the gathered slices equal the unsliced model bit for bit,
    including several iterations per exchange launch."""
    shapes, W, P = [(3000,), (17,), (64, 70), (5,)], 3, 3
    L = PsLayout(shapes, W, P, True, slice_bytes=2048)
    assert len(L.shapes) > len(shapes)
    ps = PsStep(L, seed=9, op="sgd", lr=0.02, schedule=schedule)
    if schedule == "exchange":
        ps.run_exchange(1, 6, per_launch=3)
    else:
        for it in range(1, 7):
            ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 9, 6, op="sgd", lr=0.02)
    got = [np.zeros(int(np.prod(s)), np.float32) for s in shapes]
    for u in range(len(L.shapes)):
        v, off, n = L.parent(u)
        got[v][off:off + n] = ps.variable(u).reshape(-1)
    for v in range(len(shapes)):
        assert got[v].tobytes() == want[v].reshape(-1).tobytes(), v
    ps.close()


def test_exchange_waits_for_in_place_gradients():
    """Co-located worker/shard: the apply reads the worker's gradient in place,
    so in the single-launch exchange it must wait for the gradient's ready
    byte (an apply unit can be claimed while that gradient is still being
    produced).  Large gradients, lag 0: the window is wide."""
    shapes, W, P = [(1 << 22,), (1 << 21,), (3,)], 2, 2
    L = PsLayout(shapes, W, P, True)
    ps = PsStep(L, seed=17, op="sgd", lr=0.01, schedule="exchange", exchange_lag=0)
    for it in range(1, 6):
        ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 17, 5, op="sgd", lr=0.01)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), v
    ps.close()


@pytest.mark.parametrize("shapes,W,P,coloc", CASES + [([(1 << 20,), (7,)], 2, 2, True)])
@pytest.mark.parametrize("per_launch", [3, 64])
def test_multi_iteration_exchange_matches_oracle(shapes, W, P, coloc, per_launch):
    """Several iterations per k_ps_exchange launch: a push of iteration k waits
    for its variable's apply of iteration k-1 inside the launch."""
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=31, op="sgd", lr=0.02)
    ps.step(1)
    assert ps.run_exchange(2, 10, per_launch=per_launch) == -(-10 // per_launch)
    ps.use_schedule("phases")
    ps.step(12)
    ps.sync()
    want = port.ps_expected(shapes, W, 31, 12, op="sgd", lr=0.02)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), v
    ps.close()


@pytest.mark.parametrize("shapes,W,P,coloc", CASES + [([(1 << 20,), (7,)], 2, 2, True)])
@pytest.mark.parametrize("schedule", ["phases", "exchange", "exchange_x3", "persistent",
                                      "mixed"])
def test_static_gradients_match_oracle(shapes, W, P, coloc, schedule):
    """Gradient edges forced STATIC (the reference's mechanism_override="static",
    runtime/session.py:368): workers put gradient || flag into the shard's
    receive regions; same values as the dynamic path under every schedule."""
    L = PsLayout(shapes, W, P, coloc, grad_mechanism="static")
    assert not any(k[0] in ("mslot", "mstage") for b in L.blocks.values() for k in b
                   if isinstance(k, tuple))
    ps = PsStep(L, seed=21, op="sgd", lr=0.02,
                schedule="exchange" if schedule == "exchange" else "phases")
    if schedule == "exchange_x3":
        ps.run_exchange(1, 8, per_launch=3)
    elif schedule == "persistent":
        ps.step(1)
        ps.run_persistent(2, 6)
        ps.step(8)
    else:
        for it in range(1, 9):
            if schedule == "mixed":
                ps.use_schedule("exchange" if it % 2 else "phases")
            ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 21, 8, op="sgd", lr=0.02)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), (v, schedule)
    ps.close()
    if schedule == "phases":  # parity mode: reference PCG64 gradients uploaded, XOR
        ps = PsStep(L, seed=3, op="xor")
        for it in (1, 2, 3):
            ps.upload_gradients(it)
            ps.step(it, regen=False)
            ps.sync()
        want = port.ps_expected(shapes, W, 3, 3, op="xor")
        for v in range(len(shapes)):
            assert ps.variable(v).tobytes() == want[v].tobytes()
        ps.close()


def test_static_sliced_gradients_equal_the_model():
    shapes, W, P = [(3000,), (17,), (64, 70), (5,)], 3, 3
    L = PsLayout(shapes, W, P, True, slice_bytes=2048, grad_mechanism="static")
    ps = PsStep(L, seed=9, op="sgd", lr=0.02, schedule="exchange")
    ps.run_exchange(1, 6, per_launch=4)
    ps.sync()
    want = port.ps_expected(shapes, W, 9, 6, op="sgd", lr=0.02)
    got = [np.zeros(int(np.prod(s)), np.float32) for s in shapes]
    for u in range(len(L.shapes)):
        v, off, n = L.parent(u)
        got[v][off:off + n] = ps.variable(u).reshape(-1)
    for v in range(len(shapes)):
        assert got[v].tobytes() == want[v].reshape(-1).tobytes(), v
    ps.close()


@pytest.mark.parametrize("lane", [1, 3, 128])
@pytest.mark.parametrize("grad", ["static", "dynamic"])
def test_push_lane_exchange_matches_oracle(monkeypatch, lane, grad):
    """Two-lane exchange (SRFLOW_PS_PUSH_CTAS: the first `lane` CTAs claim the
    pushes, the rest GenGrad and the applies, each lane in the global order):
    bit-identical variables, several iterations per launch, with as few as one
    push CTA (on one GPU the lanes only activate through the knob; across GPUs
    128 is the default)."""
    monkeypatch.setenv("SRFLOW_PS_PUSH_CTAS", str(lane))
    shapes, W, P = [(3000,), (17,), (64, 70), (5,)], 3, 3
    L = PsLayout(shapes, W, P, True, slice_bytes=2048, grad_mechanism=grad)
    ps = PsStep(L, seed=9, op="sgd", lr=0.02, schedule="exchange")
    ps.run_exchange(1, 7, per_launch=3)
    ps.sync()
    want = port.ps_expected(shapes, W, 9, 7, op="sgd", lr=0.02)
    got = [np.zeros(int(np.prod(s)), np.float32) for s in shapes]
    for u in range(len(L.shapes)):
        v, off, n = L.parent(u)
        got[v][off:off + n] = ps.variable(u).reshape(-1)
    for v in range(len(shapes)):
        assert got[v].tobytes() == want[v].reshape(-1).tobytes(), (v, lane, grad)
    ps.close()


@pytest.mark.parametrize("shapes,W,P,coloc", CASES)
@pytest.mark.parametrize("op", ["xor", "sgd"])
def test_fused_weight_push_matches_oracle(shapes, W, P, coloc, op):
    """PsStep(fuse_push=True): the apply of iteration k also writes the
    updated variable into every remote worker's weight receive region (the
    next iteration's weight push).  Back-to-back steps, toggling the fusion
    off and on between steps, equal the golden-pinned oracle; the forwarded
    weights equal the variable, flag set."""
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=21, op=op, lr=0.03, fuse_push=True)
    it = 0
    for fused in (True, True, False, True, True, True, False, False, True):
        ps.fuse_push = fused
        it += 1
        ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 21, it, op=op, lr=0.03)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), (v, op)
    # the last step forwarded: every remote worker holds the current weights
    for v in range(len(shapes)):
        s = L.shard_of(v)
        for w in range(W):
            if w == s:
                continue
            raw = ps.space(w).read_raw(ps.addr(w, ("wbuf", v)), L.nbytes(v) + 1)
            assert raw[:-1] == want[v].tobytes() and raw[-1] == 1, (v, w)
    with pytest.raises(errors.InvalidConfig):
        ps.run_persistent(it + 1, 1)   # a forwarded push is outstanding
    ps.fuse_push = False
    it += 1
    ps.step(it)                         # consumes it, pushes nothing
    ps.use_schedule("exchange")
    it += 1
    ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 21, it, op=op, lr=0.03)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), (v, op, "after the switch")
    ps.close()


def test_fused_weight_push_graph_replay():
    shapes = [(5000,), (33,), (16, 16)]
    L = PsLayout(shapes, 2, 1)
    ps = PsStep(L, seed=4, op="sgd", lr=0.02, fuse_push=True)
    ps.step(1)
    ps.sync()
    ps.set_iteration(2)
    graph = ps.capture(5)
    ps.replay(graph)
    ps.replay(graph)          # iterations 2..11 (the counter advances per step)
    ps.sync()
    _lib.call("srf_graph_destroy", graph)
    want = port.ps_expected(shapes, 2, 4, 11, op="sgd", lr=0.02)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), v
    ps.close()


@pytest.mark.parametrize("shapes,W,P,coloc", CASES)
@pytest.mark.parametrize("static", [False, True])
def test_fused_weight_push_in_the_exchange(shapes, W, P, coloc, static):
    """The exchange schedule with the fused weight push: the exchange built
    without weight pushes, applies forwarding; single- and multi-iteration
    launches, switching fusion on and off between launches and between
    schedules, all equal the oracle."""
    L = PsLayout(shapes, W, P, coloc, grad_mechanism="static" if static else "dynamic")
    ps = PsStep(L, seed=23, op="sgd", lr=0.02, schedule="exchange", fuse_push=True)
    it = 0
    for fused, how in ((True, "step"), (True, "multi"), (False, "step"), (True, "multi"),
                       (False, "multi"), (True, "phases"), (True, "step"), (False, "multi")):
        ps.fuse_push = fused
        if how == "multi":
            ps.run_exchange(it + 1, 4, per_launch=2)
            it += 4
        else:
            ps.use_schedule("phases" if how == "phases" else "exchange")
            it += 1
            ps.step(it)
    ps.sync()
    want = port.ps_expected(shapes, W, 23, it, op="sgd", lr=0.02)
    for v in range(len(shapes)):
        assert ps.variable(v).tobytes() == want[v].tobytes(), v
    ps.close()
