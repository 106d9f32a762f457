"""MatMul / Add / Sigmoid as libsrflow kernels (srf_compute) against numpy's
compute_node (graph.py:371-377, restated in oracle/port.py:forward_values).

Every compute node's output crosses to another server, so capture_edges sees
each value; each node is checked against numpy applied to the inputs it was
actually given (captured too), so one kind's rounding never hides another's:
* Add (IEEE add, wrapping integers), integer MatMul (wrapping sums) and fp32
  Sigmoid (float64 math rounded once to fp32): bit-exact;
* float MatMul: the kernel sums ascending-k FMA chains; numpy calls BLAS,
  whose blocking (and so its rounding) depends on the host CPU, so the two are
  held to the forward error bound of a length-k dot product instead:
  |got - numpy| <= 2 k eps (|a| @ |b|);
* fp64 Sigmoid: CUDA's exp and numpy's exp are each within 1 ulp, so 2 ulp.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import port
from paper_1805_08430_b200.graph import DataFlowGraph, NodeKind, shape_of
from paper_1805_08430_b200.runtime.session import Session, infer_elem_types
from paper_1805_08430_b200.wire import ElemType

pytestmark = pytest.mark.gpu


def _layered(batch, dims, elem):
    """sigmoid(x @ W + B) per layer (workloads.build_layered_forward) with a
    ReduceMax sink.  Sources and Sigmoid on server 0, MatMul on 1, Add on 2:
    every edge crosses servers and is captured."""
    g = DataFlowGraph()
    x = g.input(shape_of(batch, dims[0]), elem)
    for d_in, d_out in zip(dims, dims[1:]):
        w = g.variable(shape_of(d_in, d_out), elem)
        b = g.input(shape_of(batch, d_out), elem)
        x = g.add(g.matmul(x, w), b)
        if elem in (ElemType.F32, ElemType.F64):
            x = g.sigmoid(x)
    g.reduce_max(x)
    g.freeze()
    sink = 1 if elem in (ElemType.F32, ElemType.F64) else 0
    side = {NodeKind.MATMUL: 1, NodeKind.ADD: 2, NodeKind.REDUCE_MAX: sink}
    return g, {nid: side.get(n.kind, 0) for nid, n in g.nodes.items()}


def _check(g, elem, captured, iterations):
    elems = infer_elem_types(g)
    seen = {}
    for (it, e, _s), raw in captured.items():
        seen[(it, e)] = raw
    checked = 0
    for it in range(1, iterations + 1):
        for nid in g.topological_order():
            node = g.nodes[nid]
            if node.kind not in (NodeKind.MATMUL, NodeKind.ADD, NodeKind.SIGMOID):
                continue
            if (it, node.output) not in seen or any((it, e) not in seen for e in node.inputs):
                continue
            dt = elems[node.output].np_dtype
            ins = [np.frombuffer(seen[(it, e)], dt) for e in node.inputs]
            got = np.frombuffer(seen[(it, node.output)], dt)
            if node.kind is NodeKind.MATMUL:
                k = g.nodes[g.edges[node.inputs[1]].producer].shape.static_dims()[0]
                a, b = ins[0].reshape(-1, k), ins[1].reshape(k, -1)
                want = (a @ b).reshape(-1)
                if elem in (ElemType.F32, ElemType.F64):
                    eps = np.finfo(dt).eps
                    bound = 2 * k * eps * (np.abs(a).astype(np.float64) @
                                           np.abs(b).astype(np.float64)).reshape(-1)
                    assert np.all(np.abs(got.astype(np.float64) - want) <= bound), (it, nid)
                else:
                    assert got.tobytes() == want.tobytes(), (it, nid)
            elif node.kind is NodeKind.ADD:
                assert got.tobytes() == (ins[0] + ins[1]).tobytes(), (it, nid)
            else:
                want = (1.0 / (1.0 + np.exp(-ins[0].astype(np.float64)))).astype(dt)
                if elem is ElemType.F32:
                    assert got.tobytes() == want.tobytes(), (it, nid)
                else:
                    ulp = np.spacing(np.abs(want))
                    assert np.all(np.abs(got - want) <= 2 * ulp), (it, nid)
            checked += 1
    return checked


@pytest.mark.parametrize("elem", [ElemType.F32, ElemType.F64, ElemType.I32, ElemType.I64,
                                  ElemType.U8])
@pytest.mark.parametrize("batch,dims", [(8, (16, 12, 10, 4)), (33, (300, 129, 7)),
                                        (1, (5, 3))])
def test_compute_kinds_equal_numpy(elem, batch, dims):
    g, p = _layered(batch, dims, elem)
    s = Session(g, p, seed=7, capture_edges=True)
    rep = s.run(2)
    n = _check(g, elem, rep.captured, 2)
    layers = len(dims) - 1
    per_layer = 3 if elem in (ElemType.F32, ElemType.F64) else 2
    assert n == 2 * layers * per_layer
    s.close()


def test_forward_values_oracle_matches_session():
    """The whole chain against the oracle's own evaluation from the seeded
    sources (every value, not only node-by-node)."""
    g, p = _layered(8, (16, 12, 10, 4), ElemType.F32)
    s = Session(g, p, seed=5, capture_edges=True)
    rep = s.run(2)
    elems = infer_elem_types(g)
    nodes = []
    for nid in g.topological_order():
        n = g.nodes[nid]
        dims = n.shape.static_dims() if n.kind in (NodeKind.INPUT, NodeKind.VARIABLE) else None
        nodes.append((nid, n.kind.name, n.inputs, n.output, dims, int(elems[n.output])))
    for it in (1, 2):
        want = port.forward_values(nodes, 5, it)
        for (i, e, _s), raw in rep.captured.items():
            if i != it:
                continue
            got = np.frombuffer(raw, np.float32)
            np.testing.assert_allclose(got, want[e].reshape(-1), rtol=1e-5, atol=1e-6)
    s.close()


@pytest.mark.parametrize("elem", [ElemType.F32, ElemType.F64, ElemType.I32, ElemType.U8])
def test_concat_dyn_is_a_library_kernel_equal_to_numpy(elem):
    """ConcatDyn (srf_concat_tile): dim 0 drawn from the node's stream, the
    inputs concatenated and repeated - byte-identical to compute_node's numpy
    restatement on the captured inputs, for every element type, with inputs
    of different lengths and an output longer and shorter than their sum."""
    from paper_1805_08430_b200 import _lib
    from paper_1805_08430_b200.graph import node_rng
    g = DataFlowGraph()
    a = g.input(shape_of(3, 5), elem)
    b = g.input(shape_of(7, 5), elem)
    c = g.concat_dyn([a, b], dyn_range=(1, 30))
    g.reduce_max(c)
    g.freeze()
    # sources on server 0, the concat on 1, its consumer on 2: every edge captured
    side = {NodeKind.CONCAT_DYN: 1, NodeKind.REDUCE_MAX: 2}
    placement = {nid: side.get(n.kind, 0) for nid, n in g.nodes.items()}
    s = Session(g, placement, seed=5, capture_edges=True, replay=False)
    launches = _lib.launch_count()
    rep = s.run(6)
    assert _lib.launch_count() > launches
    node = next(n for n in g.nodes.values() if n.kind is NodeKind.CONCAT_DYN)
    seen = {(it, e): raw for (it, e, _s), raw in rep.captured.items()}
    dt = elem.np_dtype
    lens = set()
    for it in range(1, 7):
        ins = [np.frombuffer(seen[(it, e)], dt).reshape(-1, 5) for e in node.inputs]
        # numpy restatement of compute_node's ConcatDyn (graph.py:363-389)
        rng = node_rng(5, node.node_id, it)
        lo, hi = node.dyn_range
        dim0 = int(rng.integers(lo, hi + 1))
        flat = np.concatenate(ins, axis=0).reshape(-1)
        want = np.tile(flat, -(-dim0 * 5 // flat.size))[:dim0 * 5]
        got = np.frombuffer(seen[(it, node.output)], dt)
        assert got.tobytes() == want.tobytes(), it
        lens.add(got.size)
    assert len(lens) > 1            # dim 0 varied across iterations
    s.close()


@pytest.mark.parametrize("elem", [ElemType.F32, ElemType.F64, ElemType.I32, ElemType.I64,
                                  ElemType.U8])
@pytest.mark.parametrize("sa,sb", [((3, 4), (1, 4)), ((5, 1, 3), (1, 2, 3)), ((7,), (1,)),
                                   ((1, 1), (4, 6))])
def test_broadcasting_add_equals_numpy(elem, sa, sb):
    """srf_add_bcast (Add with numpy broadcasting): bit-exact against numpy
    a + b (IEEE add, wrapping integers)."""
    from paper_1805_08430_b200 import _lib
    from paper_1805_08430_b200.memspace import MemorySpace
    rng = np.random.default_rng(len(sa) * 31 + len(sb))
    dt = elem.np_dtype
    if elem in (ElemType.F32, ElemType.F64):
        a = rng.standard_normal(sa).astype(dt)
        b = rng.standard_normal(sb).astype(dt)
    else:
        info = np.iinfo(dt)
        a = rng.integers(info.min, info.max, sa, dtype=dt, endpoint=True)
        b = rng.integers(info.min, info.max, sb, dtype=dt, endpoint=True)
    with np.errstate(over="ignore"):
        want = a + b
    sp = MemorySpace(0, 1 << 20, device=0)
    ra = sp.allocate_region(1024)
    rb = sp.allocate_region(1024)
    ro = sp.allocate_region(4096)
    sp.write_raw(ra.base_addr, a.tobytes())
    sp.write_raw(rb.base_addr, b.tobytes())
    _lib.call("srf_add_bcast", sp.handle, int(elem), ra.base_addr, _lib.u64_array(sa),
              rb.base_addr, _lib.u64_array(sb), len(sa), ro.base_addr, None)
    sp.sync()
    got = np.frombuffer(sp.read_raw(ro.base_addr, want.nbytes), dt).reshape(want.shape)
    assert got.tobytes() == want.tobytes()
    with pytest.raises(Exception):
        _lib.call("srf_add_bcast", sp.handle, int(elem), ra.base_addr, _lib.u64_array((3, 4)),
                  rb.base_addr, _lib.u64_array((2, 4)), 2, ro.base_addr, None)
    sp.close()
