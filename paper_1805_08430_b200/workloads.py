"""Graph builders for the benchmark configurations.

``build_microbench``, ``build_layered_forward`` and ``build_ps_workload``
restate rdmaflow ``workloads.py:11-94`` (same node-id order, so plans and
buffer addresses match the reference).  Extensions for the B200 configs
(BASELINE.json configs[2..4]), all opt-in keywords:

* ``shapes=`` per-variable shapes instead of equal slabs (3-layer MLP weights,
  real VGG-16 tensors);
* ``colocate=True`` puts PS shard k on worker k's server (the paper's
  deployment) instead of on servers ``workers..``.
"""
from __future__ import annotations

import math
from typing import Optional, Sequence

from . import errors
from .graph import DataFlowGraph, shape_of
from .wire import ElemType

MLP_DIMS = (16, 12, 10, 4)

#: benchmark presets (model MB, #variables, compute ms/sample), benchcli.py:26-33
PRESETS = {
    "alexnet": (176.42, 16, 7.61),
    "inception-v3": (92.90, 196, 68.32),
    "vggnet-16": (512.32, 32, 30.92),
    "lstm": (35.93, 14, 33.33),
    "gru": (27.92, 11, 30.44),
    "fcn-5": (204.47, 10, 4.88),
}


def vgg16_shapes() -> list[tuple[int, ...]]:
    """The 32 parameter tensors of VGG-16 (13 conv + 3 fc, weights then bias),
    138,357,544 fp32 in total."""
    convs = [(3, 64), (64, 64), (64, 128), (128, 128), (128, 256), (256, 256),
             (256, 256), (256, 512), (512, 512), (512, 512), (512, 512), (512, 512),
             (512, 512)]
    out: list[tuple[int, ...]] = []
    for cin, cout in convs:
        out += [(cout, cin, 3, 3), (cout,)]
    for fin, fout in ((25088, 4096), (4096, 4096), (4096, 1000)):
        out += [(fin, fout), (fout,)]
    return out


def mlp_shapes(dims: Sequence[int] = MLP_DIMS) -> list[tuple[int, ...]]:
    """Weights of the 3-layer MLP of build_layered_forward (workloads.py:31-56)."""
    return [(a, b) for a, b in zip(dims, dims[1:])]


def preset_slabs(name: str, scale: float = 1.0) -> tuple[int, int]:
    """(model bytes, #variables) of a reference preset at ``scale``."""
    mb, nvars, _ms = PRESETS[name]
    return int(mb * 1e6 * scale), nvars


def build_microbench(tensor_bytes: int, elem_type: ElemType = ElemType.F32
                     ) -> tuple[DataFlowGraph, dict[int, int]]:
    """GenGrad on server 0 -> ReduceMax on server 1; one fully static edge."""
    if tensor_bytes < elem_type.size:
        raise errors.InvalidConfig(f"tensor_bytes must be >= {elem_type.size}")
    g = DataFlowGraph()
    payload = g.gen_grad(shape_of(tensor_bytes // elem_type.size), elem_type)
    g.reduce_max(payload)
    g.freeze()
    producer = g.edges[payload].producer
    return g, {n: 0 if n == producer else 1 for n in g.nodes}


def build_layered_forward(batch: int = 8, layer_dims: tuple[int, ...] = MLP_DIMS,
                          with_concat: bool = False
                          ) -> tuple[DataFlowGraph, int, list[int]]:
    """x = sigmoid(x @ W + B) per layer; optional dynamic concat after the input.
    Returns (graph, input edge, edges in the dynamic cone)."""
    g = DataFlowGraph()
    x = g.input(shape_of(batch, layer_dims[0]))
    cone: list[int] = []
    if with_concat:
        x = g.concat_dyn([x], dyn_range=(1, 2 * batch))
        cone.append(x)
    first = x
    for d_in, d_out in zip(layer_dims, layer_dims[1:]):
        w = g.variable(shape_of(d_in, d_out))
        b = g.input(shape_of(batch, d_out))
        h = g.matmul(x, w)
        a = g.add(h, b)
        x = g.sigmoid(a)
        if with_concat:
            cone += [h, a, x]
    g.freeze()
    return g, first, cone


def build_ps_workload(model_size: int, num_variables: int, compute_time: float,
                      workers: int, *, ps_servers: int = 1,
                      elem_type: ElemType = ElemType.F32,
                      shapes: Optional[Sequence[tuple[int, ...]]] = None,
                      colocate: bool = False
                      ) -> tuple[DataFlowGraph, dict[int, int]]:
    """Data-parallel PS skeleton: variable v on shard ``v % ps_servers``; per
    worker a GenGrad consumes the pulled weight and an ApplyGrad folds the
    pushed gradient into the variable in place.  Workers are servers
    ``0..workers-1``; shards are servers ``workers..`` (or the workers
    themselves with ``colocate``)."""
    if workers < 1 or ps_servers < 1 or num_variables < 1:
        raise errors.InvalidConfig("workers, ps_servers and num_variables must be >= 1")
    if colocate and ps_servers > workers:
        raise errors.InvalidConfig("colocate needs ps_servers <= workers")
    if shapes is None:
        slab = model_size // num_variables // elem_type.size
        if slab < 1:
            raise errors.InvalidConfig(
                f"model of {model_size} bytes cannot be divided into "
                f"{num_variables} variables of whole {elem_type.name} elements")
        shapes = [(slab,)] * num_variables
    else:
        shapes = [tuple(int(d) for d in s) for s in shapes]
        if len(shapes) != num_variables:
            raise errors.InvalidConfig("len(shapes) must equal num_variables")
    per_node = compute_time / num_variables

    g = DataFlowGraph()
    placement: dict[int, int] = {}
    for v, dims in enumerate(shapes):
        shard = (v % ps_servers) + (0 if colocate else workers)
        weight = g.variable(shape_of(*dims), elem_type)
        placement[g.edges[weight].producer] = shard
        for w in range(workers):
            grad = g.gen_grad(shape_of(*dims), elem_type, inputs=(weight,),
                              compute_time=per_node)
            placement[g.edges[grad].producer] = w
            upd = g.apply_grad(weight, grad)
            placement[g.edges[upd].producer] = shard
    g.freeze()
    return g, placement


def ps_node_ids(num_variables: int, workers: int, v: int, w: int) -> tuple[int, int, int]:
    """(variable, GenGrad, ApplyGrad) node ids of variable v / worker w in a
    build_ps_workload graph: var = v(1+2W), gen = var+1+2w, apply = var+2+2w."""
    var = v * (1 + 2 * workers)
    return var, var + 1 + 2 * w, var + 2 + 2 * w


def total_params(shapes: Sequence[tuple[int, ...]]) -> int:
    return sum(math.prod(s) for s in shapes)
