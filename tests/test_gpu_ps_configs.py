"""The benchmarked PS configurations at FULL size, on the reference's own
gradient stream, against the golden-pinned oracle (oracle.port.ps_expected).

BASELINE.json configs[2]-[4]: FCN-5 preset (10 x
5,111,750 fp32, 2 workers + 1 PS), LSTM preset (14 x 641,607 fp32, 7 workers +
1 PS, dynamic gradient edges), VGG-16 real shapes (138,357,544 fp32: worker +
PS on separate servers of one GPU, and 4 co-located worker/shard pairs).  The
device produces every gradient itself with the reference's PCG64 stream
(graph.py:333-350 -> device_pcg.cuh); the reference update XOR must be
bit-exact and the north-star SGD within 1e-6 relative (and is bit-exact: same
rounding as the restatement).  One test also uploads the host PCG64 values
(parity mode) to show both sources agree.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import port
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.ps import PsLayout, PsStep
from paper_1805_08430_b200.workloads import preset_slabs, vgg16_shapes

pytestmark = pytest.mark.gpu


def _slabs(name):
    model, nvars = preset_slabs(name)
    return [(model // nvars // 4,)] * nvars


CONFIGS = {
    # name: (shapes, workers, shards, colocate, schedule)
    "fcn5_2w_1ps": (_slabs("fcn-5"), 2, 1, False, "phases"),
    "lstm_7w_1ps": (_slabs("lstm"), 7, 1, False, "exchange"),
    "vgg16_g1": (vgg16_shapes(), 1, 1, False, "phases"),
    "vgg16_coloc4": (vgg16_shapes(), 4, 4, True, "phases"),
}


def _check(ps, L, shapes, W, seed, steps, op, lr):
    want = port.ps_expected(shapes, W, seed, steps, op=op, lr=lr)
    for v in range(len(shapes)):
        got = ps.variable(v)
        if op == "sgd":
            np.testing.assert_allclose(got, want[v], rtol=1e-6, atol=0)
        assert got.tobytes() == want[v].tobytes(), (v, op)


@pytest.mark.parametrize("name", list(CONFIGS))
@pytest.mark.parametrize("op", ["xor", "sgd"])
def test_full_config_on_reference_stream(name, op):
    shapes, W, P, coloc, schedule = CONFIGS[name]
    assert shapes[0][0] in (5_111_750, 641_607) or len(shapes) == 32
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=0, op=op, lr=0.01, schedule=schedule)
    steps = 2 if name == "vgg16_coloc4" else 3
    launches = _lib.launch_count()
    if schedule == "exchange":
        ps.run_exchange(1, steps, per_launch=steps)
    else:
        for it in range(1, steps + 1):
            ps.step(it)
    ps.sync()
    assert _lib.launch_count() > launches
    _check(ps, L, shapes, W, 0, steps, op, 0.01)
    ps.close()


def test_fcn5_parity_upload_equals_device_stream():
    """Host-uploaded PCG64 gradients (parity mode) and device-generated ones
    give the same variables after the same iterations."""
    shapes, W, P, coloc, _ = CONFIGS["fcn5_2w_1ps"]
    L = PsLayout(shapes, W, P, coloc)
    ps = PsStep(L, seed=0, op="xor")
    ps.step(1)
    ps.sync()
    ps.upload_gradients(2)
    ps.step(2, regen=False)
    ps.sync()
    _check(ps, L, shapes, W, 0, 2, "xor", 0.0)
    ps.close()
