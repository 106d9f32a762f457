"""srf_gen_reference / the PS gen batch: the reference's GenGrad values
(graph.py:333-350, numpy PCG64 via SeedSequence, float32 = 24-bit halves)
produced on the device, bit-exact against numpy (oracle.port)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle import port
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.memspace import MemorySpace

pytestmark = pytest.mark.gpu


def _gen(sp, reg, n, e0, seed, node, it):
    _lib.call("srf_gen_reference", sp.handle, reg.base_addr, n, e0, seed, node, it, None, None)
    sp.sync()
    return np.frombuffer(sp.read_raw(reg.base_addr, 4 * n), np.float32)


@pytest.mark.parametrize("n,e0,seed,node,it", [
    (1, 0, 0, 0, 0), (7, 0, 0, 1, 2), (8, 0, 0, 1, 2), (9, 1, 3, 4, 5),
    (1 << 20, 0, 0, 0, 2),                # configs[0]: build_microbench(1 MiB), it 2
    (262_143, 12_345, 7, 99, 3),          # odd start (a partitioned slice)
    (5_111_750, 0, 0, 11, 1),             # one FCN-5 slab
    (641_607, 641_607, 2**32 + 5, 2**40, 2**33),  # 64-bit mix, multi-word entropy
])
def test_device_stream_equals_numpy(n, e0, seed, node, it):
    sp = MemorySpace(0, 4 * n + (1 << 20), seed=0, device=0)
    reg = sp.allocate_region(4 * n + 64, register=True)
    got = _gen(sp, reg, n, e0, seed, node, it)
    want = port.reference_values(seed, node, it, e0, n)
    assert got.tobytes() == want.tobytes()
    if e0 == 0 and n <= (1 << 20):
        assert got.tobytes() == port.synthesize(n, 0, port.node_rng(seed, node, it)).tobytes()
    sp.close()


@pytest.mark.parametrize("offset", [4, 8, 12])
@pytest.mark.parametrize("n,e0", [(3, 0), (1001, 0), (1001, 7), (70_000, 2)])
def test_unaligned_destination(offset, n, e0):
    """Arena blocks are only 8-B aligned (memspace.py:31): the head floats
    before the first 16-B boundary take the scalar path."""
    sp = MemorySpace(0, 1 << 20, seed=0, device=0)
    reg = sp.allocate_region(4 * n + 64, register=True)
    guard = b"\xee" * 16
    sp.write_raw(reg.base_addr, guard)
    sp.write_raw(reg.base_addr + offset + 4 * n, guard)
    _lib.call("srf_gen_reference", sp.handle, reg.base_addr + offset, n, e0, 3, 5, 6, None,
              None)
    sp.sync()
    got = np.frombuffer(sp.read_raw(reg.base_addr + offset, 4 * n), np.float32)
    assert got.tobytes() == port.reference_values(3, 5, 6, e0, n).tobytes()
    assert sp.read_raw(reg.base_addr, offset) == guard[:offset]
    assert sp.read_raw(reg.base_addr + offset + 4 * n, 16) == guard
    sp.close()


def test_c1_golden_first_values(golden):
    """configs[0] payload: first four floats and the fp64 sum."""
    doc, _ = golden
    n = 1 << 18
    sp = MemorySpace(0, 4 << 20, seed=0, device=0)
    reg = sp.allocate_region(4 * n, register=True)
    got = _gen(sp, reg, n, 0, 0, 0, 2)
    assert [float(x) for x in got[:4]] == doc["c1"]["first4"]
    assert float(got.astype(np.float64).sum()) == pytest.approx(doc["c1"]["sum64"], abs=1e-9)
    sp.close()


def test_vgg_fc6_sized_stream():
    """The largest real VGG-16 tensor (fc6, 25088 x 4096 = 102.8 M fp32)."""
    n = 25088 * 4096
    sp = MemorySpace(0, 4 * n + (1 << 20), seed=0, device=0)
    reg = sp.allocate_region(4 * n, register=True)
    got = _gen(sp, reg, n, 0, 0, 29, 1)
    want = port.synthesize(n, 0, port.node_rng(0, 29, 1))
    assert got.tobytes() == want.tobytes()
    sp.close()
