"""Host cost of each primitive one dynamic transfer through the public API is
made of (tools/dyn_breakdown.py times the four calls; this times their
parts in isolation, R iterations each, microseconds per call)."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.analyzer import PlanEntry
from paper_1805_08430_b200.fabric import Fabric, MemRange
from paper_1805_08430_b200.graph import Tensor, shape_of
from paper_1805_08430_b200.memspace import ArenaAllocator, BufferRef, MemorySpace
from paper_1805_08430_b200.runtime.protocol import DynReceiver, DynSender
from paper_1805_08430_b200.wire import ElemType, Mechanism, encode_meta, meta_block_size

R = 2000
size = 4096
fab = Fabric()
sp = {s: MemorySpace(s, 16 << 20, device=0) for s in (0, 1)}
ar = {s: ArenaAllocator(sp[s], sp[s].allocate_region(8 << 20, True)) for s in (0, 1)}
dv = {s: fab.create_device(sp[s], qps_per_peer=2) for s in (0, 1)}
fwd = dv[0].connect(dv[1].endpoint)
back = dv[1].channels_to(dv[0].endpoint)
e = PlanEntry(0, 0, 1, Mechanism.DYNAMIC, shape_of(size // 4), ElemType.F32, 1)
mb = ar[1].alloc(meta_block_size(1))
sp[1].write_at(mb, mb.length - 1, b"\x00")
e.recv_buffer = mb
e.remote_addr, e.remote_token, e.remote_len = mb.base_addr, mb.access_token, mb.length
snd = DynSender(e, sp[0], ar[0], fwd[1])
rcv = DynReceiver(e, sp[1], ar[1], back[1])
t = Tensor((size // 4,), ElemType.F32, BufferRef(ar[0].alloc(size), ar[0]), 0)
lib = _lib.load()
out = {}


def timeit(name, fn, reps=R):
    for _ in range(20):
        fn()
    sp[0].sync(), sp[1].sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    out[name] = round((time.perf_counter() - t0) / reps * 1e6, 3)
    sp[0].sync(), sp[1].sync()
    # the loops above clear the flag before their write executes: reset it
    sp[1].flag_clear(mb.end - 1)
    sp[1].sync()


meta = encode_meta(t.dims, t.elem_type, t.buffer.handle.base_addr, t.buffer.handle.access_token)
stage = snd.meta_stage
buf = (C.c_uint8 * 1)()
ev = C.c_void_p()
timeit("ctypes_noop(srf_launch_count)", lambda: lib.srf_launch_count())
timeit("encode_meta", lambda: encode_meta(t.dims, t.elem_type, t.buffer.handle.base_addr,
                                           t.buffer.handle.access_token))
timeit("flag_read(doorbell)", lambda: sp[1].flag_read(mb.end - 1, 1))
timeit("event_record+free", lambda: sp[0].fence().free())


def put_inline_raw():
    _lib.call("srf_put_inline", sp[0].handle, stage.base_addr, stage.access_token, meta,
              len(meta), sp[1].handle, mb.base_addr, mb.access_token, 0, None, C.byref(ev))
    lib.srf_event_free(ev)
    sp[1].flag_clear(mb.end - 1)


timeit("srf_put_inline+event_free+flag_clear", put_inline_raw)
timeit("flag_clear", lambda: sp[1].flag_clear(mb.end - 1))


def write_inline_verb():
    v = fwd[1].one_sided_write_inline(MemRange(stage), meta, mb.base_addr, mb.access_token)
    fwd[1].take_completion(v, wait=False).detach().free()
    sp[1].flag_clear(mb.end - 1)


timeit("one_sided_write_inline+take(no wait)+flag_clear", write_inline_verb)
blk = ar[1].alloc(size)


def read_raw():
    _lib.call("srf_get", sp[1].handle, blk.base_addr, blk.access_token, sp[0].handle,
              t.buffer.handle.base_addr, t.buffer.handle.access_token, size, None, C.byref(ev))
    lib.srf_event_free(ev)


try:
    timeit("srf_get+event_free", read_raw)
except Exception as exc:  # signature drift: report, keep going
    out["srf_get+event_free"] = f"error: {exc}"


def alloc_free():
    h = ar[1].alloc(size)
    BufferRef(h, ar[1]).release()


timeit("arena alloc + BufferRef.release (fence)", alloc_free, reps=500)


def one():
    snd.send(t, stage_copy=False)
    m = None
    while m is None:
        m = rcv.poll()
    rcv.fetch(m).buffer.release()


timeit("full transfer", one, reps=500)
print(json.dumps(out, indent=1), flush=True)
