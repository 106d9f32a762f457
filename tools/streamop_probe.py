"""Do stream memory operations work on a peer's IPC-mapped pool?  rank 0's
stream waits for a word in rank 1's pool, then writes a word in its own."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.distributed import gather_descriptors, init_process_group
from paper_1805_08430_b200.memspace import MemorySpace

rank, world, local = init_process_group("nccl")
torch.cuda.set_device(local)
sp = MemorySpace(rank, 4 << 20, device=local)
reg = sp.allocate_region(1 << 20, True)
sp.write_raw(reg.base_addr, (5).to_bytes(4, "little"))
sp.write_raw(reg.base_addr + 64, (0).to_bytes(4, "little"))
table = gather_descriptors(sp.export())
peer = MemorySpace.import_remote(table[1 - rank], local)
pbase = table[1 - rank]["regions"][0][1]
torch.distributed.barrier()
res = {}
if rank == 0:
    st = C.c_void_p()
    _lib.call("srf_stream_create", sp.handle, C.byref(st))
    _lib.call("srf_stream_wait_value32", st, peer.handle, pbase, 7, 0)
    _lib.call("srf_stream_write_value32", st, sp.handle, reg.base_addr + 64, 1)
    time.sleep(0.3)
    res["before"] = int.from_bytes(sp.read_raw(reg.base_addr + 64, 4), "little")
    torch.distributed.barrier()   # rank 1 sets its word to 7 after this
    t0 = time.perf_counter()
    while int.from_bytes(sp.read_raw(reg.base_addr + 64, 4), "little") != 1:
        if time.perf_counter() - t0 > 5:
            break
    res["after"] = int.from_bytes(sp.read_raw(reg.base_addr + 64, 4), "little")
    res["latency_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    print(json.dumps(res), flush=True)
else:
    torch.distributed.barrier()
    sp.write_raw(reg.base_addr, (7).to_bytes(4, "little"))
torch.distributed.barrier()
