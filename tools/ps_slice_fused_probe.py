"""N=1 VGG-16 PS with the fused weight push over slice sizes (extension:
tensors > slice cut into slices on the same shard), every schedule
autotuned by bench.bench_ps; prints steps/s and the candidates."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_1805_08430_b200 import _lib  # noqa: E402
from paper_1805_08430_b200.distributed import env_world, init_process_group  # noqa: E402
from paper_1805_08430_b200.ps import PsLayout  # noqa: E402
from paper_1805_08430_b200.workloads import vgg16_shapes  # noqa: E402

rank, world, local = env_world()
_lib.load()
torch.cuda.set_device(local)
init_process_group("nccl")
for mib in [int(x) for x in os.environ.get("PROBE_SLICES", "0,4,8,16,32").split(",")]:
    L = (PsLayout(vgg16_shapes(), 1, 1, slice_bytes=mib << 20 if mib else None) if world == 1
         else PsLayout(vgg16_shapes(), world, world, colocate=True,
                       slice_bytes=mib << 20 if mib else None))
    r = bench.bench_ps(rank, world, local, 20, 3, op="sgd", cpu=False, layout=L, label="probe")
    if rank == 0:
        print(json.dumps({"slice_mib": mib, "world": world, "units": len(L.shapes),
                          "steps_per_s": r["steps_per_s"], "fused": r.get("fused_push"),
                          "verified": r["verified"], "autotune": r["autotune_ms_per_5"]}),
              flush=True)
