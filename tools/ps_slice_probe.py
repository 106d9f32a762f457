"""PS VGG-16 it/s at N>1 (torchrun) with the reference round-robin placement,
unsliced vs pipelined transfers (PsLayout.slice_bytes), through bench_ps
(schedule autotune, device events, max over ranks).  PROBE_SLICES: comma list
of slice sizes in MiB (0 = unsliced); PROBE_GRAD: gradient mechanism
(dynamic | static); PROBE_PARTITION: partition_bytes in MiB."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1805_08430_b200.distributed import init_process_group
from paper_1805_08430_b200.ps import PsLayout
from paper_1805_08430_b200.workloads import vgg16_shapes

rank, world, local = init_process_group("nccl")
torch.cuda.set_device(local)
for mib in [int(x) for x in os.environ.get("PROBE_SLICES", "0,64,16,4").split(",")]:
    kw = {"slice_bytes": mib << 20} if mib else {}
    kw["grad_mechanism"] = os.environ.get("PROBE_GRAD", "dynamic")
    if os.environ.get("PROBE_PARTITION"):
        kw.update(placement="bytes", partition_bytes=int(os.environ["PROBE_PARTITION"]) << 20)
    cfg = os.environ.get("PROBE_CFG", "vgg")
    if cfg == "vgg" and world == 1:   # N=1: worker server 0 + PS server 1 on GPU 0
        L = PsLayout(vgg16_shapes(), 1, 1, False, **kw)
    elif cfg == "vgg":
        L = PsLayout(vgg16_shapes(), world, world, colocate=True, **kw)
    elif cfg == "fcn5":   # configs[2] preset: 2 workers + 1 PS, server s on GPU s % world
        L = PsLayout([(int(204.47e6) // 10 // 4,)] * 10, 2, 1, False, **kw)
    else:                 # configs[4] LSTM preset: 7 workers + 1 PS
        L = PsLayout([(int(35.93e6) // 14 // 4,)] * 14, 7, 1, False, **kw)
    r = bench.bench_ps(rank, world, local, 10, 3, op="sgd", cpu=False, layout=L,
                       label=f"slice {mib} MiB")
    if rank == 0:
        print(json.dumps({"cfg": cfg, "world": world, "slice_mib": mib, "grad": kw["grad_mechanism"], "units": len(L.shapes),
                          **{k: r.get(k) for k in ("steps_per_s", "schedule", "verified", "roofline",
                                                    "autotune_ms_per_5")}}), flush=True)
