"""PS it/s vs GenGrad work-unit size (knob 12) for the benchmarked layouts
(torchrun for N>1; N=1 runs the VGG/FCN-5/LSTM device-engine lines)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1805_08430_b200 import _lib
from paper_1805_08430_b200.distributed import init_process_group
from paper_1805_08430_b200.ps import PsLayout
from paper_1805_08430_b200.workloads import vgg16_shapes

rank, world, local = init_process_group("nccl")
torch.cuda.set_device(local)
if world == 1:
    layouts = {"vgg": PsLayout(vgg16_shapes(), 1, 1),
               "fcn5": PsLayout([(int(204.47e6) // 10 // 4,)] * 10, 2, 1, False),
               "lstm": PsLayout([(int(35.93e6) // 14 // 4,)] * 14, 7, 1, False)}
else:
    layouts = {"vgg": PsLayout(vgg16_shapes(), world, world, colocate=True),
               "vgg_sliced_static": PsLayout(vgg16_shapes(), world, world, colocate=True,
                                             slice_bytes=2 << 20, grad_mechanism="static")}
for kib in [int(x) for x in os.environ.get("PROBE_UNITS", "128,512,2048").split(",")]:
    _lib.tune("gen_unit_kib", kib)
    for name, L in layouts.items():
        r = bench.bench_ps(rank, world, local, 10, 3, op="sgd", cpu=False, layout=L, label=name)
        if rank == 0:
            print(json.dumps({"world": world, "cfg": name, "gen_unit_kib": kib,
                              "steps_per_s": r["steps_per_s"], "frac": r["roofline"]["frac"],
                              "schedule": r["schedule"][:30], "verified": r["verified"]}),
                  flush=True)
