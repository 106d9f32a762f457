"""A few PS steps of configs[3] VGG-16 (N=1: worker server 0 + PS server 1 on
GPU 0) in the phase schedule with the fused weight push, for an ncu capture
of the fused pull+apply+forward batch:
  ncu --set full -k regex:k_apply_batch -s 2 -c 1 python tools/ps_ncu_once.py
Algorithmic bytes of one apply batch launch: per variable read var + read
grad + write var + write the worker's weight region = 4 S (2.21 GB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200.ps import PsLayout, PsStep  # noqa: E402
from paper_1805_08430_b200.workloads import vgg16_shapes  # noqa: E402

L = PsLayout(vgg16_shapes(), 1, 1)
ps = PsStep(L, seed=0, op="sgd", lr=0.01, fuse_push=os.environ.get("PROBE_FUSE", "1") == "1")
for it in range(1, 5):
    ps.step(it)
ps.sync()
print("ps_ncu_once ok", sum(L.nbytes(v) for v in range(len(L.shapes))), flush=True)
ps.close()
