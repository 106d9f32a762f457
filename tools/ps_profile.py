"""Run a few PS iterations of one config (for ncu launch lists / captures).
usage: ps_profile.py [vgg|lstm|fcn5|mlp] [phases|exchange]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_08430_b200.ps import PsLayout, PsStep
from paper_1805_08430_b200.workloads import mlp_shapes, vgg16_shapes

cfg = sys.argv[1] if len(sys.argv) > 1 else "vgg"
schedule = sys.argv[2] if len(sys.argv) > 2 else "phases"
if cfg == "vgg":
    L = PsLayout(vgg16_shapes(), 1, 1)
elif cfg == "fcn5":
    L = PsLayout([(int(204.47e6) // 10 // 4,)] * 10, 2, 1)
elif cfg == "mlp":
    L = PsLayout(mlp_shapes(), 2, 1)
else:
    L = PsLayout([(int(35.93e6) // 14 // 4,)] * 14, 7, 1)
ps = PsStep(L, seed=0, op="sgd", lr=0.01, schedule=schedule)
for it in range(1, 8):
    ps.step(it)
ps.sync()
ps.close()
print("ok", cfg, schedule)
