"""Host-side cost of one dynamic transfer through the public API (cProfile)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

print(bench.dynamic_rate(1 << 20, 0), flush=True)
pr = cProfile.Profile()
pr.enable()
print(bench.dynamic_rate(1 << 20, 0, reps=200), flush=True)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
