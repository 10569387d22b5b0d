"""ncu driver: one multi-step launch of N steps on a small config.
    python tools/prof_multi.py <config> <steps> [exact]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1309_1230_b200 import ExecutorKind, Stepper  # noqa: E402

cfg = sys.argv[1]
steps = int(sys.argv[2])
exact = "exact" in sys.argv[3:]
sc, _ = bench.scenario_for(cfg, 1)
st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact))
st.load(sc.build())
st.advance(1e18, 0, math.nan, 10)
r = st.advance(1e18, 10, math.nan, steps)
print("steps", r.steps, "launches", st.launch_count())
