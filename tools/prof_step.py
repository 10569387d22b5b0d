"""Small driver for ncu captures: load a bench config, run a few device-resident steps.

    python tools/prof_step.py <config> <steps> [fast] [early]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1309_1230_b200 import ExecutorKind, Stepper  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3f"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
fast = "fast" in sys.argv[3:]
early = "early" in sys.argv[3:] or cfg == "c5"
sc, _ = bench.scenario_for(cfg, 1)
st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=not fast, graph=False, early_exit=early))
st.load(sc.build())
r = st.advance(1e18, 0, math.nan, steps)
print("steps", r.steps, "t", r.t_final, "launches", st.launch_count())
