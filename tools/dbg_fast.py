import math, sys, os
sys.path.insert(0, '.')
import numpy as np
from paper_1309_1230_b200 import ExecutorKind, Stepper
from paper_1309_1230_b200 import scenarios as S
for n in (64, 130, 512, 2048, 8192):
    sc = S.gen_channel_flood(n, manning_n=0.0)
    for exact in (True, False):
        g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact))
        g.load(sc.build())
        try:
            r = g.advance(1e18, 0, math.nan, 5)
            st = g.state()
            print(n, exact, "ok", r.steps, np.isnan(st.h).sum())
        except Exception as e:
            print(n, exact, "ERR", e)
