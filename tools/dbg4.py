import math, sys
sys.path.insert(0, '.')
import numpy as np
from paper_1309_1230_b200 import ExecutorKind, Stepper
from paper_1309_1230_b200 import scenarios as S
from oracle.oracle import OracleStepper
sc = S.gen_square_dam(256)
g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=True))
o = OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
g.load(sc.build()); o.load(sc.build())
dg = g.compute_dt(math.inf); do = o.compute_dt(math.inf)
try:
    rg = g.step(dg, 0); ro = o.step(do, 0)
    a, b = g.state(), o.state()
    d = a.h != b.h
    print("dt", rg.dt_next, ro.dt_next, "mismatch cells", d.sum())
    js, is_ = np.nonzero(d)
    print(sorted(set(is_.tolist()))[:40], sorted(set(js.tolist()))[:10])
except Exception as e:
    print("ERR", e)
