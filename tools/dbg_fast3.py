import math, sys
sys.path.insert(0, '.')
from paper_1309_1230_b200 import ExecutorKind, Stepper
from paper_1309_1230_b200 import scenarios as S
sc = S.gen_square_dam(64)
for exact in (True, False):
    g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact))
    g.load(sc.build())
    dt = g.compute_dt(math.inf)
    try:
        g.step(dt, 0)
    except Exception as e:
        print("err", e)
    sys.stdout.flush()
