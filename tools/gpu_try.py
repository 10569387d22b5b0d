import sys, math, time
sys.path.insert(0, '.')
import numpy as np
from oracle.oracle import OracleStepper, five_drops, vortex
from paper_1309_1230_b200 import *
from paper_1309_1230_b200.scenarios import gen_square_dam, gen_channel_flood

def cmp(a, b):
    out = {}
    for n in ("h","qx","qy"):
        x, y = getattr(a,n), getattr(b,n)
        out[n] = (int((x.view(np.uint64) != y.view(np.uint64)).sum()), float(np.nanmax(np.abs(x-y))))
    return out

def run(name, spec, phys, pol, bounds, fs, steps):
    g = Stepper(spec, phys, pol, bounds, ExecutorKind(exact=True))
    r = OracleStepper(spec, phys, pol, bounds)
    g.load(fs); r.load(fs)
    dg = g.compute_dt(math.inf); dr = r.compute_dt(math.inf)
    first = None
    for k in range(steps):
        try:
            rg = g.step(dg, k)
        except Exception as e:
            print(name, "GPU error at step", k, type(e).__name__, e); return
        rr = r.step(dr, k)
        if first is None and rg.dt_next != rr.dt_next:
            first = k
        dg, dr = rg.dt_next, rr.dt_next
        if k < 3 or k == steps-1:
            c = cmp(g.state(), r.state())
            print(name, "step", k, "dt", dg == dr, c)
    print(name, "first dt mismatch", first, "t", g.time(), r.time())

sc = gen_square_dam(64); run("dam64", sc.spec, sc.phys, sc.pol, sc.bounds, sc.build(), 20)
sc = gen_square_dam(200); run("dam200", sc.spec, sc.phys, sc.pol, sc.bounds, sc.build(), 50)
fs = five_drops(48); sc = gen_square_dam(48); run("drops48", sc.spec, sc.phys, sc.pol, sc.bounds, fs, 60)
sc = gen_square_dam(48, nu_art=0.05); run("drops48nu", sc.spec, sc.phys, sc.pol, sc.bounds, fs, 60)
sc = gen_channel_flood(67, manning_n=0.0); run("chan67", sc.spec, sc.phys, sc.pol, sc.bounds, sc.build(), 80)
sc = gen_channel_flood(67); run("chan67man", sc.spec, sc.phys, sc.pol, sc.bounds, sc.build(), 80)
mixed = BoundarySet(BoundaryKind.transmissive(), BoundaryKind.transmissive(), BoundaryKind.fixed_eta(1.0), BoundaryKind.inflow(0.1, 1.0))
fs = five_drops(40); sc = gen_square_dam(40); run("mixed40", sc.spec, sc.phys, sc.pol, mixed, fs, 50)
# larger + advance
sc = gen_square_dam(1024); g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds); g.load(sc.build())
t0 = time.time(); res = g.advance(1e18, 0, math.nan, 1000); el = time.time()-t0
print("advance 1024^2 x1000", res, el, "cells/s", 1024*1024*1000/el)

# fast mode tolerance probe
def run_fast(name, sc, fs, steps):
    g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=False))
    r = OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    g.load(fs); r.load(fs)
    dg = g.compute_dt(math.inf); dr = r.compute_dt(math.inf)
    for k in range(steps):
        dg = g.step(dg, k).dt_next; dr = r.step(dr, k).dt_next
    a, b = g.state(), r.state()
    ua, ub = a.qx / a.h, b.qx / b.h; va, vb = a.qy / a.h, b.qy / b.h
    print("FAST", name, steps, "max|dh|", np.abs(a.h - b.h).max(), "max|du|", np.abs(ua - ub).max(), "max|dv|", np.abs(va - vb).max(), "dt rel", abs(dg - dr) / dr)
sc = gen_square_dam(256); run_fast("dam256", sc, sc.build(), 1000)
sc = gen_square_dam(48); run_fast("drops48", sc, five_drops(48), 200)
sc = gen_channel_flood(128); run_fast("chan128man", sc, sc.build(), 500)
