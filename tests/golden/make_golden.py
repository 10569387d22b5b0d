"""Generate the golden parity fixtures from the UNMODIFIED reference solver.

    python tests/golden/make_golden.py

Runs oracle/_ref/libswe_ref.so (the reference headers under
/root/reference/proj/include compiled in place by oracle/Makefile, naive
executor) on the cases of the reference's own test suite
(proj/tests/test_executor.cpp, test_timestep.cpp, validate.hpp) and writes one
compressed .npz per case: inputs (grid, physics, policy, boundaries, initial
state, step schedule) and outputs (final h/qx/qy, t, dt_next, warnings, or the
error the reference raised).  Only needed where /root/reference exists; the
fixtures are committed and travel with the repo.
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1309_1230_b200.stepper import (BoundaryKind, BoundarySet, FieldSet, GridSpec, PhysicsParams,  # noqa: E402
                                          SweError, StabilityPolicy)
from paper_1309_1230_b200 import scenarios as S  # noqa: E402


def bk_arr(b: BoundaryKind):
    return [b.type, b.q_n, b.h_in, b.eta_out]


def run_case(name, spec, phys, pol, bounds, ic: FieldSet, steps, dt0=None, parity0=0, note=""):
    st = O.RefStepper(spec, phys, pol, bounds)
    st.load(ic)
    dt = st.compute_dt(1e18) if dt0 is None else dt0
    dts = []
    err = None
    warnings = 0
    for k in range(steps):
        try:
            r = st.step(dt, parity0 + k)
        except SweError as e:
            err = {"step": k, "code": e.code, "i": getattr(e, "i", -1), "j": getattr(e, "j", -1),
                   "t": getattr(e, "t", 0.0) if hasattr(e, "t") and not callable(getattr(e, "t")) else 0.0,
                   "msg": str(e)}
            if hasattr(e, "sim_time"):
                err["t"] = e.sim_time()
            break
        dts.append(dt)
        warnings += r.guard_warnings
        dt = r.dt_next
    fin = st.state()
    meta = {"name": name, "note": note, "steps": steps, "parity0": parity0, "dt0_given": dt0 is not None,
            "grid": [spec.nx, spec.ny, spec.dx, spec.dy], "physics": [phys.g, phys.manning_n, phys.nu_art],
            "policy": [pol.cfl, pol.dt_max, pol.dt_min, pol.h_min],
            "bounds": [bk_arr(bounds.north), bk_arr(bounds.south), bk_arr(bounds.east), bk_arr(bounds.west)],
            "error": err, "warnings": warnings, "t_final": fin.t, "dt_next": dt,
            "generator": "oracle/_ref (reference swe::Stepper, naive executor)"}
    np.savez_compressed(os.path.join(HERE, name + ".npz"), meta=json.dumps(meta),
                        z=ic.z, h0=ic.h, qx0=ic.qx, qy0=ic.qy, h=fin.h, qx=fin.qx, qy=fin.qy,
                        dts=np.array(dts, dtype=np.float64), dt0=np.float64(dt0 if dt0 is not None else np.nan))
    print(f"{name:24s} steps={len(dts):4d} err={err['code'] if err else None} t={fin.t!r}")


def main():
    walls = BoundarySet.all(BoundaryKind.wall())
    pol = StabilityPolicy(cfl=0.45)

    # test_executor.cpp:151-167 -- five drops 48, nu 0 and 0.05, 60 steps
    for nu in (0.0, 0.05):
        sp, ph, po, bd, te, ic = O.ref_scenario("five-drops", 48)
        run_case(f"drops48_nu{int(nu * 100):02d}", sp, PhysicsParams(nu_art=nu), pol, walls, ic, 60)
    # test_executor.cpp:169-177 -- mixed open boundaries
    sp, ph, po, bd, te, ic = O.ref_scenario("five-drops", 40)
    mixed = BoundarySet(BoundaryKind.transmissive(), BoundaryKind.transmissive(), BoundaryKind.fixed_eta(1.0),
                        BoundaryKind.inflow(0.1, 1.0))
    run_case("mixed40", sp, PhysicsParams(), pol, mixed, ic, 50)
    # mixed boundaries with smoothing (both parities of every edge kind through the smoothing ghosts)
    run_case("mixed40_nu05", sp, PhysicsParams(nu_art=0.05), pol, mixed, ic, 50)
    # test_executor.cpp:179-190 -- vortex
    sp, ph, po, bd, te, ic = O.ref_scenario("vortex", 48)
    run_case("vortex48", sp, ph, po, bd, ic, 60)
    # test_executor.cpp:224-244 -- soak: bathymetry, friction, diffusion, non-square
    spec = GridSpec(67, 45, 1.0, 1.0)
    sc = S.gen_channel_flood(67)
    ic = S.channel_slope(spec, 1.0, 0.5 / 66.0)
    run_case("soak67x45", spec, PhysicsParams(manning_n=0.035, nu_art=0.04), sc.pol, sc.bounds, ic, 80,
             note="Manning on: std::pow, tolerance-only on CUDA")
    run_case("soak67x45_frictionless", spec, PhysicsParams(manning_n=0.0, nu_art=0.04), sc.pol, sc.bounds, ic, 80)
    # channel flood preset (Manning)
    sc = S.gen_channel_flood(96)
    run_case("channel96", sc.spec, sc.phys, sc.pol, sc.bounds, sc.build(), 120, note="Manning on")
    # test_executor.cpp:192-222 -- inflow on each edge
    for e in ("north", "south", "east", "west"):
        spec = GridSpec(24, 18, 1.0, 1.0)
        ic = S.flat_pool(spec, 1.0)
        kw = {k: BoundaryKind.wall() for k in ("north", "south", "east", "west")}
        kw[e] = BoundaryKind.inflow(0.05, 1.0)
        run_case(f"inflow_{e}", spec, PhysicsParams(), pol, BoundarySet(**kw), ic, 60)
    # test_executor.cpp:118-133 -- still water fixed point
    spec = GridSpec(24, 24, 1.0, 1.0)
    run_case("still24", spec, PhysicsParams(), pol, walls, S.flat_pool(spec, 1.0), 20)
    # test_executor.cpp:377-416 -- transposition (one step each parity at half the CFL dt)
    rng = np.random.Generator(np.random.PCG64(31))
    a = FieldSet(GridSpec(9, 13, 1.0, 1.0))
    a.h[:] = rng.uniform(0.8, 1.4, a.h.shape)
    a.qx[:] = rng.uniform(-0.2, 0.2, a.h.shape)
    a.qy[:] = rng.uniform(-0.2, 0.2, a.h.shape)
    b = FieldSet(GridSpec(13, 9, 1.0, 1.0), None, a.h.T.copy(), a.qy.T.copy(), a.qx.T.copy())
    for par in (0, 1):
        st = O.RefStepper(a.spec, PhysicsParams(), pol, walls)
        st.load(a)
        dt = 0.5 * st.compute_dt(1e9)
        run_case(f"transpose_a_p{par}", a.spec, PhysicsParams(), pol, walls, a, 1, dt0=dt, parity0=par)
        run_case(f"transpose_b_p{par}", b.spec, PhysicsParams(), pol, walls, b, 1, dt0=dt, parity0=par)
    # scenarios.hpp:285-306 -- thin-channel dam break (3 rows, transmissive N/S, nu 0.05)
    sc = S.gen_dam_break(400)
    run_case("dambreak400", sc.spec, sc.phys, sc.pol, sc.bounds, sc.build(), 300)
    # test_executor.cpp:349-375 -- engineered dry shelf must fail (nu = 0)
    sc = S.gen_dam_break(48, 1.0, 1e-4)
    run_case("shelf48", sc.spec, PhysicsParams(nu_art=0.0), sc.pol, sc.bounds, sc.build(), 200,
             note="InstabilityError expected")
    # guard: a NaN momentum mid-grid (executor.hpp:543-556)
    spec = GridSpec(20, 16, 1.0, 1.0)
    ic = S.flat_pool(spec, 1.0)
    ic.qx[9, 13] = math.nan
    run_case("guard_nan", spec, PhysicsParams(), pol, walls, ic, 3, dt0=0.1, note="guard InstabilityError")
    # test_executor.cpp:418-431 -- fixed-elevation clamp warning
    spec = GridSpec(12, 12, 1.0, 1.0)
    ic = S.flat_pool(spec, 0.5)
    bd = BoundarySet(east=BoundaryKind.fixed_eta(1e-7))
    st = O.RefStepper(spec, PhysicsParams(), pol, bd)
    st.load(ic)
    run_case("fixedeta_clamp", spec, PhysicsParams(), pol, bd, ic, 1, dt0=0.9 * st.compute_dt(1e9))
    # SURVEY.md §8(c) config 1 at 200 steps (square 256 dam break; SWS1 sha256 also pinned)
    sc = S.gen_square_dam(256)
    run_case("dam256_200", sc.spec, sc.phys, sc.pol, sc.bounds, sc.build(), 200)


if __name__ == "__main__":
    main()
