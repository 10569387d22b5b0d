"""GPU parity of the early-exit tiles (SWE_EXEC_EARLY_EXIT).

Skipping a quiet item is exact by construction (a flat bed at rest is a
bit-exact fixed point of the step, and the skipped item's CFL speed is folded
into the reduction), so every run with early exit must be bit-identical to
the same run without it -- in both arithmetic modes -- and, in exact mode,
to the CPU oracle.  The reference has no early exit; its executors all
compute every cell (executor.hpp:846-911), which is what the comparison
against the non-skipping kernel and the oracle pins.
"""
import math

import numpy as np
import pytest

from golden_cases import bits_equal
from oracle import oracle as O
from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200.stepper import ExecutorKind, Stepper

pytestmark = pytest.mark.gpu


def run(sc, exact, early, steps, api="advance"):
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact, early_exit=early))
    st.load(sc.build())
    if api == "advance":
        r = st.advance(1e18, 0, math.nan, steps)
        assert r.steps == steps
        dt_next = r.dt_next
    else:
        dt = st.compute_dt(math.inf)
        for k in range(steps):
            dt = st.step(dt, k).dt_next
        dt_next = dt
    fs = st.state()
    act = st.activity()
    st.close()
    return fs, dt_next, act


def same(a, b):
    return bits_equal(a.h, b.h) and bits_equal(a.qx, b.qx) and bits_equal(a.qy, b.qy) and a.t == b.t


SCEN = {
    # C5 shape at test size: thin-film floodplain, smoothing on (radius-3 dependency)
    "floodplain384": lambda: S.gen_floodplain(384),
    # frictionless dam break without smoothing (radius-2 dependency)
    "dam384": lambda: S.gen_square_dam(384, 1.0, 0.5),
    # rectangular, tile/chunk counts not dividing the grid
    "floodplain_rect": lambda: _rect(),
}


def _rect():
    from paper_1309_1230_b200.stepper import GridSpec
    sc = S.gen_floodplain(400)
    sc.spec = GridSpec(331, 517, 1.0, 1.0)
    return sc


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
@pytest.mark.parametrize("name", sorted(SCEN))
def test_early_exit_is_bit_identical(name, exact):
    sc = SCEN[name]()
    ref, dref, a0 = run(sc, exact, False, 80)
    got, dgot, act = run(sc, exact, True, 80)
    assert a0["skipped_cells"] == 0
    assert act["eligible_items"] > 0
    assert act["skipped_cells"] > 0, act  # the quiet floodplain / far field is skipped
    assert same(ref, got)
    assert dref == dgot


def test_early_exit_host_step_api():
    """Stepper::step loop (host round trip each step) with early exit."""
    sc = S.gen_floodplain(256)
    ref, dref, _ = run(sc, True, False, 40, api="step")
    got, dgot, act = run(sc, True, True, 40, api="step")
    assert act["skipped_cells"] > 0
    assert same(ref, got) and dref == dgot


def test_early_exit_matches_oracle():
    sc = S.gen_floodplain(160)
    got, dgot, act = run(sc, True, True, 60, api="step")
    assert act["skipped_cells"] > 0
    ora = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    ora.load(sc.build())
    dt = ora.compute_dt(math.inf)
    for k in range(60):
        dt = ora.step(dt, k).dt_next
    assert same(got, ora.state())
    assert dgot == dt


def test_early_exit_inactive_on_sloped_bed():
    """A non-flat bed has no early-exit kernel: no item is eligible, results unchanged."""
    sc = S.gen_channel_flood(192, manning_n=0.0)
    ref, dref, _ = run(sc, True, False, 30)
    got, dgot, act = run(sc, True, True, 30)
    assert act["eligible_items"] == 0 and act["skipped_cells"] == 0
    assert same(ref, got) and dref == dgot


def test_early_exit_wave_reenters_quiet_region():
    """Items skipped while quiet must be recomputed once the bore reaches them:
    run long enough for the front to cross many items and compare each chunk."""
    sc = S.gen_square_dam(256, 1.0, 0.5, split_x=32.0)
    a = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=True, early_exit=False))
    b = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=True, early_exit=True))
    fs = sc.build()
    a.load(fs)
    b.load(fs)
    ka = kb = 0
    da = db = math.nan
    for _ in range(6):
        ra = a.advance(1e18, ka, da, 50)
        rb = b.advance(1e18, kb, db, 50)
        ka, da, kb, db = ra.step_index, ra.dt_next, rb.step_index, rb.dt_next
        assert da == db
        assert same(a.state(), b.state())
    assert b.activity()["skipped_cells"] > 0
