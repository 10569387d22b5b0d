"""The reference's validation suites (validate.hpp:45-357, oracle.hpp) run
against the CUDA stepper instead of the CPU executors.

equivalence      five drops 128^2, 200 steps: one domain and 2/4/8 row strips
                 SWS1-byte-identical to the oracle (validate.hpp:63-90)
dt-determinism   50 seeded states: compute_dt on one domain and on 2/4/8
                 strips bit-identical to the reference's (validate.hpp:93-118)
conservation     closed five-drops box 65^2, 500 steps: volume drift <= 1e-11
                 (validate.hpp:145-166, oracle.hpp:110-128)
dam-break        Stoker's analytic wet-bed dam break: L2 depth error <= 3 %,
                 star plateau within 2 % (validate.hpp:168-212, oracle.hpp:47-108)
guard            near-dry shelf: InstabilityError at the reference's cell and
                 time (validate.hpp:215-255)
symmetry         mirror symmetry_error of a five-drops run equals the
                 reference's (oracle.hpp:147-166; zero on the initial state)
halo mutation    strips exchanging R - 1 halo rows are detected (differ from
                 one domain); R rows are bit-identical (test_executor.cpp:246-303)
"""
import math
import os

import numpy as np
import pytest

from golden_cases import bits_equal
from oracle import oracle as O
from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200.io import snapshot_bytes
from paper_1309_1230_b200.stepper import (BoundaryKind, BoundarySet, ExecutorKind, FieldSet, GridSpec,
                                          InstabilityError, PhysicsParams, StabilityPolicy, Stepper)
from test_gpu_strips import run_single, run_strips, same

pytestmark = pytest.mark.gpu


def five_drops_scenario(n):
    """gen_five_drops(n) (scenarios.hpp:186-208): walls, cfl 0.45, frictionless."""
    ic = O.five_drops(n)
    return S.Scenario("five-drops", ic.spec, PhysicsParams(), StabilityPolicy(cfl=S.SCENARIO_CFL),
                      BoundarySet.all(BoundaryKind.wall()), 100.0, lambda sp, ic=ic: ic.copy())


# ---------------------------------------------------------------- criterion 1
def test_equivalence_strips_and_oracle_sws1_bytes():
    sc = five_drops_scenario(128)
    ora = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    ora.load(sc.build())
    ora.advance(1e18, 0, math.nan, 200)
    ref = snapshot_bytes(ora.state(), 9.81)
    one, _ = run_single(sc, True, 200)
    assert snapshot_bytes(one, 9.81) == ref
    for n in (2, 4, 8):
        got, _ = run_strips(sc, n, True, 200)
        assert snapshot_bytes(got, 9.81) == ref, n


# ---------------------------------------------------------------- criterion 2
def _random_state(trial, rng):
    fs = FieldSet(GridSpec(128, 128, 1.0, 1.0))
    if trial % 2 == 0:
        fs.h[:] = rng.uniform(0.2, 4.0)
    else:
        fs.h[:] = rng.uniform(0.2, 4.0, fs.h.shape)
        fs.qx[:] = rng.uniform(-2.0, 2.0, fs.h.shape)
        fs.qy[:] = rng.uniform(-2.0, 2.0, fs.h.shape)
    return fs


def test_dt_determinism_across_strip_counts():
    import threading
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    pol, phys = StabilityPolicy(), PhysicsParams()
    walls = BoundarySet.all(BoundaryKind.wall())
    rng = np.random.default_rng(0xC0FFEE)
    mismatches = 0
    for trial in range(50):
        fs = _random_state(trial, rng)
        r = O.RefStepper(fs.spec, phys, pol, walls)
        r.load(fs)
        want = r.compute_dt(1e18)
        one = Stepper(fs.spec, phys, pol, walls, ExecutorKind())
        one.load(fs)
        mismatches += one.compute_dt(1e18) != want
        one.close()
        for n in (2, 4, 8):
            key = os.urandom(16).hex().encode()
            got = [None] * n

            def worker(k):
                st = Stepper(fs.spec, phys, pol, walls, ExecutorKind(rank=k, nranks=n, local_group=True),
                             nccl_id=key)
                st.load_rows(fs.z[st.row_begin:st.row_end], fs.h[st.row_begin:st.row_end],
                             fs.qx[st.row_begin:st.row_end], fs.qy[st.row_begin:st.row_end], 0.0)
                got[k] = st.compute_dt(1e18)
                st.close()

            th = [threading.Thread(target=worker, args=(k,)) for k in range(n)]
            [t.start() for t in th]
            [t.join(timeout=120) for t in th]
            mismatches += sum(g != want for g in got)
    assert mismatches == 0


# ---------------------------------------------------------------- criterion 4
@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_conservation_closed_box(exact):
    sc = five_drops_scenario(65)
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact))
    fs = sc.build()
    st.load(fs)
    v0 = float(np.sum(fs.h) * sc.spec.dx * sc.spec.dy)
    dt = st.compute_dt(math.inf)
    worst = 0.0
    for k in range(500):
        dt = st.step(dt, k).dt_next
        worst = max(worst, abs(float(np.sum(st.state().h)) - v0))
    assert worst / v0 <= 1e-11


# ---------------------------------------------------------------- criterion 5
def solve_stoker(h_l, h_r, g):
    """oracle.hpp:47-80: star depth by bisection of the compatibility equation."""
    def f(h):
        ur = 2.0 * (math.sqrt(g * h_l) - math.sqrt(g * h))
        us = (h - h_r) * math.sqrt(0.5 * g * (h + h_r) / (h * h_r))
        return ur - us
    lo, hi = h_r, h_l
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if f(mid) > 0.0:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-12 * hi:
            break
    hs = 0.5 * (lo + hi)
    us = 2.0 * (math.sqrt(g * h_l) - math.sqrt(g * hs))
    return hs, us, hs * us / (hs - h_r)


def sample_profile(h_l, h_r, g, hs, us, s, x, t):
    """oracle.hpp:88-108."""
    cl, cs = math.sqrt(g * h_l), math.sqrt(g * hs)
    xi = x / t
    if xi <= -cl:
        return h_l
    if xi < us - cs:
        c = (2.0 * cl - xi) / 3.0
        return c * c / g
    if xi < s:
        return hs
    return h_r


def test_stoker_known_answer():
    hs, us, s = solve_stoker(1.0, 0.5, 9.81)  # test_oracle.cpp:18-24
    assert abs(hs - 0.726920446187478) < 1e-10
    assert abs(us - 0.923363901976376) < 1e-10
    assert abs(s - 2.95791812018356) < 1e-9


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_dam_break_against_stoker(exact):
    sc = S.gen_dam_break(400, 1.0, 0.5)
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact))
    st.load(sc.build())
    st.advance(sc.t_end)  # run_from to t_end (run.hpp:149-163)
    fin = st.state()
    t = fin.t
    assert t == sc.t_end
    g = sc.phys.g
    hs, us, s = solve_stoker(1.0, 0.5, g)
    split = 0.5 * 400
    mid = sc.spec.ny // 2
    x = (np.arange(sc.spec.nx) + 0.5) * sc.spec.dx - split
    ex = np.array([sample_profile(1.0, 0.5, g, hs, us, s, xx, t) for xx in x])
    h = fin.h[mid]
    l2 = math.sqrt(float(np.sum((h - ex) ** 2)) / float(np.sum(ex ** 2)))
    x_tail, x_shock = (us - math.sqrt(g * hs)) * t, s * t
    margin = 0.1 * (x_shock - x_tail)
    band = (x > x_tail + margin) & (x < x_shock - margin)
    plateau = float(h[band].mean())
    assert l2 <= 0.03
    assert abs(plateau - hs) / hs <= 0.02
    # the reference's own values: 9.77e-3 and 2.24e-4
    assert abs(l2 - 9.77e-3) < 5e-5
    assert abs(abs(plateau - hs) / hs - 2.24e-4) < 5e-6


# ---------------------------------------------------------------- criterion 6
@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_guard_aborts_near_dry_shelf_like_the_reference(exact):
    sc = S.gen_dam_break(101, 1.0, 1e-4)
    sc.phys = PhysicsParams(nu_art=0.0)  # raw scheme: the undershoot drains the shelf
    ora = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    ora.load(sc.build())
    with pytest.raises(InstabilityError) as eo:
        ora.advance(20.0)
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact))
    st.load(sc.build())
    with pytest.raises(InstabilityError) as eg:
        st.advance(20.0)
    e = eg.value
    assert e.i >= 0 and e.j >= 0 and e.t > 0.0
    if exact:
        assert (e.i, e.j, e.t) == (eo.value.i, eo.value.j, eo.value.t)
    # the committed state stays finite (no NaN reaches a snapshot)
    fin = st.state()
    assert np.isfinite(fin.h).all() and np.isfinite(fin.qx).all() and np.isfinite(fin.qy).all()


# ---------------------------------------------------------------- symmetry
def symmetry_error(fs, axis):
    """oracle.hpp:147-166."""
    if axis == "x":
        m = lambda a: a[:, ::-1]  # noqa: E731
        dqn = np.abs(fs.qx + m(fs.qx))
        dqt = np.abs(fs.qy - m(fs.qy))
    else:
        m = lambda a: a[::-1, :]  # noqa: E731
        dqn = np.abs(fs.qy + m(fs.qy))
        dqt = np.abs(fs.qx - m(fs.qx))
    return float(max(np.abs(fs.h - m(fs.h)).max(), dqn.max(), dqt.max()))


def test_mirror_symmetry_matches_reference():
    sc = five_drops_scenario(65)
    ic = sc.build()
    assert symmetry_error(ic, "x") == 0.0 and symmetry_error(ic, "y") == 0.0  # test_oracle.cpp:100-104
    ora = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    ora.load(ic)
    ora.advance(1e18, 0, math.nan, 100)
    b = ora.state()
    for exact in (True, False):
        st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact))
        st.load(ic)
        st.advance(1e18, 0, math.nan, 100)
        a = st.state()
        for ax in ("x", "y"):
            ea, eb = symmetry_error(a, ax), symmetry_error(b, ax)
            # the alternating one-sided sweeps are not mirror-symmetric step by step
            # (~1e-2 after 100 steps in the reference too): the CUDA stepper must
            # reproduce the reference's asymmetry, not remove it
            if exact:
                assert ea == eb
            assert abs(ea - eb) <= 1e-12


# ---------------------------------------------------------------- halo mutation
@pytest.mark.parametrize("name", ["dam", "floodplain"])
def test_shrunk_strip_halo_is_detected(name, monkeypatch):
    sc = S.gen_square_dam(96, 1.0, 0.5) if name == "dam" else S.gen_floodplain(96)
    R = 2 if sc.phys.nu_art > 0 else 1
    ref, rr = run_single(sc, True, 20)
    monkeypatch.setenv("SWE_DEBUG_HALO_ROWS", str(R))
    good, rg = run_strips(sc, 3, True, 20)
    assert rg == rr and same(ref, good)
    monkeypatch.setenv("SWE_DEBUG_HALO_ROWS", str(R - 1))
    bad, _ = run_strips(sc, 3, True, 20)
    assert not same(ref, bad)
    # the damage starts at the strip boundaries
    diff = np.nonzero(np.any(ref.h != bad.h, axis=1))[0]
    assert diff.size and any(abs(int(d) - b) <= 20 for d in diff for b in (32, 64))
