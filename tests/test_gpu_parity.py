"""GPU parity: libswe_cuda.so against the CPU oracle and the reference goldens.

Exact mode (SWE_EXEC_EXACT, -fmad=false) must be bit-identical to the
reference on every case without Manning friction (std::pow is not
bit-reproducible on CUDA).  Fast mode (FMA + shared
reciprocals) must agree within the stated tolerance:
    max |dh|, |du|, |dv| <= FAST_TOL after the case's steps.
All calls go through the C-ABI (ctypes mirror in paper_1309_1230_b200/stepper.py).
"""
import math
import os
import subprocess

import numpy as np
import pytest

from golden_cases import bits_equal, cases
from oracle import oracle as O
from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200 import abi
from paper_1309_1230_b200.stepper import (BoundaryKind, BoundarySet, ConfigError, ExecutorKind, FieldSet, GridSpec,
                                          InstabilityError, PhysicsParams, StabilityPolicy, Stepper)

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAST_TOL = 1e-12   # absolute, on h, u = qx/h, v = qy/h (O(1) fields); measured <= 6e-14
MANNING_TOL = 1e-12
CASES = cases()
EXACT = ExecutorKind(exact=True)
FAST = ExecutorKind(exact=False)


def uv(fs_h, fs_qx, fs_qy):
    return fs_qx / fs_h, fs_qy / fs_h


def max_err(a_h, a_qx, a_qy, b_h, b_qx, b_qy):
    ua, va = uv(a_h, a_qx, a_qy)
    ub, vb = uv(b_h, b_qx, b_qy)
    return max(np.abs(a_h - b_h).max(), np.abs(ua - ub).max(), np.abs(va - vb).max())


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_exact_mode_matches_reference_golden(case):
    st = Stepper(case.spec, case.phys, case.pol, case.bounds, EXACT)
    fin, err, dt_next, warnings = case.run(st)
    exp = case.expected_error()
    if case.manning:  # pow(h, 4/3): tolerance-only
        assert err == exp
        assert max_err(fin.h, fin.qx, fin.qy, case.h, case.qx, case.qy) <= MANNING_TOL
        return
    assert err == exp, (err, exp)
    assert bits_equal(fin.h, case.h) and bits_equal(fin.qx, case.qx) and bits_equal(fin.qy, case.qy)
    assert fin.t == case.meta["t_final"]
    if err is None:
        assert dt_next == case.meta["dt_next"]
        assert warnings == case.meta["warnings"]


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_fast_mode_within_tolerance(case):
    st = Stepper(case.spec, case.phys, case.pol, case.bounds, FAST)
    fin, err, dt_next, warnings = case.run(st)
    exp = case.expected_error()
    if exp is None:
        assert err is None
        assert max_err(fin.h, fin.qx, fin.qy, case.h, case.qx, case.qy) <= FAST_TOL
        assert abs(dt_next - case.meta["dt_next"]) <= 1e-12 * case.meta["dt_next"]
    else:
        assert err is not None and err[1] == exp[1]


def test_shared_reciprocal_division_is_ieee():
    rng = np.random.Generator(np.random.PCG64(7))
    n = 1 << 22
    a = rng.standard_normal(n) * np.exp2(rng.integers(-60, 60, n))
    b = np.abs(rng.standard_normal(n)) * np.exp2(rng.integers(-60, 60, n)) + 1e-300
    special = np.array([0.0, -0.0, 1e-320, -1e-320, 5e-324, 1e300, -1e300, 1.7e308, np.inf, -np.inf, np.nan,
                        2.2250738585072014e-308, 1.0, -1.0, 3.0, 1e-308, 4.9e-310])
    sa, sb = np.meshgrid(special, np.concatenate([special, [0.5, 2.0, 1e-10, 1e10, 7.0]]))
    a = np.concatenate([a, sa.ravel(), (a[:1000] * 0.0)])
    b = np.concatenate([b, sb.ravel(), b[:1000]])
    out = np.empty_like(a)
    st = abi.swe_status()
    lib = abi.load_library()
    assert lib.swe_cuda_selftest_div(abi.dptr(a), abi.dptr(b), a.size, 1, abi.dptr(out), st) == 0
    with np.errstate(all="ignore"):
        ref = a / b
    same = (out.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (a[~same][:5], b[~same][:5], out[~same][:5], ref[~same][:5])


def test_state_checked_division_is_ieee():
    """SWE_EXACT_STATE_CHECK: inside the range test (|h| in [2^-400, 2^400),
    momentum 0 or of magnitude in [2^-200, 2^200)) the shared-reciprocal
    quotient without ptxas's per-division test is the IEEE quotient, signed
    zeros included; outside it the IEEE division runs -- across the range
    edges, the specials and random operands."""
    rng = np.random.Generator(np.random.PCG64(11))
    n = 1 << 22
    a = rng.standard_normal(n) * np.exp2(rng.integers(-215, 215, n).astype(np.float64))
    b = np.abs(rng.standard_normal(n)) * np.exp2(rng.integers(-415, 415, n).astype(np.float64))
    edges_a = np.array([2.0 ** -200, -(2.0 ** -200), np.nextafter(2.0 ** -200, 0), 2.0 ** 200,
                        np.nextafter(2.0 ** 200, 0), -(2.0 ** 200), 0.0, -0.0, np.inf, -np.inf, np.nan, 1e-310])
    edges_b = np.array([2.0 ** -400, np.nextafter(2.0 ** -400, 0), 2.0 ** 400, np.nextafter(2.0 ** 400, 0),
                        -(2.0 ** -400), 1.0, 3.0, 0.1, 1e-320, np.inf, 0.0, -0.0, np.nan])
    sa, sb = np.meshgrid(edges_a, edges_b)
    a = np.concatenate([a, sa.ravel(), a[:1000] * 0.0, -(a[:1000] * 0.0)])
    b = np.concatenate([b, sb.ravel(), b[:2000]])
    out = np.empty_like(a)
    st = abi.swe_status()
    lib = abi.load_library()
    assert lib.swe_cuda_selftest_div(abi.dptr(a), abi.dptr(b), a.size, 2, abi.dptr(out), st) == 0
    with np.errstate(all="ignore"):
        ref = a / b
    same = (out.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (a[~same][:5], b[~same][:5], out[~same][:5], ref[~same][:5])


def test_step_equals_device_resident_advance():
    sc = S.gen_square_dam(200)
    fs = sc.build()
    for kind in (EXACT, FAST):
        a = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind)
        b = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind)
        a.load(fs)
        b.load(fs)
        dt = a.compute_dt(math.inf)
        for k in range(150):
            dt = a.step(dt, k).dt_next
        r = b.advance(1e18, 0, math.nan, 150)
        assert r.steps == 150 and r.step_index == 150 and r.dt_next == dt
        x, y = a.state(), b.state()
        assert x.t == y.t
        assert bits_equal(x.h, y.h) and bits_equal(x.qx, y.qx) and bits_equal(x.qy, y.qy)


def test_advance_lands_on_t_end_like_run_from():
    # run.hpp:149-163: identical to driving the oracle with the same loop
    sc = S.gen_square_dam(64)
    g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, EXACT)
    o = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    g.load(sc.build())
    o.load(sc.build())
    rg = g.advance(7.3)
    ro = o.advance(7.3)
    assert rg.t_final == 7.3 == ro.t_final
    assert (rg.steps, rg.step_index, rg.dt_next) == (ro.steps, ro.step_index, ro.dt_next)
    a, b = g.state(), o.state()
    assert bits_equal(a.h, b.h) and bits_equal(a.qx, b.qx)
    # resume (odd parity origin, given first dt) continues bit-identically
    rg2 = g.advance(9.0, rg.step_index, rg.dt_next)
    ro2 = o.advance(9.0, ro.step_index, ro.dt_next)
    assert (rg2.steps, rg2.t_final, rg2.dt_next) == (ro2.steps, ro2.t_final, ro2.dt_next)
    assert bits_equal(g.state().h, o.state().h)


def test_failure_is_atomic_and_located_like_the_oracle():
    sc = S.gen_dam_break(48, 1.0, 1e-4)
    phys = PhysicsParams(nu_art=0.0)
    g = Stepper(sc.spec, phys, sc.pol, sc.bounds, EXACT)
    o = O.OracleStepper(sc.spec, phys, sc.pol, sc.bounds)
    g.load(sc.build())
    o.load(sc.build())
    dg, do = g.compute_dt(1e9), o.compute_dt(1e9)
    assert dg == do
    for k in range(200):
        before = g.state()
        try:
            rg = g.step(dg, k)
        except InstabilityError as e:
            with pytest.raises(InstabilityError) as eo:
                o.step(do, k)
            assert (e.cell_i(), e.cell_j(), e.sim_time()) == (eo.value.cell_i(), eo.value.cell_j(),
                                                              eo.value.sim_time())
            assert e.cell_i() >= 0 and e.cell_j() >= 0 and e.sim_time() > 0.0
            after = g.state()
            assert bits_equal(after.h, before.h) and after.t == before.t  # failure atomicity
            return
        ro = o.step(do, k)
        assert rg.dt_next == ro.dt_next
        dg, do = rg.dt_next, ro.dt_next
    pytest.fail("engineered dry shelf did not fail")


def test_guard_error_reports_first_offender_and_values():
    spec = GridSpec(20, 16, 1.0, 1.0)
    fs = S.flat_pool(spec, 1.0)
    fs.qx[9, 13] = math.nan
    fs.qx[12, 2] = math.nan
    g = Stepper(spec, PhysicsParams(), StabilityPolicy(cfl=0.45), BoundarySet.all(BoundaryKind.wall()), EXACT)
    g.load(fs)
    with pytest.raises(InstabilityError) as e:
        g.guard()
    assert (e.value.cell_i(), e.value.cell_j()) == (13, 9)
    with pytest.raises(InstabilityError) as e2:
        g.step(0.1, 0)
    o = O.OracleStepper(spec, PhysicsParams(), StabilityPolicy(cfl=0.45), BoundarySet.all(BoundaryKind.wall()))
    o.load(fs)
    with pytest.raises(InstabilityError) as e3:
        o.step(0.1, 0)
    assert (e2.value.cell_i(), e2.value.cell_j(), e2.value.sim_time()) == \
        (e3.value.cell_i(), e3.value.cell_j(), e3.value.sim_time())
    # NaN momentum poisons the predicted depth next door: the corrector (K4) raises
    # before the guard (K5), exactly as in the reference's plan order
    assert str(e2.value).startswith("predicted depth")


def test_config_errors():
    with pytest.raises(ConfigError):
        Stepper(GridSpec(8, 8), PhysicsParams(nu_art=0.7), StabilityPolicy(), BoundarySet())
    st = Stepper(GridSpec(8, 8), PhysicsParams(), StabilityPolicy(), BoundarySet())
    with pytest.raises(ConfigError):
        st.step(0.1, 0)  # no state loaded
    st.load(S.flat_pool(GridSpec(8, 8), 1.0))
    with pytest.raises(ConfigError):
        st.step(math.inf, 0)


def test_still_water_fixed_point_full_size():
    # test_executor.cpp:118-133 at the BASELINE size: bit-exact fixed point incl. signbit
    spec = GridSpec(8192, 8192, 1.0, 1.0)
    g = Stepper(spec, PhysicsParams(), StabilityPolicy(cfl=0.45), BoundarySet.all(BoundaryKind.wall()), EXACT)
    fs = S.flat_pool(spec, 1.0)
    g.load(fs)
    r = g.advance(1e18, 0, math.nan, 20)
    assert r.steps == 20
    out = g.state()
    assert (out.h == 1.0).all()
    assert (out.qx.view(np.uint64) == 0).all() and (out.qy.view(np.uint64) == 0).all()


def test_closed_box_conserves_volume_full_size():
    # validate.hpp:145-165: closed-box drift <= 1e-11 (reference measures ~1e-15)
    sc = S.gen_square_dam(8192)
    g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, FAST)
    fs = sc.build()
    v0 = math.fsum(fs.h.ravel())
    g.load(fs)
    g.advance(1e18, 0, math.nan, 50)
    v1 = math.fsum(g.state().h.ravel())
    assert abs(v1 - v0) / v0 <= 1e-11


def test_transpose_symmetry_large():
    # test_executor.cpp:377-416 on a 1536 x 1024 random state, both parities, exact mode
    rng = np.random.Generator(np.random.PCG64(31))
    a = FieldSet(GridSpec(1536, 1024, 1.0, 1.0))
    a.h[:] = rng.uniform(0.8, 1.4, a.h.shape)
    a.qx[:] = rng.uniform(-0.2, 0.2, a.h.shape)
    a.qy[:] = rng.uniform(-0.2, 0.2, a.h.shape)
    b = FieldSet(GridSpec(1024, 1536, 1.0, 1.0), None, a.h.T.copy(), a.qy.T.copy(), a.qx.T.copy())
    walls = BoundarySet.all(BoundaryKind.wall())
    pol = StabilityPolicy(cfl=0.45)
    for par in (0, 1):
        ga = Stepper(a.spec, PhysicsParams(), pol, walls, EXACT)
        gb = Stepper(b.spec, PhysicsParams(), pol, walls, EXACT)
        ga.load(a)
        gb.load(b)
        dt = 0.5 * ga.compute_dt(1e9)
        ga.step(dt, par)
        gb.step(dt, par)
        x, y = ga.state(), gb.state()
        assert bits_equal(x.h, y.h.T) and bits_equal(x.qx, y.qy.T) and bits_equal(x.qy, y.qx.T)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_full_size_c3_frictionless_against_reference():
    # BASELINE config 3 at 8192^2 (frictionless variant): 2 steps vs the reference decomposed:N
    sc = S.gen_channel_flood(8192, manning_n=0.0)
    fs = sc.build()
    g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, EXACT)
    g.load(fs)
    r = O.RefStepper(sc.spec, sc.phys, sc.pol, sc.bounds, O.REF_DECOMPOSED, os.cpu_count() or 1)
    r.load(fs)
    dg, dr = g.compute_dt(math.inf), r.compute_dt(math.inf, os.cpu_count() or 1)
    assert dg == dr
    for k in range(2):
        dg = g.step(dg, k).dt_next
        dr = r.step(dr, k).dt_next
        assert dg == dr
    x, y = g.state(), r.state()
    assert bits_equal(x.h, y.h) and bits_equal(x.qx, y.qx) and bits_equal(x.qy, y.qy)


def test_cpp_shim():
    exe = os.path.join(ROOT, "build", "shim_test")
    assert os.path.exists(exe), "run __graft_entry__.build()"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def test_launch_count_is_one_kernel_per_step():
    sc = S.gen_square_dam(512)
    g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, EXACT)
    g.load(sc.build())
    n0 = g.launch_count()
    g.advance(1e18, 0, math.nan, 128)
    # one step kernel per step, or (small grids) one multi-step launch
    assert g.launch_count() - n0 in (128, 1)


@pytest.mark.parametrize("edge", ["north", "south", "east", "west"])
@pytest.mark.parametrize("kind", [EXACT, FAST], ids=["exact", "fast"])
def test_inflow_admits_the_prescribed_volume_on_every_edge(edge, kind):
    """test_executor.cpp:192-222: one inflow edge at a time, 60 steps; the added
    volume equals q_n * edge length * t to 1e-12."""
    spec = GridSpec(24, 18, 1.0, 1.0)
    fs = FieldSet(spec)
    fs.h[:] = 1.0
    walls = dict(north=BoundaryKind.wall(), south=BoundaryKind.wall(), east=BoundaryKind.wall(),
                 west=BoundaryKind.wall())
    walls[edge] = BoundaryKind.inflow(0.05, 1.0)
    bounds = BoundarySet(**walls)
    pol = StabilityPolicy(cfl=0.45)
    st = Stepper(spec, PhysicsParams(), pol, bounds, kind)
    st.load(fs)
    dt = st.compute_dt(1e18)
    t = 0.0
    for k in range(60):
        t += dt
        dt = st.step(dt, k).dt_next
    added = st.state().h.sum() - fs.h.sum()
    edge_len = 18.0 if edge in ("east", "west") else 24.0
    assert abs(added - 0.05 * edge_len * t) <= 1e-12 * (0.05 * edge_len * t)


@pytest.mark.parametrize("bed", ["x", "y", "xy"])
def test_bed_variants_match_oracle(bed):
    """Sloped beds select the kernel that reads both slopes, or -- when every
    dz/dy bit pattern is +0.0 -- the one that reads dz/dx only; both must be
    bit-identical to the oracle (exact mode) and within tolerance (fast)."""
    spec = GridSpec(96, 80, 1.0, 1.0)
    i = np.arange(spec.nx, dtype=np.float64)[None, :]
    j = np.arange(spec.ny, dtype=np.float64)[:, None]
    z = np.zeros((spec.ny, spec.nx))
    if "x" in bed:
        z = z + 0.002 * (spec.nx - 1 - i) + 0.01 * np.sin(0.3 * i)
    if "y" in bed:
        z = z + 0.003 * j + 0.01 * np.cos(0.25 * j)
    fs = FieldSet(spec, z=z, h=1.0 - z + 0.02 * np.exp(-((i - 40) ** 2 + (j - 30) ** 2) / 50.0))
    phys, pol = PhysicsParams(manning_n=0.0), StabilityPolicy(cfl=0.45)
    bounds = BoundarySet(north=BoundaryKind.wall(), south=BoundaryKind.transmissive(),
                         east=BoundaryKind.fixed_eta(1.0), west=BoundaryKind.inflow(0.05, 1.0))
    ora = O.OracleStepper(spec, phys, pol, bounds)
    ora.load(fs)
    dt = ora.compute_dt(math.inf)
    for k in range(40):
        dt = ora.step(dt, k).dt_next
    ref = ora.state()
    for kind in (EXACT, FAST):
        st = Stepper(spec, phys, pol, bounds, kind)
        st.load(fs)
        d = st.compute_dt(math.inf)
        for k in range(40):
            d = st.step(d, k).dt_next
        got = st.state()
        if kind is EXACT:
            assert bits_equal(got.h, ref.h) and bits_equal(got.qx, ref.qx) and bits_equal(got.qy, ref.qy)
            assert d == dt
        else:
            assert max_err(got.h, got.qx, got.qy, ref.h, ref.qx, ref.qy) <= FAST_TOL


def _dt_outcome(st, fs):
    """compute_dt's value, or the error it raises (type, cell), for one state."""
    try:
        st.load(fs)
        return ("ok", st.compute_dt(math.inf))
    except Exception as e:  # noqa: BLE001 -- the error itself is compared
        cell = (e.cell_i(), e.cell_j()) if hasattr(e, "cell_i") else None
        return (type(e).__name__, cell)


@pytest.mark.parametrize("kind", [EXACT, FAST], ids=["exact", "fast"])
def test_compute_dt_extreme_speeds_match_oracle(kind):
    # The exact scan folds cells whose CFL quotients are certainly finite into
    # two speed maxima and takes per-cell quotients only for the others
    # (swe_aux.cu scan_kernel): both paths, the bad-ratio error and the
    # reference's std::min NaN asymmetry, against the oracle's compute_dt.
    spec = GridSpec(40, 24, 1.0, 2.0)
    j, i = np.mgrid[0:spec.ny, 0:spec.nx].astype(float)
    base_h = 1.0 + 0.1 * np.sin(0.3 * i) * np.cos(0.2 * j)
    base_qx = 0.3 * np.cos(0.1 * i)
    base_qy = -0.2 * np.sin(0.15 * j)
    pol = StabilityPolicy(cfl=0.45, dt_min=1e-310)
    cases_ = {
        "plain": {},
        "huge_qx": {"qx": (7, 5, 5e302)},          # dx/sx ~ 2e-303: per-cell path, still finite
        "huge_qy": {"qy": (20, 11, -3e305)},       # dy/sy ~ 7e-306
        "nan_qy": {"qy": (3, 2, math.nan)},        # std::min(dx/sx, NaN) keeps dx/sx: not bad
        "nan_qx": {"qx": (9, 9, math.nan)},        # std::min(NaN, dy/sy) is NaN: bad at (9, 9)
        "inf_qx": {"qx": (30, 4, math.inf)},       # dx/inf = 0: bad
        "tiny_h": {"h": (12, 6, 1e-310)},          # subnormal depth: huge speeds
    }
    for name, mods in cases_.items():
        h, qx, qy = base_h.copy(), base_qx.copy(), base_qy.copy()
        for field, (ci, cj, val) in mods.items():
            {"h": h, "qx": qx, "qy": qy}[field][cj, ci] = val
        fs = FieldSet(spec, z=np.zeros_like(h), h=h, qx=qx, qy=qy)
        g = Stepper(spec, PhysicsParams(), pol, BoundarySet(), kind)
        o = O.OracleStepper(spec, PhysicsParams(), pol, BoundarySet())
        got, want = _dt_outcome(g, fs), _dt_outcome(o, fs)
        assert got == want, name
        if O.ref_available():  # the reference itself, one worker (its first-offender order)
            r = O.RefStepper(spec, PhysicsParams(), pol, BoundarySet(), O.REF_NAIVE, 1)
            assert _dt_outcome(r, fs) == want, name


@pytest.mark.parametrize("nx,ny", [(31, 17), (61, 33), (95, 200), (130, 67), (257, 129), (300, 41)])
def test_odd_shapes_channel_flood_match_oracle(nx, ny):
    # Window / item geometry edge cases for every kernel family the channel
    # flood selects (sloped bed along x, Manning friction: the fast kernels
    # with the padding-column epilogue and the late ring refill; the exact
    # ones): widths that leave partial windows, heights that leave partial
    # items and row groups.  Exact mode within the Manning tolerance (std::pow),
    # fast mode within FAST_TOL, dt_next alike.
    base = S.gen_channel_flood(64)
    spec = GridSpec(nx, ny, 1.0, 1.0)
    slope = 0.5 / (nx - 1)
    i = np.arange(nx, dtype=float)[None, :].repeat(ny, axis=0)
    z = slope * (nx - 1 - i)
    fs = FieldSet(spec, z=z, h=np.maximum(1.0 - z, 0.05) + 0.01 * np.sin(0.2 * i), qx=np.zeros_like(z),
                  qy=np.zeros_like(z))
    ora = O.OracleStepper(spec, base.phys, base.pol, base.bounds)
    ora.load(fs)
    dt = ora.compute_dt(math.inf)
    d_o = dt
    for k in range(25):
        d_o = ora.step(d_o, k).dt_next
    ref = ora.state()
    for kind in (EXACT, FAST):
        st = Stepper(spec, base.phys, base.pol, base.bounds, kind)
        st.load(fs)
        d = st.compute_dt(math.inf)
        assert d == dt
        for k in range(25):
            d = st.step(d, k).dt_next
        got = st.state()
        assert max_err(got.h, got.qx, got.qy, ref.h, ref.qx, ref.qy) <= (MANNING_TOL if kind is EXACT else FAST_TOL)
        assert abs(d - d_o) <= 1e-12 * d_o
        # the same 25 steps through the device-resident loop (multi-step
        # launches at these sizes: one march body, run-time group rows, their
        # own item heights, grid sync)
        sa = Stepper(spec, base.phys, base.pol, base.bounds, kind)
        sa.load(fs)
        r = sa.advance(1e18, 0, dt, 25)
        assert r.steps == 25
        ga = sa.state()
        assert bits_equal(ga.h, got.h) and bits_equal(ga.qx, got.qx) and bits_equal(ga.qy, got.qy)
        assert r.dt_next == d


@pytest.mark.parametrize("nx,ny", [(61, 33), (130, 67), (257, 129)])
@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_odd_shapes_smoothing_and_early_exit(nx, ny, exact):
    # Smoothing (R = 2: 28-column windows, 5-row stencil) and wet/dry early
    # exit on odd shapes: a square dam with a quiet right half.  Smoothing vs
    # the oracle; early exit bit-identical to the non-skipping kernel, both
    # through step() and advance().
    spec = GridSpec(nx, ny, 1.0, 1.0)
    i = np.arange(nx, dtype=float)[None, :].repeat(ny, axis=0)
    h = np.where(i < nx // 3, 1.0, 0.6)
    fs = FieldSet(spec, z=np.zeros_like(h), h=h, qx=np.zeros_like(h), qy=np.zeros_like(h))
    bounds = BoundarySet.all(BoundaryKind.wall())
    pol = StabilityPolicy(cfl=0.45)
    # smoothing
    phys = PhysicsParams(nu_art=0.05)
    ora = O.OracleStepper(spec, phys, pol, bounds)
    ora.load(fs)
    d_o = dt = ora.compute_dt(math.inf)
    for k in range(20):
        d_o = ora.step(d_o, k).dt_next
    ref = ora.state()
    st = Stepper(spec, phys, pol, bounds, ExecutorKind(exact=exact))
    st.load(fs)
    d = st.compute_dt(math.inf)
    assert d == dt
    for k in range(20):
        d = st.step(d, k).dt_next
    got = st.state()
    if exact:
        assert bits_equal(got.h, ref.h) and bits_equal(got.qx, ref.qx) and bits_equal(got.qy, ref.qy) and d == d_o
    else:
        assert max_err(got.h, got.qx, got.qy, ref.h, ref.qx, ref.qy) <= FAST_TOL
    # early exit (no smoothing) against the non-skipping kernel
    phys = PhysicsParams()
    runs = []
    for early in (False, True):
        for api in ("step", "advance"):
            s2 = Stepper(spec, phys, pol, bounds, ExecutorKind(exact=exact, early_exit=early))
            s2.load(fs)
            d2 = s2.compute_dt(math.inf)
            if api == "step":
                for k in range(40):
                    d2 = s2.step(d2, k).dt_next
            else:
                d2 = s2.advance(1e18, 0, d2, 40).dt_next
            runs.append((s2.state(), d2))
    base, d_base = runs[0]
    for got, d2 in runs[1:]:
        assert bits_equal(got.h, base.h) and bits_equal(got.qx, base.qx) and bits_equal(got.qy, base.qy)
        assert d2 == d_base


def test_graph_capture_failure_falls_back_to_plain_launches(monkeypatch, capfd):
    # a step graph that cannot be captured (SWE_DEBUG_GRAPH_FAIL simulates it)
    # is not a run error: advance() launches the same steps without graphs
    sc = S.gen_channel_flood(1100, manning_n=0.035)  # > kMultiMaxCells: per-step launches
    fs = sc.build()
    out = []
    for fail in ("0", "1"):
        monkeypatch.setenv("SWE_DEBUG_GRAPH_FAIL", fail)
        st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, FAST)
        st.load(fs)
        r = st.advance(1e18, 0, math.nan, 20)
        out.append((st.state(), r.steps, r.dt_next, st.launch_count()))
        st.close()
    (a, na, da, la), (b, nb, db, lb) = out
    assert na == nb == 20 and da == db and la == lb == 20
    assert bits_equal(a.h, b.h) and bits_equal(a.qx, b.qx) and bits_equal(a.qy, b.qy)
    assert "launching steps without graphs" in capfd.readouterr().err
