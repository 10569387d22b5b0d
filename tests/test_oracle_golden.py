"""The CPU oracle (oracle/swe_oracle.c) is pinned to the reference before it
is trusted: bit-exact on every golden fixture made by the unmodified
reference, on the SURVEY.md §8(c) SWS1 digests, and on the reference's own
known-answer values (test_timestep.cpp:36-44)."""
import hashlib
import math

import numpy as np
import pytest

from golden_cases import bits_equal, cases
from oracle import oracle as O
from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200.io import parse_snapshot, snapshot_bytes
from paper_1309_1230_b200.stepper import (BoundaryKind, BoundarySet, FieldSet, GridSpec, InstabilityError,
                                          PhysicsParams, StabilityPolicy)

CASES = cases()


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_oracle_matches_reference_golden(case):
    st = O.OracleStepper(case.spec, case.phys, case.pol, case.bounds)
    fin, err, dt_next, warnings = case.run(st)
    assert err == case.expected_error()
    assert bits_equal(fin.h, case.h) and bits_equal(fin.qx, case.qx) and bits_equal(fin.qy, case.qy)
    assert fin.t == case.meta["t_final"]
    if err is None:
        assert dt_next == case.meta["dt_next"]
        assert warnings == case.meta["warnings"]


def _config1_hash(steps):
    sc = S.gen_square_dam(256)
    st = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    st.load(sc.build())
    dt = st.compute_dt(math.inf)
    for k in range(steps):
        dt = st.step(dt, k).dt_next
    fin = st.state()
    return hashlib.sha256(snapshot_bytes(fin, 9.81)).hexdigest(), fin.t, dt


def test_config1_200_steps_sha256():
    # identical at -O0 and -O3 in the reference
    h, t, _ = _config1_hash(200)
    assert h == "80558353ce400f9234ab754787dbcd000acbb12fdc0ee2c6042eed2c3d963efe"


@pytest.mark.slow
def test_config1_1000_steps_sha256():
    h, t, dt = _config1_hash(1000)
    assert h == "d7bfdd4a414e20cc1ca2a1efbec15df2964480eff75aad38d719aae8296708d1"
    assert t == 119.62189476928548
    assert dt == 0.11430104431145062


def test_compute_dt_frozen_value():
    # test_timestep.cpp:36-44: still water 9x9, cfl 0.9 -> 0.28734788556634544
    spec = GridSpec(9, 9, 1.0, 1.0)
    st = O.OracleStepper(spec, PhysicsParams(), StabilityPolicy(), BoundarySet.all(BoundaryKind.wall()))
    st.load(S.flat_pool(spec, 1.0))
    assert st.compute_dt(1e9) == 0.28734788556634544


def test_compute_dt_clamps_to_remaining_time():
    # test_timestep.cpp:47-56
    spec = GridSpec(9, 9, 1.0, 1.0)
    fs = S.flat_pool(spec, 1.0)
    fs.t = 5.0
    st = O.OracleStepper(spec, PhysicsParams(), StabilityPolicy(), BoundarySet.all(BoundaryKind.wall()))
    st.load(fs)
    assert abs(st.compute_dt(5.1) - 0.1) < 1e-15


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [3, 11, 2024])
def test_oracle_equals_reference_on_random_states(seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    spec = GridSpec(19, 23, 1.0, 1.0)
    fs = FieldSet(spec)
    fs.h[:] = rng.uniform(0.5, 3.0, fs.h.shape)
    fs.qx[:] = rng.uniform(-0.5, 0.5, fs.h.shape)
    fs.qy[:] = rng.uniform(-0.5, 0.5, fs.h.shape)
    fs.z[:] = rng.uniform(-0.05, 0.05, fs.h.shape)
    bounds = BoundarySet(BoundaryKind.transmissive(), BoundaryKind.inflow(0.07, 1.0), BoundaryKind.fixed_eta(1.2),
                         BoundaryKind.wall())
    for nu in (0.0, 0.03):
        phys = PhysicsParams(nu_art=nu)
        pol = StabilityPolicy(cfl=0.3)
        a, b = O.OracleStepper(spec, phys, pol, bounds), O.RefStepper(spec, phys, pol, bounds)
        a.load(fs)
        b.load(fs)
        da, db = a.compute_dt(1e9), b.compute_dt(1e9)
        assert da == db
        for k in range(8):
            try:
                ra = a.step(da, k)
            except InstabilityError as e:
                with pytest.raises(InstabilityError) as eb:
                    b.step(db, k)
                assert (e.i, e.j, e.t) == (eb.value.i, eb.value.j, eb.value.t)
                break
            rb = b.step(db, k)
            assert ra.dt_next == rb.dt_next
            da, db = ra.dt_next, rb.dt_next
        x, y = a.state(), b.state()
        assert bits_equal(x.h, y.h) and bits_equal(x.qx, y.qx) and bits_equal(x.qy, y.qy)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_snapshot_bytes_match_reference_writer():
    sc = S.gen_channel_flood(33)
    fs = sc.build()
    fs.t = 1.25
    L = O.ref_lib()
    import ctypes as C
    from paper_1309_1230_b200 import abi
    g = abi.swe_grid(fs.spec.nx, fs.spec.ny, fs.spec.dx, fs.spec.dy)
    n = L.swr_snapshot_bytes(C.byref(g), fs.t, 9.81, *[abi.dptr(np.ascontiguousarray(a)) for a in
                                                       (fs.z, fs.h, fs.qx, fs.qy)], None, 0)
    buf = C.create_string_buffer(n)
    L.swr_snapshot_bytes(C.byref(g), fs.t, 9.81, *[abi.dptr(np.ascontiguousarray(a)) for a in
                                                   (fs.z, fs.h, fs.qx, fs.qy)], buf, n)
    assert snapshot_bytes(fs, 9.81) == buf.raw
    back, g2, ex = parse_snapshot(snapshot_bytes(fs, 9.81, dt_next=0.5, step_index=7))
    assert g2 == 9.81 and ex == {"dt_next": 0.5, "step_index": 7}
    assert bits_equal(back.h, fs.h) and back.t == 1.25


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,n", [("channel-flood", 67), ("dam-break", 64)])
def test_numpy_scenarios_match_reference_build_initial_state(name, n):
    sp, ph, po, bd, te, ref = O.ref_scenario(name, n)
    sc = S.gen_channel_flood(n) if name == "channel-flood" else S.gen_dam_break(n)
    mine = sc.build()
    assert sc.spec == sp and sc.phys == ph and sc.pol == po and sc.bounds == bd and sc.t_end == te
    for f in ("z", "h", "qx", "qy"):
        assert bits_equal(getattr(mine, f), getattr(ref, f))
