"""The BASELINE.json configurations at their real sizes.

C1  256^2 square dam break, 1000 steps: exact mode reproduces the reference's
    SWS1 digest, final time and dt_next bit for bit; fast mode is within the
    stated tolerance (1e-12 absolute and relative on h, u = qx/h, v = qy/h).
C2  512^2 square dam break: exact mode bit-identical to the oracle.
C3  8192^2 channel flood with Manning friction (the headline workload): fast
    and exact mode within tolerance of the unmodified reference
    (oracle/_ref, decomposed executor) after 10 steps.
C4  32768^2 square dam break: one domain and 2/4/8 row strips (local-group
    transport on this device) reach the same state bit for bit after 20 steps
    (swe_cuda_state_digest, no host copy of the 26 GB state).
C5  16384^2 mostly-dry floodplain: early-exit tiles bit-identical to the
    non-skipping kernel over 300 steps, in both arithmetic modes.
"""
import hashlib
import math
import os
import threading

import numpy as np
import pytest

from golden_cases import bits_equal
from oracle import oracle as O
from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200.io import snapshot_bytes
from paper_1309_1230_b200.stepper import ExecutorKind, Stepper

pytestmark = pytest.mark.gpu

TOL = 1e-12  # absolute and relative (max |d| / max |ref|) on h, u, v: DESIGN.md "Fast mode"

C1_SHA1000 = "d7bfdd4a414e20cc1ca2a1efbec15df2964480eff75aad38d719aae8296708d1"
C1_T1000 = 119.62189476928548
C1_DT1000 = 0.11430104431145062


def errors(a, b):
    """max abs and max relative (normwise) differences of h, u, v."""
    out = {}
    for name, x, y in (("h", a.h, b.h), ("u", a.qx / a.h, b.qx / b.h), ("v", a.qy / a.h, b.qy / b.h)):
        d = float(np.abs(x - y).max())
        m = float(np.abs(y).max())
        out[name] = (d, d / m if m > 0 else d)
    return out


def gpu_run(sc, exact, steps, early=False, initial=False):
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact, early_exit=early))
    if initial:
        st.load_initial(sc.initial)
    else:
        st.load(sc.build())
    r = st.advance(1e18, 0, math.nan, steps)
    assert r.steps == steps
    return st, r


def test_c1_exact_1000_steps_reproduces_the_reference_digest():
    st, r = gpu_run(S.gen_square_dam(256), True, 1000)
    fin = st.state()
    assert fin.t == C1_T1000
    assert r.dt_next == C1_DT1000
    assert hashlib.sha256(snapshot_bytes(fin, 9.81)).hexdigest() == C1_SHA1000


def test_c1_fast_1000_steps_within_tolerance():
    sc = S.gen_square_dam(256)
    st, r = gpu_run(sc, False, 1000)
    fin = st.state()
    ref = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    ref.load(sc.build())
    rr = ref.advance(1e18, 0, math.nan, 1000)
    e = errors(fin, ref.state())
    for name, (ab, rel) in e.items():
        assert ab <= TOL and rel <= TOL, (name, ab, rel)
    assert abs(r.t_final - rr.t_final) <= TOL * rr.t_final
    assert abs(r.dt_next - rr.dt_next) <= TOL * rr.dt_next


def test_c2_exact_bit_identical_to_oracle():
    sc = S.gen_square_dam(512)
    st, r = gpu_run(sc, True, 200)
    ref = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    ref.load(sc.build())
    rr = ref.advance(1e18, 0, math.nan, 200)
    a, b = st.state(), ref.state()
    assert bits_equal(a.h, b.h) and bits_equal(a.qx, b.qx) and bits_equal(a.qy, b.qy)
    assert (r.t_final, r.dt_next) == (rr.t_final, rr.dt_next)


@pytest.fixture(scope="module")
def c3_reference():
    """10 steps of the unmodified reference on the full C3 grid (host cores)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    sc = S.gen_channel_flood(8192)
    st = O.RefStepper(sc.spec, sc.phys, sc.pol, sc.bounds, O.REF_DECOMPOSED, os.cpu_count() or 1)
    st.load(sc.build())
    dt = st.compute_dt(math.inf)
    for k in range(10):
        dt = st.step(dt, k).dt_next
    return sc, st.state(), dt


@pytest.mark.parametrize("exact", [False, True], ids=["fast", "exact"])
def test_c3_full_size_manning_against_reference(c3_reference, exact):
    sc, ref, dt_ref = c3_reference
    st, r = gpu_run(sc, exact, 10, initial=True)
    fin = st.state()
    st.close()
    e = errors(fin, ref)
    for name, (ab, rel) in e.items():
        assert ab <= TOL and rel <= TOL, (name, ab, rel)
    assert abs(r.t_final - ref.t) <= TOL * ref.t
    assert abs(r.dt_next - dt_ref) <= TOL * dt_ref


@pytest.mark.parametrize("exact", [False, True], ids=["fast", "exact"])
def test_c5_early_exit_bit_identical_over_300_steps(exact):
    sc = S.gen_floodplain(16384)
    a, ra = gpu_run(sc, exact, 300, early=True, initial=True)
    skipped = a.activity()["skipped_cells"]
    da = a.state_digest()
    a.close()
    b, rb = gpu_run(sc, exact, 300, early=False, initial=True)
    db = b.state_digest()
    b.close()
    assert skipped > 0  # the early-exit path did skip work
    assert (ra.t_final, ra.dt_next) == (rb.t_final, rb.dt_next)
    assert da == db


def _strip_digest(sc, nranks, exact, steps):
    key = os.urandom(16).hex().encode()
    out = [None] * nranks
    errs = []

    def worker(r):
        try:
            kind = ExecutorKind(exact=exact, rank=r, nranks=nranks, local_group=True, graph=False)
            st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind, nccl_id=key)
            st.load_initial(sc.initial)
            res = st.advance(1e18, 0, math.nan, steps)
            out[r] = (st.state_digest(), res.t_final, res.dt_next, res.steps)
            st.close()
        except Exception as e:  # surfaced below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not errs, errs
    assert len({o[1:] for o in out}) == 1  # every rank agrees on t, dt_next, steps
    return sum(o[0] for o in out) % (1 << 64), out[0][1:]


def test_c4_full_size_strips_bit_identical_to_one_domain():
    sc = S.gen_square_dam(32768)
    st, r = gpu_run(sc, False, 20, initial=True)
    d1 = st.state_digest()
    st.close()
    for n in (2, 4, 8):
        dn, (t, dt, steps) = _strip_digest(sc, n, False, 20)
        assert steps == 20
        assert (t, dt) == (r.t_final, r.dt_next), n
        assert dn == d1, n


def _np_digest(fs):
    """numpy restatement of swe_cuda_state_digest (splitmix64 mix, sum mod 2^64)."""
    def mix(x):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))
    with np.errstate(over="ignore"):
        idx = np.arange(fs.spec.cell_count(), dtype=np.uint64)
        x = mix(idx)
        for a in (fs.h, fs.qx, fs.qy):
            x = mix(x ^ np.ascontiguousarray(a).reshape(-1).view(np.uint64))
        return int(x.sum(dtype=np.uint64))


def test_state_digest_matches_host_restatement():
    sc = S.gen_floodplain(96)
    st, _ = gpu_run(sc, True, 7)
    assert st.state_digest() == _np_digest(st.state())
