"""Row-strip decomposition on one B200 through the local-group transport.

The strip path (partition_scanlines bands, per-strip padded buffers with R
halo rows, no in-kernel finalize, unsigned-max allreduce of the reduction
words, halo send/recv, finalize kernel, bed-halo exchange at load) is the one
the NCCL build runs across GPUs; SWE_EXEC_LOCAL_GROUP swaps only the
transport (CUDA-event-ordered device copies between contexts of this process,
one host thread per rank), so the kernels and the protocol are checked here
bit for bit against the single-domain run -- the reference's own contract for
its decomposed executor (executor.hpp:913-1084: bit-identical to naive).
"""
import math
import os
import threading

import numpy as np
import pytest

from golden_cases import bits_equal
from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200.stepper import ExecutorKind, FieldSet, GridSpec, InstabilityError, Stepper

pytestmark = pytest.mark.gpu


def run_single(sc, exact, steps, early=False, api="advance"):
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact, early_exit=early))
    st.load(sc.build())
    out = _drive(st, steps, api)
    fs = st.state()
    st.close()
    return fs, out


def _drive(st, steps, api):
    try:
        if api == "advance":
            r = st.advance(1e18, 0, math.nan, steps)
            return ("ok", r.steps, r.dt_next, r.t_final)
        dt = st.compute_dt(math.inf)
        for k in range(steps):
            dt = st.step(dt, k).dt_next
        return ("ok", steps, dt, st.time())
    except InstabilityError as e:
        return ("instability", e.i, e.j, e.t)


def run_strips(sc, nranks, exact, steps, early=False, api="advance"):
    key = os.urandom(16).hex().encode()
    full = sc.build()
    results = [None] * nranks
    states = [None] * nranks
    launches = [0] * nranks
    acc = [None] * nranks
    xt = [None] * nranks
    errors = []

    def worker(r):
        try:
            kind = ExecutorKind(exact=exact, early_exit=early, rank=r, nranks=nranks, local_group=True,
                                graph=False)
            st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind, nccl_id=key)
            r0, r1 = st.row_begin, st.row_end
            st.load_rows(full.z[r0:r1], full.h[r0:r1], full.qx[r0:r1], full.qy[r0:r1], full.t)
            results[r] = _drive(st, steps, api)
            shape = (r1 - r0, sc.spec.nx)
            h, qx, qy = np.empty(shape), np.empty(shape), np.empty(shape)
            st.state_rows(h, qx, qy)
            states[r] = (r0, r1, h, qx, qy, st.time())
            launches[r] = st.launch_count()
            acc[r] = st.accounting()
            xt[r] = st.exchange_timing()
            st.close()
        except Exception as e:  # surfaced by the caller
            errors.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errors, errors
    fs = FieldSet(sc.spec, full.z.copy())
    for r0, r1, h, qx, qy, t in states:
        fs.h[r0:r1], fs.qx[r0:r1], fs.qy[r0:r1], fs.t = h, qx, qy, t
    assert all(x == results[0] for x in results), results  # every rank sees the same outcome
    run_strips.launches = launches
    run_strips.accounting = acc
    run_strips.exchange = xt
    return fs, results[0]


def same(a, b):
    return bits_equal(a.h, b.h) and bits_equal(a.qx, b.qx) and bits_equal(a.qy, b.qy) and a.t == b.t


def _rect_channel():
    sc = S.gen_channel_flood(200, manning_n=0.0)
    sc.spec = GridSpec(200, 173, 1.0, 1.0)
    return sc


def _rect_channel_manning():
    sc = S.gen_channel_flood(300, manning_n=0.035)
    sc.spec = GridSpec(300, 181, 1.0, 1.0)
    return sc


SCEN = {
    "dam256": lambda: S.gen_square_dam(256, 1.0, 0.5),                       # R = 1, walls
    "floodplain256": lambda: S.gen_floodplain(256),                          # R = 2 (smoothing)
    "channel_rect": _rect_channel,                                           # sloped bed, inflow / fixed eta
    "channel_manning_rect": _rect_channel_manning,                           # + Manning: the padding-column epilogue
}


@pytest.mark.parametrize("halo", ["push", "sendrecv"])
@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("name", sorted(SCEN))
def test_strips_bit_identical_exact(name, nranks, halo, monkeypatch):
    monkeypatch.setenv("SWE_P2P", "1" if halo == "push" else "0")
    sc = SCEN[name]()
    ref, rr = run_single(sc, True, 60)
    got, rg = run_strips(sc, nranks, True, 60)
    assert rr == rg
    assert same(ref, got)
    rows = sc.spec.ny // nranks
    if halo == "push":
        # fused halo push: one step kernel (it stores its edge rows into the
        # neighbours' halos), the local group's allreduce kernel, the finalize
        assert all(n == 3 * 60 for n in run_strips.launches), run_strips.launches
    else:
        # send/recv: edge + interior step kernels when strips of >= 32 rows
        # overlap the halo exchange (one step kernel otherwise), the finalize
        # kernel, and the local group's allreduce kernel
        assert all(n == (4 if rows >= 32 else 3) * 60 for n in run_strips.launches), run_strips.launches
    # StepAccounting: R halo rows of h, qx, qy from each neighbour
    R = 2 if sc.phys.nu_art > 0 else 1
    halo = [a["halo_values_exchanged"] for a in run_strips.accounting]
    assert halo == [(1 if r in (0, nranks - 1) else 2) * R * 3 * sc.spec.nx for r in range(nranks)]


@pytest.mark.parametrize("halo", ["push", "sendrecv"])
@pytest.mark.parametrize("name", sorted(SCEN))
def test_strips_bit_identical_fast(name, halo, monkeypatch):
    monkeypatch.setenv("SWE_P2P", "1" if halo == "push" else "0")
    sc = SCEN[name]()
    ref, rr = run_single(sc, False, 60)
    got, rg = run_strips(sc, 4, False, 60)
    assert rr == rg
    assert same(ref, got)


@pytest.mark.parametrize("halo", ["push", "sendrecv"])
def test_strips_host_step_api(halo, monkeypatch):
    monkeypatch.setenv("SWE_P2P", "1" if halo == "push" else "0")
    sc = S.gen_floodplain(192)
    ref, rr = run_single(sc, True, 30, api="step")
    got, rg = run_strips(sc, 3, True, 30, api="step")
    assert rr == rg and same(ref, got)
    # step() times the halo exchange (none with the fused push: the step kernel
    # stores the rows) and the allreduce of every strip
    for x in run_strips.exchange:
        assert x["steps"] == 30 and x["allreduce_seconds"] > 0.0
        assert (x["exchange_seconds"] == 0.0) if halo == "push" else (x["exchange_seconds"] > 0.0)


@pytest.mark.parametrize("halo", ["push", "sendrecv"])
def test_strips_with_early_exit(halo, monkeypatch):
    monkeypatch.setenv("SWE_P2P", "1" if halo == "push" else "0")
    sc = S.gen_floodplain(320)
    ref, rr = run_single(sc, True, 60)
    got, rg = run_strips(sc, 2, True, 60, early=True)
    assert rr == rg and same(ref, got)


def test_strips_report_first_offender_like_single_domain():
    """A thin film without smoothing collapses (SURVEY.md §8(d) C5 note); the
    strips must raise the same InstabilityError (cell and time) as one domain."""
    sc = S.gen_square_dam(96, 1.0, 0.01)
    ref, rr = run_single(sc, True, 200)
    assert rr[0] == "instability"
    got, rg = run_strips(sc, 4, True, 200)
    assert rg == rr
    assert same(ref, got)  # committed state untouched by the failed step, on every strip


# ---------------------------------------------------------------- on-device initial conditions
def _load_both(sc):
    a = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=True))
    b = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=True))
    a.load(sc.build())
    b.load_initial(sc.initial)
    return a, b


@pytest.mark.parametrize("name", ["dam256", "channel_rect", "floodplain256"])
def test_load_initial_matches_host_build(name):
    """swe_cuda_load_initial == build_initial_state + load, bit for bit (z too)."""
    sc = SCEN[name]()
    a, b = _load_both(sc)
    sa, sb = a.state(), b.state()
    assert same(sa, sb) and bits_equal(sa.z, sb.z)
    ra = a.advance(1e18, 0, math.nan, 25)
    rb = b.advance(1e18, 0, math.nan, 25)
    assert ra.dt_next == rb.dt_next and same(a.state(), b.state())


def test_load_initial_rejects_guard_failure_and_exp_kinds():
    from paper_1309_1230_b200.stepper import ConfigError, InitialCondition
    sc = S.gen_square_dam(64, 1.0, 0.0)  # h_right below h_min: build_initial_state's guard throws
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind())
    with pytest.raises(ConfigError):
        st.load_initial(sc.initial)
    with pytest.raises(ConfigError):
        st.load_initial(InitialCondition(kind=1))  # drops: std::exp, host-built only


def test_load_initial_on_strips():
    sc = S.gen_channel_flood(160, manning_n=0.0)
    ref, rr = run_single(sc, True, 30)
    key = os.urandom(16).hex().encode()
    outs, errs = [None] * 3, []

    def worker(r):
        try:
            st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds,
                         ExecutorKind(rank=r, nranks=3, local_group=True), nccl_id=key)
            st.load_initial(sc.initial)
            res = _drive(st, 30, "advance")
            outs[r] = (st.row_begin, st.row_end, st.state(), res)
            st.close()
        except Exception as e:
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(3)]
    [t.start() for t in th]
    [t.join(timeout=600) for t in th]
    assert not errs, errs
    for r0, r1, fs, res in outs:
        assert res == rr
        assert bits_equal(fs.h[r0:r1], ref.h[r0:r1]) and bits_equal(fs.qx[r0:r1], ref.qx[r0:r1])
        assert bits_equal(fs.qy[r0:r1], ref.qy[r0:r1]) and bits_equal(fs.z[r0:r1], ref.z[r0:r1])


def test_strips_mixing_overlapped_and_plain_steps(monkeypatch):
    """ny = 127 on 4 strips gives bands of 32, 32, 32 and 31 rows: the first
    three overlap their halo exchange, the last does not -- the collectives
    must still pair up (same order on every rank) and the result must equal
    the single domain (send/recv halo transport)."""
    monkeypatch.setenv("SWE_P2P", "0")
    sc = S.gen_square_dam(127, 1.0, 0.5)
    ref, rr = run_single(sc, True, 40)
    got, rg = run_strips(sc, 4, True, 40)
    assert rr == rg and same(ref, got)
    assert run_strips.launches == [4 * 40, 4 * 40, 4 * 40, 3 * 40]
