#!/usr/bin/env python3
"""Small step-kernel workloads covering every kernel family the library
launches, at sizes that finish in seconds: the driver of the SWE_CHECKED
build (tools/checked_run.sh: device-side bounds/protocol assertions, guard
bands around every allocation, results compared with the CPU oracle) and of
compute-sanitizer where it is available.

  SWE_CUDA_LIB=paper_1309_1230_b200/lib/libswe_cuda_checked.so python tools/sanitize_cases.py [case ...]
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases: exact / fast x {walls, smoothing, sloped bed + inflow/fixed-eta +
Manning}, early exit (schedule kernel + quiet flags), local-group strips
(edge/interior launches, allreduce kernel, finalize kernel), the device
initial-condition loader and the exact CFL scan.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1309_1230_b200 import scenarios as S  # noqa: E402
from paper_1309_1230_b200.stepper import ExecutorKind, GridSpec, Stepper  # noqa: E402


def _channel(n=96, manning=0.035):
    sc = S.gen_channel_flood(n, manning_n=manning)
    sc.spec = GridSpec(n, n - 7, 1.0, 1.0)
    return sc


def one(sc, exact, steps=6, early=False, graph=True, initial=False):
    st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact, early_exit=early, graph=graph))
    if initial and sc.initial is not None:
        st.load_initial(sc.initial)
    else:
        st.load(sc.build())
    dt = st.compute_dt(math.inf)
    for k in range(2):
        dt = st.step(dt, k).dt_next
    st.advance(1e18, 2, dt, steps)
    st.guard()
    got = st.state()
    check_guards(f"{sc.name} {sc.spec.nx}x{sc.spec.ny}")  # while the buffers are live
    st.close()
    # the checked build must compute what the product build does: compare
    # with the CPU oracle (bit for bit in exact mode without friction)
    from oracle import oracle as O
    ora = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    ora.load(sc.build())
    ora.advance(1e18, 0, math.nan, steps + 2)
    ref = ora.state()
    d = max(float(np.abs(got.h - ref.h).max()), float(np.abs(got.qx - ref.qx).max()),
            float(np.abs(got.qy - ref.qy).max()))
    tol = 0.0 if exact and sc.phys.manning_n == 0.0 else 1e-12
    if not d <= tol:
        raise SystemExit(f"max |gpu - oracle| = {d} > {tol}")


def strips(sc, nranks, exact, steps=6):
    key = os.urandom(16).hex().encode()
    full = sc.build()
    errors = []
    done = threading.Barrier(nranks)

    def worker(r):
        try:
            kind = ExecutorKind(exact=exact, rank=r, nranks=nranks, local_group=True, graph=False)
            st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind, nccl_id=key)
            r0, r1 = st.row_begin, st.row_end
            st.load_rows(full.z[r0:r1], full.h[r0:r1], full.qx[r0:r1], full.qy[r0:r1], 0.0)
            st.advance(1e18, 0, math.nan, steps)
            done.wait()  # every strip's buffers are live for the guard check
            if r == 0:
                check_guards(f"{nranks} strips")
            done.wait()
            st.close()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise SystemExit("strips failed: " + "; ".join(errors))


CASES = {
    "walls_exact": lambda: one(S.gen_square_dam(64), True),
    "walls_fast": lambda: one(S.gen_square_dam(64), False),
    "smooth_exact": lambda: one(S.gen_floodplain(64), True),
    "smooth_fast": lambda: one(S.gen_floodplain(64), False),
    "channel_exact": lambda: one(_channel(), True),
    "channel_fast": lambda: one(_channel(), False),
    "channel_initial": lambda: one(S.gen_channel_flood(96), False, initial=True),
    "early_exact": lambda: one(S.gen_floodplain(128), True, steps=8, early=True),
    "early_fast": lambda: one(S.gen_floodplain(128), False, steps=8, early=True),
    "strips2_exact": lambda: strips(S.gen_square_dam(96), 2, True),
    "strips2_smooth_fast": lambda: strips(S.gen_floodplain(96), 2, False),
}


def check_guards(what):
    g = guard_check()
    if g is None:
        return
    print(f"  {what}: guard bands {g[0]} corrupted bytes in {g[1]} live allocations", flush=True)
    if g[0]:
        raise SystemExit(f"{what}: guard bands corrupted")


def guard_check():
    """Guard bands of every live allocation (SWE_CHECKED builds)."""
    from paper_1309_1230_b200 import abi
    bad, n = C.c_uint64(), C.c_uint64()
    st = abi.swe_status()
    if abi.load_library().swe_cuda_debug_guard_check(C.byref(bad), C.byref(n), C.byref(st)):
        return None
    return bad.value, n.value


def main(argv):
    names = argv or list(CASES)
    for n in names:
        CASES[n]()
        print(f"case {n}: ok", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
