#!/usr/bin/env python3
"""Small step-kernel workloads for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family the library launches, at sizes the
sanitizers finish in seconds.

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases: exact / fast x {walls, smoothing, sloped bed + inflow/fixed-eta +
Manning}, early exit (schedule kernel + quiet flags), local-group strips
(edge/interior launches, allreduce kernel, finalize kernel), the device
initial-condition loader and the exact CFL scan.
"""
from __future__ import annotations

import math
import os
import sys
import threading

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
    st.state()
    st.close()


def strips(sc, nranks, exact, steps=6):
    key = os.urandom(16).hex().encode()
    full = sc.build()
    errors = []

    def worker(r):
        try:
            kind = ExecutorKind(exact=exact, rank=r, nranks=nranks, local_group=True, graph=False)
            st = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind, nccl_id=key)
            r0, r1 = st.row_begin, st.row_end
            st.load_rows(full.z[r0:r1], full.h[r0:r1], full.qx[r0:r1], full.qy[r0:r1], 0.0)
            st.advance(1e18, 0, math.nan, steps)
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


def main(argv):
    names = argv or list(CASES)
    for n in names:
        CASES[n]()
        print(f"case {n}: ok", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
