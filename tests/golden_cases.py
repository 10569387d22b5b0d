"""Loader for the golden fixtures in tests/golden/ (made by make_golden.py from
the unmodified reference solver)."""
from __future__ import annotations

import glob
import json
import os

import numpy as np

from paper_1309_1230_b200.stepper import (BoundaryKind, BoundarySet, FieldSet, GridSpec, PhysicsParams,
                                          StabilityPolicy)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Case:
    def __init__(self, path):
        d = np.load(path)
        self.meta = json.loads(str(d["meta"]))
        m = self.meta
        self.name = m["name"]
        self.spec = GridSpec(int(m["grid"][0]), int(m["grid"][1]), m["grid"][2], m["grid"][3])
        self.phys = PhysicsParams(*m["physics"])
        self.pol = StabilityPolicy(*m["policy"])
        bk = [BoundaryKind(int(b[0]), b[1], b[2], b[3]) for b in m["bounds"]]
        self.bounds = BoundarySet(*bk)
        self.ic = FieldSet(self.spec, d["z"], d["h0"], d["qx0"], d["qy0"], 0.0)
        self.h, self.qx, self.qy = d["h"], d["qx"], d["qy"]
        self.dts = d["dts"]
        self.dt0 = float(d["dt0"])
        self.error = m["error"]
        self.manning = self.phys.manning_n > 0.0

    def run(self, stepper):
        """Drive `stepper` exactly like make_golden did; returns (state, error-or-None, dt_next, warnings)."""
        from paper_1309_1230_b200.stepper import SweError
        stepper.load(self.ic)
        dt = stepper.compute_dt(1e18) if not self.meta["dt0_given"] else self.dt0
        warnings = 0
        err = None
        for k in range(self.meta["steps"]):
            try:
                r = stepper.step(dt, self.meta["parity0"] + k)
            except SweError as e:
                err = (k, e.code, getattr(e, "i", -1), getattr(e, "j", -1),
                       e.sim_time() if hasattr(e, "sim_time") else 0.0)
                break
            warnings += r.guard_warnings
            dt = r.dt_next
        return stepper.state(), err, dt, warnings

    def expected_error(self):
        e = self.error
        return None if e is None else (e["step"], e["code"], e["i"], e["j"], e["t"])


def cases():
    return [Case(p) for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))]


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))
