"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

  OracleStepper : oracle/_build/libswe_oracle.so, the plain-C restatement of the
                  reference's naive executor (oracle/swe_oracle.c)
  RefStepper    : oracle/_ref/libswe_ref.so, the UNMODIFIED reference headers
                  compiled in place (oracle/Makefile, oracle/ref_driver.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module; the product path (paper_1309_1230_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from paper_1309_1230_b200 import abi
from paper_1309_1230_b200.stepper import (FieldSet, GridSpec, PhysicsParams, StabilityPolicy, BoundarySet,
                                          BoundaryKind, StepResult, RunResult, raise_status, _bc)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libswe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libswe_ref.so")

DP = abi.DP
ST = abi.ST

_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = C.CDLL(ORACLE_SO)
        L.swo_create.restype = C.c_void_p
        L.swo_create.argtypes = [C.POINTER(abi.swe_grid), C.POINTER(abi.swe_physics), C.POINTER(abi.swe_policy),
                                 C.POINTER(abi.swe_boundary_set)]
        L.swo_destroy.argtypes = [C.c_void_p]
        L.swo_load.argtypes = [C.c_void_p, DP, DP, DP, DP, C.c_double]
        L.swo_state.argtypes = [C.c_void_p, DP, DP, DP, DP]
        L.swo_time.restype = C.c_double
        L.swo_time.argtypes = [C.c_void_p]
        L.swo_guard_warnings.argtypes = [C.c_void_p]
        L.swo_step.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_double, DP, C.POINTER(C.c_int), ST]
        L.swo_compute_dt.argtypes = [C.c_void_p, C.c_double, DP, ST]
        L.swo_guard.argtypes = [C.c_void_p, ST]
        L.swo_advance.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_double, C.c_uint64,
                                  C.POINTER(abi.swe_run_result), ST]
        L.swo_build_initial.argtypes = [C.POINTER(abi.swe_grid), C.c_int, C.c_double, DP, C.c_int, C.c_double,
                                        C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                        C.c_double, DP, DP, DP, DP]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing: build with `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(REF_SO)
        L.swr_create.restype = C.c_void_p
        L.swr_create.argtypes = [C.POINTER(abi.swe_grid), C.POINTER(abi.swe_physics), C.POINTER(abi.swe_policy),
                                 C.POINTER(abi.swe_boundary_set), C.c_int, C.c_int, C.c_int, ST]
        L.swr_destroy.argtypes = [C.c_void_p]
        L.swr_load.argtypes = [C.c_void_p, DP, DP, DP, DP, C.c_double, ST]
        L.swr_state.argtypes = [C.c_void_p, DP, DP, DP, DP]
        L.swr_step.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_double, DP, C.POINTER(C.c_int), ST]
        L.swr_time.restype = C.c_double
        L.swr_time.argtypes = [C.c_void_p]
        L.swr_compute_dt.argtypes = [C.c_void_p, C.c_double, C.c_int, DP, ST]
        L.swr_guard.argtypes = [C.c_void_p, ST]
        L.swr_guard_warnings.argtypes = [C.c_void_p]
        L.swr_scenario.argtypes = [C.c_char_p, C.c_int, C.POINTER(abi.swe_grid), C.POINTER(abi.swe_physics),
                                   C.POINTER(abi.swe_policy), C.POINTER(abi.swe_boundary_set), DP, DP, DP, DP,
                                   DP, ST]
        L.swr_run_config.argtypes = [C.c_char_p, C.c_char_p, C.c_double, ST]
        L.swr_snapshot_bytes.restype = C.c_longlong
        L.swr_snapshot_bytes.argtypes = [C.POINTER(abi.swe_grid), C.c_double, C.c_double, DP, DP, DP, DP,
                                         C.c_char_p, C.c_longlong]
        _ref = L
    return _ref


def _structs(spec, phys, pol, bounds):
    return (abi.swe_grid(spec.nx, spec.ny, float(spec.dx), float(spec.dy)),
            abi.swe_physics(phys.g, phys.manning_n, phys.nu_art),
            abi.swe_policy(pol.cfl, pol.dt_max, pol.dt_min, pol.h_min),
            abi.swe_boundary_set(_bc(bounds.north), _bc(bounds.south), _bc(bounds.east), _bc(bounds.west)))


class OracleStepper:
    """Same interface as paper_1309_1230_b200.Stepper, computed by the C restatement."""

    def __init__(self, spec: GridSpec, phys: PhysicsParams, pol: StabilityPolicy, bounds: BoundarySet):
        self.L = oracle_lib()
        self.spec = spec
        self._s = _structs(spec, phys, pol, bounds)
        self.h = self.L.swo_create(*[C.byref(x) for x in self._s])

    def __del__(self):
        if getattr(self, "h", None):
            self.L.swo_destroy(self.h)
            self.h = None

    def load(self, fs: FieldSet):
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (fs.z, fs.h, fs.qx, fs.qy)]
        self.z = self._keep[0].copy()
        self.L.swo_load(self.h, *[abi.dptr(a) for a in self._keep], float(fs.t))

    def state(self) -> FieldSet:
        shape = (self.spec.ny, self.spec.nx)
        h, qx, qy = (np.empty(shape) for _ in range(3))
        self.L.swo_state(self.h, abi.dptr(h), abi.dptr(qx), abi.dptr(qy), None)
        return FieldSet(self.spec, self.z.copy(), h, qx, qy, self.L.swo_time(self.h))

    def time(self):
        return self.L.swo_time(self.h)

    def guard_warnings(self):
        return self.L.swo_guard_warnings(self.h)

    def step(self, dt, step_index, t_after=math.nan) -> StepResult:
        dtn = C.c_double()
        w = C.c_int()
        st = abi.swe_status()
        rc = self.L.swo_step(self.h, float(dt), int(step_index), float(t_after), C.byref(dtn), C.byref(w),
                             C.byref(st))
        if rc:
            raise_status(st)
        return StepResult(dt, dtn.value, w.value)

    def compute_dt(self, t_end):
        dt = C.c_double()
        st = abi.swe_status()
        rc = self.L.swo_compute_dt(self.h, float(t_end), C.byref(dt), C.byref(st))
        if rc:
            raise_status(st)
        return dt.value

    def guard(self):
        st = abi.swe_status()
        rc = self.L.swo_guard(self.h, C.byref(st))
        if rc:
            raise_status(st)

    def advance(self, t_end, step_index0=0, dt_first=math.nan, max_steps=0) -> RunResult:
        res = abi.swe_run_result()
        st = abi.swe_status()
        rc = self.L.swo_advance(self.h, float(t_end), int(step_index0), float(dt_first), int(max_steps),
                                C.byref(res), C.byref(st))
        self.last_run = RunResult(res.steps, res.step_index, res.t_final, res.dt_next, res.guard_warnings)
        if rc:
            raise_status(st)
        return self.last_run


# executor kinds of the reference (ref_driver.cpp to_kind)
REF_NAIVE, REF_TILED, REF_DECOMPOSED, REF_DECOMPOSED_TILED = 0, 1, 2, 3


class RefStepper:
    """The unmodified reference swe::Stepper (naive / tiled / decomposed:N)."""

    def __init__(self, spec, phys, pol, bounds, kind=REF_NAIVE, workers=1, tile=16):
        self.L = ref_lib()
        self.spec = spec
        self._s = _structs(spec, phys, pol, bounds)
        st = abi.swe_status()
        self.h = self.L.swr_create(*[C.byref(x) for x in self._s], kind, workers, tile, C.byref(st))
        if not self.h:
            raise_status(st)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.swr_destroy(self.h)
            self.h = None

    def load(self, fs: FieldSet):
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (fs.z, fs.h, fs.qx, fs.qy)]
        self.z = arrs[0].copy()
        st = abi.swe_status()
        rc = self.L.swr_load(self.h, *[abi.dptr(a) for a in arrs], float(fs.t), C.byref(st))
        if rc:
            raise_status(st)

    def state(self) -> FieldSet:
        shape = (self.spec.ny, self.spec.nx)
        h, qx, qy = (np.empty(shape) for _ in range(3))
        t = C.c_double()
        self.L.swr_state(self.h, abi.dptr(h), abi.dptr(qx), abi.dptr(qy), C.byref(t))
        return FieldSet(self.spec, self.z.copy(), h, qx, qy, t.value)

    def time(self):
        return self.L.swr_time(self.h)

    def guard_warnings(self):
        return self.L.swr_guard_warnings(self.h)

    def step(self, dt, step_index, t_after=math.nan) -> StepResult:
        dtn = C.c_double()
        w = C.c_int()
        st = abi.swe_status()
        rc = self.L.swr_step(self.h, float(dt), int(step_index), float(t_after), C.byref(dtn), C.byref(w),
                             C.byref(st))
        if rc:
            raise_status(st)
        return StepResult(dt, dtn.value, w.value)

    def compute_dt(self, t_end, workers=1):
        dt = C.c_double()
        st = abi.swe_status()
        rc = self.L.swr_compute_dt(self.h, float(t_end), int(workers), C.byref(dt), C.byref(st))
        if rc:
            raise_status(st)
        return dt.value

    def guard(self):
        st = abi.swe_status()
        rc = self.L.swr_guard(self.h, C.byref(st))
        if rc:
            raise_status(st)


def ref_run_config(text: str, out_dir: str, snapshot_every: float = -1.0) -> int:
    """The reference's `run` (parse_config + run, run.hpp:101-179) into out_dir; returns its exit code."""
    st = abi.swe_status()
    return ref_lib().swr_run_config(text.encode(), out_dir.encode(), float(snapshot_every), C.byref(st))


def ref_scenario(name: str, n: int = 0):
    """(spec, phys, pol, bounds, t_end, FieldSet) of the reference preset gen_<name>(n)."""
    L = ref_lib()
    g, p, po, b = abi.swe_grid(), abi.swe_physics(), abi.swe_policy(), abi.swe_boundary_set()
    t_end = C.c_double()
    st = abi.swe_status()
    rc = L.swr_scenario(name.encode(), n, C.byref(g), C.byref(p), C.byref(po), C.byref(b), C.byref(t_end),
                        None, None, None, None, C.byref(st))
    if rc:
        raise_status(st)
    spec = GridSpec(g.nx, g.ny, g.dx, g.dy)
    arrs = [np.empty((g.ny, g.nx)) for _ in range(4)]
    rc = L.swr_scenario(name.encode(), n, C.byref(g), C.byref(p), C.byref(po), C.byref(b), C.byref(t_end),
                        *[abi.dptr(a) for a in arrs], C.byref(st))
    if rc:
        raise_status(st)

    def bk(x):
        return BoundaryKind(x.type, x.q_n, x.h_in, x.eta_out)

    return (spec, PhysicsParams(p.g, p.manning_n, p.nu_art), StabilityPolicy(po.cfl, po.dt_max, po.dt_min, po.h_min),
            BoundarySet(bk(b.north), bk(b.south), bk(b.east), bk(b.west)), t_end.value,
            FieldSet(spec, *arrs, t=0.0))


def oracle_initial(spec: GridSpec, kind: str, **kw) -> FieldSet:
    """build_initial_state via the C restatement (uses libm exp like std::exp)."""
    L = oracle_lib()
    kinds = {"flat_pool": 0, "drops": 1, "channel_slope": 2, "vortex": 3, "dam_break": 4}
    drops = np.ascontiguousarray(np.array(kw.get("drops", [[0, 0, 1, 0]]), dtype=np.float64).reshape(-1, 4))
    arrs = [np.empty((spec.ny, spec.nx)) for _ in range(4)]
    g = abi.swe_grid(spec.nx, spec.ny, float(spec.dx), float(spec.dy))
    L.swo_build_initial(C.byref(g), kinds[kind], float(kw.get("depth", 1.0)), abi.dptr(drops),
                        int(len(drops)) if "drops" in kw else 0, float(kw.get("slope", 0.0)),
                        float(kw.get("center_x", 0.0)), float(kw.get("center_y", 0.0)), float(kw.get("v_peak", 0.0)),
                        float(kw.get("core_radius", 1.0)), float(kw.get("split_x", 0.0)),
                        float(kw.get("h_left", 1.0)), float(kw.get("h_right", 1.0)), *[abi.dptr(a) for a in arrs])
    return FieldSet(spec, *arrs, t=0.0)


def five_drops(n: int) -> FieldSet:
    """gen_five_drops(n) initial state (scenarios.hpp:192-213) via the C restatement."""
    c = (n - 1) / 2.0
    d = n / 4.0
    r0 = n / 20.0
    drops = [[c, c, r0, 0.3], [c - d, c - d, r0, 0.3], [c - d, c + d, r0, 0.3], [c + d, c - d, r0, 0.3],
             [c + d, c + d, r0, 0.3]]
    return oracle_initial(GridSpec(n, n, 1.0, 1.0), "drops", depth=1.0, drops=drops)


def vortex(n: int) -> FieldSet:
    """gen_vortex(n) initial state (scenarios.hpp:259-276)."""
    return oracle_initial(GridSpec(n, n, 1.0, 1.0), "vortex", depth=2.0, center_x=(n - 1) / 2.0,
                          center_y=(n - 1) / 2.0, v_peak=0.5, core_radius=n / 8.0)
