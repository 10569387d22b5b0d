"""Host-side mirror of the reference's Stepper API over the libswe_cuda.so C-ABI.

Same names, fields, argument meaning and error behaviour as
/root/reference/proj/include/swe/{grid,scheme,timestep,executor,errors}.hpp,
so parity tests read like the reference's own tests.  There is no CPU path:
construction fails loudly when the CUDA library (or a GPU) is missing.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import abi


# ---------------------------------------------------------------- errors.hpp:9-70
class SweError(RuntimeError):
    code = abi.SWE_ERR_RUNTIME


class ConfigError(SweError):
    code = abi.SWE_ERR_CONFIG


class InstabilityError(SweError):
    """errors.hpp:27-40: carries the first offending cell and the sim time."""

    code = abi.SWE_ERR_INSTABILITY

    def __init__(self, msg, i=-1, j=-1, t=0.0):
        super().__init__(msg)
        self.i, self.j, self.t = i, j, t

    def cell_i(self):
        return self.i

    def cell_j(self):
        return self.j

    def sim_time(self):
        return self.t


class StepCollapseError(SweError):
    code = abi.SWE_ERR_STEP_COLLAPSE

    def __init__(self, msg, dt=0.0, t=0.0):
        super().__init__(msg)
        self._dt, self._t = dt, t

    def dt(self):
        return self._dt

    def sim_time(self):
        return self._t


class IoError(SweError):
    code = abi.SWE_ERR_IO


class DeviceError(SweError):
    code = abi.SWE_ERR_RUNTIME


def raise_status(st: abi.swe_status):
    msg = st.msg.decode(errors="replace")
    if st.code == abi.SWE_ERR_CONFIG:
        raise ConfigError(msg)
    if st.code == abi.SWE_ERR_INSTABILITY:
        raise InstabilityError(msg, st.i, st.j, st.t)
    if st.code == abi.SWE_ERR_STEP_COLLAPSE:
        raise StepCollapseError(msg, st.dt, st.t)
    if st.code == abi.SWE_ERR_IO:
        raise IoError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------- grid.hpp / scheme.hpp / timestep.hpp
@dataclass(frozen=True)
class GridSpec:
    nx: int
    ny: int
    dx: float = 1.0
    dy: float = 1.0

    def cell_count(self) -> int:
        return self.nx * self.ny


@dataclass(frozen=True)
class PhysicsParams:
    g: float = 9.81
    manning_n: float = 0.0
    nu_art: float = 0.0


@dataclass(frozen=True)
class StabilityPolicy:
    cfl: float = 0.9
    dt_max: float = math.inf
    dt_min: float = 1e-9
    h_min: float = 1e-6


@dataclass(frozen=True)
class BoundaryKind:
    type: int = abi.SWE_BC_WALL
    q_n: float = 0.0
    h_in: float = 0.0
    eta_out: float = 0.0

    @staticmethod
    def wall():
        return BoundaryKind()

    @staticmethod
    def transmissive():
        return BoundaryKind(abi.SWE_BC_TRANSMISSIVE)

    @staticmethod
    def inflow(q_n, h_in):
        return BoundaryKind(abi.SWE_BC_INFLOW, q_n, h_in, 0.0)

    @staticmethod
    def fixed_eta(eta):
        return BoundaryKind(abi.SWE_BC_FIXED_ETA, 0.0, 0.0, eta)


@dataclass(frozen=True)
class BoundarySet:
    north: BoundaryKind = BoundaryKind()
    south: BoundaryKind = BoundaryKind()
    east: BoundaryKind = BoundaryKind()
    west: BoundaryKind = BoundaryKind()

    @staticmethod
    def all(bk: BoundaryKind):
        return BoundarySet(bk, bk, bk, bk)


@dataclass
class FieldSet:
    """grid.hpp:136-164: SoA fp64, row-major, x fastest (arrays shaped (ny, nx))."""

    spec: GridSpec
    z: np.ndarray = None
    h: np.ndarray = None
    qx: np.ndarray = None
    qy: np.ndarray = None
    t: float = 0.0

    def __post_init__(self):
        shape = (self.spec.ny, self.spec.nx)
        for name in ("z", "h", "qx", "qy"):
            a = getattr(self, name)
            a = np.zeros(shape) if a is None else np.ascontiguousarray(a, dtype=np.float64).reshape(shape)
            setattr(self, name, a)

    def copy(self):
        return FieldSet(self.spec, self.z.copy(), self.h.copy(), self.qx.copy(), self.qy.copy(), self.t)


@dataclass(frozen=True)
class InitialCondition:
    """InitialCondition (scenarios.hpp:26-42) for the kinds generated on the device."""

    kind: int = abi.SWE_IC_FLAT_POOL
    depth: float = 1.0
    slope: float = 0.0
    split_x: float = 0.0
    h_left: float = 1.0
    h_right: float = 1.0

    @staticmethod
    def flat_pool(depth):
        return InitialCondition(abi.SWE_IC_FLAT_POOL, depth)

    @staticmethod
    def channel_slope(depth, slope):
        return InitialCondition(abi.SWE_IC_CHANNEL_SLOPE, depth, slope)

    @staticmethod
    def dam_break(split_x, h_left, h_right):
        return InitialCondition(abi.SWE_IC_DAM_BREAK, 1.0, 0.0, split_x, h_left, h_right)


@dataclass
class StepResult:
    dt_used: float = 0.0
    dt_next: float = 0.0
    guard_warnings: int = 0


@dataclass
class RunResult:
    steps: int = 0
    step_index: int = 0
    t_final: float = 0.0
    dt_next: float = 0.0
    guard_warnings: int = 0


@dataclass(frozen=True)
class ExecutorKind:
    """ExecutorKind (executor.hpp:27-67) restricted to the new `cuda` strategy."""

    exact: bool = True
    device: int = 0
    graph: bool = True
    rank: int = 0
    nranks: int = 1
    early_exit: bool = False  # skip quiet items on a flat bed (bit-exact; SWE_EXEC_EARLY_EXIT)
    local_group: bool = False  # strips as contexts of one process on one device (SWE_EXEC_LOCAL_GROUP)

    def name(self):
        return ("cuda" + ("" if self.nranks == 1 else f":{self.nranks}") + ("" if self.exact else ":fast")
                + (":early" if self.early_exit else ""))


def _bc(bk: BoundaryKind) -> abi.swe_boundary:
    return abi.swe_boundary(int(bk.type), float(bk.q_n), float(bk.h_in), float(bk.eta_out))


class Stepper:
    """swe::Stepper (executor.hpp:726-1116) on one B200 (or one row strip)."""

    def __init__(self, spec: GridSpec, phys: PhysicsParams, pol: StabilityPolicy,
                 bounds: BoundarySet, kind: ExecutorKind = ExecutorKind(), nccl_id: bytes | None = None):
        self._lib = abi.load_library()
        self.spec, self.phys, self.pol, self.bounds, self.kind = spec, phys, pol, bounds, kind
        g = abi.swe_grid(spec.nx, spec.ny, float(spec.dx), float(spec.dy))
        p = abi.swe_physics(phys.g, phys.manning_n, phys.nu_art)
        po = abi.swe_policy(pol.cfl, pol.dt_max, pol.dt_min, pol.h_min)
        b = abi.swe_boundary_set(_bc(bounds.north), _bc(bounds.south), _bc(bounds.east), _bc(bounds.west))
        flags = ((abi.SWE_EXEC_EXACT if kind.exact else 0) | (0 if kind.graph else abi.SWE_EXEC_NO_GRAPH)
                 | (abi.SWE_EXEC_EARLY_EXIT if kind.early_exit else 0)
                 | (abi.SWE_EXEC_LOCAL_GROUP if kind.local_group else 0))
        self._id_buf = C.create_string_buffer(nccl_id, abi.SWE_NCCL_ID_BYTES) if nccl_id else None
        ex = abi.swe_exec(kind.device, flags, kind.rank, kind.nranks,
                          C.cast(self._id_buf, C.c_void_p) if self._id_buf is not None else None)
        self._ctx = C.c_void_p()
        st = abi.swe_status()
        rc = self._lib.swe_cuda_create(C.byref(g), C.byref(p), C.byref(po), C.byref(b), C.byref(ex),
                                       C.byref(self._ctx), C.byref(st))
        if rc:
            if self._ctx:
                self._lib.swe_cuda_destroy(self._ctx)
                self._ctx = C.c_void_p()
            raise_status(st)
        rb, re_ = C.c_int32(), C.c_int32()
        self._lib.swe_cuda_rows(self._ctx, C.byref(rb), C.byref(re_))
        self.row_begin, self.row_end = rb.value, re_.value

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.swe_cuda_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, st):
        if rc:
            raise_status(st)

    # executor.hpp:764-780
    def load(self, fs: FieldSet):
        if fs.spec != self.spec:
            raise ConfigError("Stepper::load: grid mismatch")
        rows = slice(self.row_begin, self.row_end)
        arrs = [np.ascontiguousarray(a[rows], dtype=np.float64) for a in (fs.z, fs.h, fs.qx, fs.qy)]
        self.load_rows(*arrs, t=fs.t)

    def load_rows(self, z, h, qx, qy, t=0.0):
        """Load this rank's rows [row_begin, row_end) directly (strip mode)."""
        st = abi.swe_status()
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (z, h, qx, qy)]
        rc = self._lib.swe_cuda_load(self._ctx, *[abi.dptr(a) for a in arrs], float(t), C.byref(st))
        self._check(rc, st)

    def load_initial(self, ic: InitialCondition, t: float = 0.0):
        """build_initial_state (scenarios.hpp:95-171) + load, generated on the device."""
        st = abi.swe_status()
        c_ic = abi.swe_initial(int(ic.kind), float(ic.depth), float(ic.slope), float(ic.split_x),
                               float(ic.h_left), float(ic.h_right))
        rc = self._lib.swe_cuda_load_initial(self._ctx, C.byref(c_ic), float(t), C.byref(st))
        self._check(rc, st)

    # executor.hpp:783-797
    def state(self) -> FieldSet:
        nrows = self.row_end - self.row_begin
        shape = (nrows, self.spec.nx)
        z, h, qx, qy = (np.empty(shape) for _ in range(4))
        t = C.c_double()
        st = abi.swe_status()
        rc = self._lib.swe_cuda_state(self._ctx, abi.dptr(z), abi.dptr(h), abi.dptr(qx), abi.dptr(qy),
                                      C.byref(t), C.byref(st))
        self._check(rc, st)
        if nrows == self.spec.ny:
            return FieldSet(self.spec, z, h, qx, qy, t.value)
        fs = FieldSet(self.spec, t=t.value)
        for name, a in (("z", z), ("h", h), ("qx", qx), ("qy", qy)):
            getattr(fs, name)[self.row_begin:self.row_end] = a
        return fs

    def state_rows(self, h=None, qx=None, qy=None):
        """Copy this rank's rows into preallocated (nrows, nx) arrays."""
        st = abi.swe_status()
        t = C.c_double()
        rc = self._lib.swe_cuda_state(self._ctx, None, abi.dptr(h), abi.dptr(qx), abi.dptr(qy), C.byref(t),
                                      C.byref(st))
        self._check(rc, st)
        return t.value

    def time(self) -> float:
        return self._lib.swe_cuda_time(self._ctx)

    def guard_warnings(self) -> int:
        return self._lib.swe_cuda_guard_warnings(self._ctx)

    # executor.hpp:812-841
    def step(self, dt: float, step_index: int, t_after: float = math.nan) -> StepResult:
        res = abi.swe_step_result()
        st = abi.swe_status()
        rc = self._lib.swe_cuda_step(self._ctx, float(dt), int(step_index), float(t_after), C.byref(res),
                                     C.byref(st))
        self._check(rc, st)
        return StepResult(res.dt_used, res.dt_next, res.guard_warnings)

    # timestep.hpp:128-179 on the loaded state
    def compute_dt(self, t_end: float) -> float:
        dt = C.c_double()
        st = abi.swe_status()
        rc = self._lib.swe_cuda_compute_dt(self._ctx, float(t_end), C.byref(dt), C.byref(st))
        self._check(rc, st)
        return dt.value

    # timestep.hpp:112-115 on the loaded state
    def guard(self):
        st = abi.swe_status()
        rc = self._lib.swe_cuda_guard(self._ctx, C.byref(st))
        self._check(rc, st)

    # run.hpp:149-163, device resident
    def advance(self, t_end: float, step_index0: int = 0, dt_first: float = math.nan,
                max_steps: int = 0, t_mark: float = math.inf) -> RunResult:
        """t_mark: also stop after the first committed step with t >= t_mark
        (snapshot cadence, run.hpp:159-163; swe_cuda_advance_marked)."""
        res = abi.swe_run_result()
        st = abi.swe_status()
        if math.isinf(t_mark):
            rc = self._lib.swe_cuda_advance(self._ctx, float(t_end), int(step_index0), float(dt_first),
                                            int(max_steps), C.byref(res), C.byref(st))
        else:
            rc = self._lib.swe_cuda_advance_marked(self._ctx, float(t_end), float(t_mark), int(step_index0),
                                                   float(dt_first), int(max_steps), C.byref(res), C.byref(st))
        self.last_run = RunResult(res.steps, res.step_index, res.t_final, res.dt_next, res.guard_warnings)
        self._check(rc, st)
        return self.last_run

    def launch_count(self) -> int:
        return self._lib.swe_cuda_launch_count(self._ctx)

    def timing(self):
        t = abi.swe_timing()
        self._lib.swe_cuda_timing(self._ctx, C.byref(t))
        return t.steps, t.step_seconds

    def exchange_timing(self) -> dict:
        """Strips, step() calls only: device time of the halo send/recv
        (overlapped with the interior rows) and of the allreduce."""
        t = abi.swe_timing()
        self._lib.swe_cuda_timing(self._ctx, C.byref(t))
        return {"steps": t.exchange_steps, "exchange_seconds": t.exchange_seconds,
                "allreduce_seconds": t.allreduce_seconds}

    def accounting(self) -> dict:
        """StepAccounting (executor.hpp:218-222, 804) of this rank, per step."""
        a = abi.swe_accounting()
        self._lib.swe_cuda_accounting(self._ctx, C.byref(a))
        return {"halo_values_exchanged": a.halo_values_exchanged, "redundant_star_rows": a.redundant_star_rows,
                "redundant_corrector_rows": a.redundant_corrector_rows}

    def plan(self) -> list:
        """StepPlan::standard(nu_art > 0) (executor.hpp:134-148); one fused launch runs all of it."""
        k = ["k1_ghost_committed", "k2_predictor", "k3_ghost_star", "k4_corrector"]
        return k + (["smooth"] if self.phys.nu_art > 0 else []) + ["k5_guard", "k6_dt_reduce"]

    def activity(self) -> dict:
        """Early-exit counters since the last load (swe_cuda_activity)."""
        a = abi.swe_activity()
        self._lib.swe_cuda_activity(self._ctx, C.byref(a))
        return {"cells_per_step": a.cells_per_step, "items_per_step": a.items_per_step,
                "eligible_items": a.eligible_items, "skipped_cells": a.skipped_cells}

    def halo_rows(self) -> int:
        return self._lib.swe_cuda_halo_rows(self._ctx)

    def state_digest(self) -> int:
        """This rank's additive digest of the committed state (swe_cuda_state_digest);
        the whole grid's digest is the sum of the ranks' values mod 2**64."""
        d = C.c_uint64()
        st = abi.swe_status()
        rc = self._lib.swe_cuda_state_digest(self._ctx, C.byref(d), C.byref(st))
        self._check(rc, st)
        return d.value


def strip_rows(ny: int, nranks: int, rank: int):
    """The rows (begin, end) libswe_cuda gives `rank` of `nranks` strips
    (swe_cuda_strip_rows: partition_scanlines + the >= 4-row band rule).  Host
    only: callable without a GPU."""
    b, e = C.c_int32(), C.c_int32()
    st = abi.swe_status()
    if abi.load_library().swe_cuda_strip_rows(int(ny), int(nranks), int(rank), C.byref(b), C.byref(e), C.byref(st)):
        raise_status(st)
    return b.value, e.value


def partition_scanlines(ny: int, workers: int):
    """executor.hpp:189-208: contiguous bands, sizes differ by <= 1, larger first."""
    if workers < 1:
        raise ConfigError("partition_scanlines: workers must be >= 1")
    if ny < workers:
        raise ConfigError(f"partition_scanlines: {workers} workers need at least as many rows, grid has {ny}")
    base, rem = divmod(ny, workers)
    bands, j = [], 0
    for w in range(workers):
        rows = base + (1 if w < rem else 0)
        bands.append((j, j + rows))
        j += rows
    return bands
