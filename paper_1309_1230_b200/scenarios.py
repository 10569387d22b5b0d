"""Initial conditions that need no transcendental functions (host data prep).

Bit-identical to build_initial_state (scenarios.hpp:95-171) for the flat_pool,
channel_slope and dam_break kinds, and to the presets gen_channel_flood /
gen_dam_break (scenarios.hpp:237-256, 285-306) plus the BASELINE.json synthetic
configs.  Drops and vortex use std::exp and are produced by the test oracle.
"""
from __future__ import annotations

import math

import numpy as np

from .stepper import (BoundaryKind, BoundarySet, FieldSet, GridSpec, InitialCondition, PhysicsParams,
                      StabilityPolicy)

SCENARIO_CFL = 0.45  # scenarios.hpp:177


def flat_pool(spec: GridSpec, depth: float = 1.0) -> FieldSet:
    fs = FieldSet(spec)
    fs.h[:] = depth
    return fs


def channel_slope(spec: GridSpec, depth: float, slope: float) -> FieldSet:
    """scenarios.hpp:125-137: z = slope*dx*(nx-1-i), h = depth - z."""
    fs = FieldSet(spec)
    i = np.arange(spec.nx, dtype=np.float64)
    z = (slope * spec.dx) * (float(spec.nx - 1) - i)
    fs.z[:] = z[None, :]
    fs.h[:] = (depth - z)[None, :]
    return fs


def dam_break(spec: GridSpec, split_x: float, h_left: float, h_right: float) -> FieldSet:
    """scenarios.hpp:155-163: x = (i + 0.5)*dx; h = x < split ? h_l : h_r."""
    fs = FieldSet(spec)
    x = (np.arange(spec.nx, dtype=np.float64) + 0.5) * spec.dx
    fs.h[:] = np.where(x < split_x, h_left, h_right)[None, :]
    return fs


class Scenario:
    """ScenarioConfig subset (scenarios.hpp:57-70).  `ic(spec)` builds the initial
    state on a grid; every IC here is uniform along y, so build_rows() can
    materialise one rank's strip without the full grid."""

    def __init__(self, name, spec, phys, pol, bounds, t_end, ic, initial=None):
        self.name, self.spec, self.phys, self.pol, self.bounds, self.t_end, self.ic = (
            name, spec, phys, pol, bounds, t_end, ic)
        self.initial = initial  # InitialCondition for on-device generation (Stepper.load_initial)

    def build(self) -> FieldSet:
        return self.ic(self.spec)

    def build_rows(self, r0: int, r1: int) -> FieldSet:
        s = self.spec
        return self.ic(GridSpec(s.nx, r1 - r0, s.dx, s.dy))


def gen_channel_flood(n: int = 1024, manning_n: float = 0.035) -> Scenario:
    """scenarios.hpp:237-256 (C3 at n=8192; manning_n=0 gives the frictionless variant)."""
    spec = GridSpec(n, n, 1.0, 1.0)
    slope = 0.5 * 1.0 / ((n - 1) * spec.dx)
    bounds = BoundarySet(north=BoundaryKind.wall(), south=BoundaryKind.wall(),
                         east=BoundaryKind.fixed_eta(1.0), west=BoundaryKind.inflow(0.1, 1.0))
    return Scenario("channel-flood", spec, PhysicsParams(manning_n=manning_n), StabilityPolicy(cfl=SCENARIO_CFL),
                    bounds, 1000.0, lambda sp: channel_slope(sp, 1.0, slope),
                    InitialCondition.channel_slope(1.0, slope))


def gen_square_dam(n: int, h_left: float = 1.0, h_right: float = 0.5, nu_art: float = 0.0,
                   split_x: float | None = None) -> Scenario:
    """BASELINE configs C1/C2/C4/C5: square basin, walls, dam at split_x (default n/2)."""
    spec = GridSpec(n, n, 1.0, 1.0)
    sx = 0.5 * n * spec.dx if split_x is None else split_x
    return Scenario("square-dam", spec, PhysicsParams(nu_art=nu_art), StabilityPolicy(cfl=SCENARIO_CFL),
                    BoundarySet.all(BoundaryKind.wall()), 1e18, lambda sp: dam_break(sp, sx, h_left, h_right),
                    InitialCondition.dam_break(sx, h_left, h_right))


def gen_dam_break(n: int = 400, h_l: float = 1.0, h_r: float = 0.5) -> Scenario:
    """scenarios.hpp:285-306: 3-row channel, transmissive N/S, nu_art 0.05."""
    spec = GridSpec(n, 3, 1.0, 1.0)
    phys = PhysicsParams(nu_art=0.05)
    bounds = BoundarySet(north=BoundaryKind.transmissive(), south=BoundaryKind.transmissive(),
                         east=BoundaryKind.wall(), west=BoundaryKind.wall())
    split = 0.5 * n * spec.dx
    t_end = 0.25 * n * spec.dx / math.sqrt(phys.g * h_l)
    return Scenario("dam-break", spec, phys, StabilityPolicy(cfl=SCENARIO_CFL), bounds, t_end,
                    lambda sp: dam_break(sp, split, h_l, h_r))


def gen_floodplain(n: int = 16384) -> Scenario:
    """C5: mostly-dry floodplain dam break: split_x=n/8, h_r=1e-3, nu_art=0.05."""
    return gen_square_dam(n, 1.0, 1e-3, nu_art=0.05, split_x=n / 8.0)
