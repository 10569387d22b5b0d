"""Row-strip domain decomposition, exercised on CPU with world_size 2 (gloo).

The multi-GPU path of libswe_cuda.so splits the grid into row strips with
partition_scanlines (executor.hpp:189-208), exchanges committed halo rows with
the strip neighbours every step and all-reduces the CFL minimum
(SURVEY.md §8(e)).  This test runs the same protocol with torch.distributed
(gloo) between two processes, each stepping its strip (plus halo) with the CPU
oracle, and checks that the assembled result is bit-identical to the
single-domain run — the decomposition contract the reference's decomposed
executor pins (test_executor.cpp:151-167).  Each rank takes its rows from
libswe_cuda itself (swe_cuda_strip_rows, host only)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1309_1230_b200 import scenarios as S
from paper_1309_1230_b200.stepper import (BoundaryKind, BoundarySet, FieldSet, GridSpec, PhysicsParams,
                                          StabilityPolicy, partition_scanlines, strip_rows)

HALO = 3  # committed rows beyond the strip that a one-step redundant update needs (2 with smoothing + 1)


def cfl_rows(h, qx, qy, g, dx, dy):
    """min over cells of std::min(dx/sx, dy/sy) (executor.hpp:560-580) with IEEE numpy ops."""
    c = np.sqrt(g * h)
    sx = np.abs(qx / h) + c
    sy = np.abs(qy / h) + c
    a, b = dx / sx, dy / sy
    r = np.where(b < a, b, a)
    return float(r.min())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nu, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ic = O.five_drops(40)
    spec = ic.spec
    bounds = BoundarySet(BoundaryKind.transmissive(), BoundaryKind.wall(), BoundaryKind.fixed_eta(1.0),
                         BoundaryKind.inflow(0.1, 1.0))
    phys, pol = PhysicsParams(nu_art=nu), StabilityPolicy(cfl=0.45)
    # this rank's strip as libswe_cuda assigns it (swe_cuda_strip_rows, the
    # partition swe_cuda_create uses: host only, no GPU needed), checked
    # against the reference's partition_scanlines
    j0, j1 = strip_rows(spec.ny, world, rank)
    assert (j0, j1) == partition_scanlines(spec.ny, world)[rank]
    a, b = max(j0 - HALO, 0), min(j1 + HALO, spec.ny)
    sub = GridSpec(spec.nx, b - a, spec.dx, spec.dy)
    h, qx, qy, z = (x[a:b].copy() for x in (ic.h, ic.qx, ic.qy, ic.z))
    # first dt: all-reduced CFL minimum over own rows (timestep.hpp:128-179)
    m = torch.tensor([cfl_rows(ic.h[j0:j1], ic.qx[j0:j1], ic.qy[j0:j1], phys.g, spec.dx, spec.dy)],
                     dtype=torch.float64)
    dist.all_reduce(m, op=dist.ReduceOp.MIN)
    dt = min(pol.cfl * m.item(), pol.dt_max)
    t = 0.0
    dts = []
    for k in range(steps):
        st = O.OracleStepper(sub, phys, pol, bounds)
        st.load(FieldSet(sub, z, h, qx, qy, t))
        st.step(dt, k)
        fs = st.state()
        own = [f[j0 - a:j1 - a].copy() for f in (fs.h, fs.qx, fs.qy)]
        # halo exchange: own edge rows to the neighbours (the NCCL send/recv of the CUDA path)
        new = [f.copy() for f in (fs.h, fs.qx, fs.qy)]
        reqs = []
        if rank + 1 < world:
            blk = np.ascontiguousarray(np.stack([o[-HALO:] for o in own]))
            reqs.append(dist.isend(torch.from_numpy(blk), rank + 1))
            rbuf = torch.empty((3, b - j1, spec.nx), dtype=torch.float64)
            dist.recv(rbuf, rank + 1)
            for f in range(3):
                new[f][j1 - a:] = rbuf[f].numpy()
        if rank > 0:
            blk = np.ascontiguousarray(np.stack([o[:HALO] for o in own]))
            reqs.append(dist.isend(torch.from_numpy(blk), rank - 1))
            rbuf = torch.empty((3, j0 - a, spec.nx), dtype=torch.float64)
            dist.recv(rbuf, rank - 1)
            for f in range(3):
                new[f][:j0 - a] = rbuf[f].numpy()
        for r in reqs:
            r.wait()
        h, qx, qy = new
        t = t + dt
        dts.append(dt)
        m = torch.tensor([cfl_rows(own[0], own[1], own[2], phys.g, spec.dx, spec.dy)], dtype=torch.float64)
        dist.all_reduce(m, op=dist.ReduceOp.MIN)  # the allreduce-min of the CUDA path
        dt = min(pol.cfl * m.item(), pol.dt_max)
    gathered = [torch.empty(0)] * world
    mine = torch.from_numpy(np.ascontiguousarray(np.stack([h[j0 - a:j1 - a], qx[j0 - a:j1 - a], qy[j0 - a:j1 - a]])))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine.numpy())
    if rank == 0:
        full = np.concatenate(gathered, axis=1)
        np.save(out, full)
        np.save(out + ".dts.npy", np.array(dts + [dt]))
    dist.destroy_process_group()


@pytest.mark.parametrize("nu", [0.0, 0.05])
def test_two_strips_match_single_domain(tmp_path, nu):
    steps = 25
    out = str(tmp_path / "strips.npy")
    mp.spawn(_worker, args=(2, _free_port(), nu, steps, out), nprocs=2, join=True)
    full = np.load(out)
    dts = np.load(out + ".dts.npy")
    ic = O.five_drops(40)
    bounds = BoundarySet(BoundaryKind.transmissive(), BoundaryKind.wall(), BoundaryKind.fixed_eta(1.0),
                         BoundaryKind.inflow(0.1, 1.0))
    ref = O.OracleStepper(ic.spec, PhysicsParams(nu_art=nu), StabilityPolicy(cfl=0.45), bounds)
    ref.load(ic)
    dt = ref.compute_dt(math.inf)
    for k in range(steps):
        assert dt == dts[k]
        dt = ref.step(dt, k).dt_next
    assert dt == dts[-1]
    fin = ref.state()
    for f, x in zip(("h", "qx", "qy"), full):
        assert np.array_equal(x.view(np.uint64), getattr(fin, f).view(np.uint64)), f
