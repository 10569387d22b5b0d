#!/usr/bin/env python3
"""Throughput of the fused MacCormack step on B200 (cell-steps/s, % of HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c3f|c1|c2|c4|c5|d8k]

N=1 runs BASELINE.json's headline workload: the 8192^2 synthetic channel flood
(gen_channel_flood(8192), scenarios.hpp:237-256; Manning 0.035, inflow west,
fixed elevation east, walls N/S).  N>1 (torchrun, one rank per GPU) runs the
same channel with 8192 rows per GPU as NCCL-exchanged row strips (weak
scaling) and adds a `strong_scaling` block: config C4 (32768^2 dam break) on
one GPU and as N strips (north_star's efficiency target).  One JSON line is
printed by rank 0.

--impl reference times the unmodified reference solver (oracle/_ref: the
reference headers compiled in place, decomposed:<host cores> executor) on the
same workload, config and step counts, on the host cores.

--dry-run exercises the multi-rank plumbing (process group, communicator id
broadcast, strip partition, max-over-ranks timing, the JSON line) on CPU with
the gloo backend and no kernel launch (tests/test_bench_gloo.py).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-steps/sec (full 16-substep step) at 8192² and % of HBM roofline"
EXACT_MODE = ("exact (-fmad=false IEEE expression trees: bit-identical to the reference without Manning "
              "friction; within 1e-12 with it, std::pow not being reproducible on CUDA)")
FAST_MODE = ("fast (FMA, refined reciprocals; max |dh|,|du|,|dv| <= 1e-12 after 1000 steps of C1 and "
             "within 1e-12 of the reference after 10 steps of C3, see the parity key)")

CONFIGS = {
    "c3": "8192x8192 synthetic channel flood (gen_channel_flood(8192), Manning 0.035), HBM-roofline benchmark",
    "c3f": "8192x8192 channel flood, frictionless variant (manning_n = 0; bit-exact parity config)",
    "c1": "256x256 square dam break (h_l 1.0, h_r 0.5, walls)",
    "d8k": "8192x8192 square dam break (flat bed; 48 B/cell), roofline probe",
    "c2": "512x512 square dam break (interactive size)",
    "c4": "32768x32768 square dam break (row strips)",
    "c5": "16384x16384 mostly-dry floodplain dam break (split_x = n/8, h_r = 1e-3, nu_art = 0.05)",
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def scenario_for(cfg: str, nranks: int = 1):
    """(scenario, algorithmic bytes per cell-step)."""
    from paper_1309_1230_b200 import scenarios as S
    if cfg in ("c3", "c3f"):
        sc = S.gen_channel_flood(8192, manning_n=0.035 if cfg == "c3" else 0.0)
        if nranks > 1:  # weak scaling: 8192 rows per GPU, same physics per strip
            from paper_1309_1230_b200.stepper import GridSpec
            sc.spec = GridSpec(8192, 8192 * nranks, 1.0, 1.0)
        return sc, 56  # read h,qx,qy,dz/dx + write h,qx,qy (fp64)
    if cfg == "c1":
        return S.gen_square_dam(256), 48
    if cfg == "d8k":
        return S.gen_square_dam(8192), 48
    if cfg == "c2":
        return S.gen_square_dam(512), 48
    if cfg == "c4":
        return S.gen_square_dam(32768), 48
    if cfg == "c5":
        return S.gen_floodplain(16384), 48
    raise SystemExit(f"unknown config {cfg}")


def config_dict(cfg, spec, world, exact, early):
    """The `config` object of both arms' lines (same keys and values)."""
    return {"workload": CONFIGS[cfg], "grid": [spec.nx, spec.ny], "rows_per_gpu": spec.ny // max(world, 1),
            "parallelism": f"row-strips{world}", "dtype": "f64",
            "mode": EXACT_MODE if exact else FAST_MODE,
            "early_exit": bool(early),
            "l2": "state + slopes (>= 48 B/cell x 67M cells) >> 126 MB L2 at 8192^2; no flush needed",
            "timing": "device: CUDA events on the library stream around device-resident advance() "
                      "(CUDA graphs of power-of-two step chunks), max over ranks; reference arm: host wall "
                      "clock around K Stepper::step calls"}


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled in-process through
    NVML every ~2 ms while the timed region runs (the device is found by its
    PCI bus id, so CUDA_VISIBLE_DEVICES does not matter)."""

    REASONS = [("nvmlClocksEventReasonHwSlowdown", "hw_slowdown"),
               ("nvmlClocksEventReasonHwThermalSlowdown", "hw_thermal_slowdown"),
               ("nvmlClocksEventReasonSwThermalSlowdown", "sw_thermal_slowdown"),
               ("nvmlClocksEventReasonSwPowerCap", "sw_power_cap"),
               ("nvmlClocksEventReasonHwPowerBrakeSlowdown", "hw_power_brake_slowdown")]

    def __init__(self, device: int):
        self.samples, self.reasons, self.power = [], set(), []
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            self.N = N
            try:
                pr = torch.cuda.get_device_properties(device)
                bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                self.h = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report why
            self.err = str(e)

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for attr, name in self.REASONS:
                    if r & getattr(N, attr, 0):
                        self.reasons.add(name)
                self.power.append(N.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._stop.clear()
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.thread.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": getattr(self, "err", "")}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s),
                "power_w_max": round(max(self.power), 1) if self.power else None,
                "source": "NVML, in-process, every ~2 ms during the timed region"}


# ------------------------------------------------------------------ reference (CPU) arm
def _ref_stepper(sc, cores):
    from oracle import oracle as O
    return O.RefStepper(sc.spec, sc.phys, sc.pol, sc.bounds, O.REF_DECOMPOSED, cores)


def cpu_baseline_sample(sc, cfg, steps=10):
    """The reference itself (oracle/_ref, decomposed:<cores>) on a bounded sample.
    Grids above 8192^2 are sampled on the same scenario at 8192^2 (per-cell rate):
    the reference needs ~192 B/cell of host memory."""
    from oracle import oracle as O
    from paper_1309_1230_b200 import scenarios as S
    if sc.spec.cell_count() > 8192 * 8192:
        sc = S.gen_floodplain(8192) if cfg == "c5" else S.gen_square_dam(8192)
    cores = os.cpu_count() or 1
    if O.ref_available():
        kind, st = "reference", _ref_stepper(sc, cores)
    else:
        kind, cores = "port", 1
        st = O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)
    st.load(sc.build())
    dt = st.compute_dt(math.inf)
    dt = st.step(dt, 0).dt_next  # warm-up
    t0 = time.perf_counter()
    for k in range(1, steps + 1):
        dt = st.step(dt, k).dt_next
    el = time.perf_counter() - t0
    return {"value": sc.spec.cell_count() * steps / el, "unit": "cell-steps/s", "cores": cores, "kind": kind,
            "sample": f"{sc.spec.nx}x{sc.spec.ny} {cfg}, {steps} timed steps after 1 warm-up, "
                      f"{'decomposed:%d' % cores if kind == 'reference' else 'naive C port'} executor",
            "seconds": round(el, 3)}


def run_reference(args):
    """`--impl reference`: the unmodified reference, same config/metric/steps."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    sc, _ = scenario_for(args.config, 1)
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libswe_ref.so not built"}))
        return 0
    cores = os.cpu_count() or 1
    st = _ref_stepper(sc, cores)
    st.load(sc.build())
    dt = st.compute_dt(math.inf)
    k = 0
    for _ in range(args.warmup):
        dt = st.step(dt, k).dt_next
        k += 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dt = st.step(dt, k).dt_next
        k += 1
    el = time.perf_counter() - t0
    v = sc.spec.cell_count() * args.steps / el
    line = {"metric": METRIC, "value": v, "unit": "cell-steps/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, sc.spec, 1, False, args.config == "c5"),
            "executor": f"reference decomposed:{cores} (oracle/_ref: the reference headers, -O3 -ffp-contract=off)",
            "cpu_baseline": {"value": v, "unit": "cell-steps/s", "cores": cores, "kind": "reference",
                             "sample": f"{args.warmup} warm-up + {args.steps} timed steps of the full "
                                       f"{sc.spec.nx}x{sc.spec.ny} grid on one host"},
            "e2e": {"value": v, "unit": "cell-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ GPU arm
def new_stepper(sc, kind, nccl_id, world, initial=True):
    from paper_1309_1230_b200 import Stepper
    stp = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind, nccl_id=nccl_id)
    if initial and sc.initial is not None:  # generated on the device, bit-identical to the host build
        stp.load_initial(sc.initial)
    elif world == 1:
        stp.load(sc.build())
    else:
        fsr = sc.build_rows(stp.row_begin, stp.row_end)
        stp.load_rows(fsr.z, fsr.h, fsr.qx, fsr.qy, 0.0)
    return stp


def timed_run(sc, kind, nccl_id, args, dist, local, sampler=None, steps=None):
    """W untimed warm-up steps, then exactly K device-resident steps timed with
    CUDA events on the library's stream (max over ranks)."""
    import torch
    steps = steps or args.steps
    world = kind.nranks
    stp = new_stepper(sc, kind, nccl_id, world)
    r0, r1 = stp.row_begin, stp.row_end
    res = stp.advance(1e18, 0, math.nan, args.warmup)
    step0, dt_next = res.step_index, res.dt_next
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0, s0 = stp.timing()
    l0 = stp.launch_count()
    a0 = stp.activity()["skipped_cells"]
    if sampler:
        sampler.__enter__()
    try:
        res = stp.advance(1e18, step0, dt_next, steps)
    finally:
        if sampler:
            sampler.__exit__()
    torch.cuda.synchronize()
    skipped = stp.activity()["skipped_cells"] - a0
    n1, s1 = stp.timing()
    launches = stp.launch_count() - l0
    dev_s = s1 - s0
    if res.steps != steps:
        raise SystemExit(f"bench: only {res.steps} of {steps} steps committed")
    if dist:
        t = torch.tensor([dev_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
        dist.barrier()
    stp.close()
    return dev_s, launches, (r1 - r0) * sc.spec.nx, skipped


def e2e_run(sc, kind, steps, nccl_id=None, dist=None, local=0, api="step"):
    """The reference-facing API end to end: host FieldSet (pinned) -> load ->
    K x Stepper.step() (dt_next read back each step) -> state() to host.
    With N ranks every rank moves its own strip; the time is the max over ranks."""
    import torch
    from paper_1309_1230_b200 import Stepper
    spec = sc.spec
    st = Stepper(spec, sc.phys, sc.pol, sc.bounds, kind, nccl_id=nccl_id)
    r0, r1 = st.row_begin, st.row_end
    rows = r1 - r0
    pinned = [torch.empty((rows, spec.nx), dtype=torch.float64).pin_memory() for _ in range(4)]
    src = sc.build_rows(r0, r1) if kind.nranks > 1 else sc.build()
    for tns, a in zip(pinned, (src.z, src.h, src.qx, src.qy)):
        tns.numpy()[:] = a
    del src
    outs = [torch.empty((rows, spec.nx), dtype=torch.float64).pin_memory() for _ in range(3)]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    st.load_rows(*[p.numpy() for p in pinned], t=0.0)
    t1 = time.perf_counter()
    if api == "advance":
        st.advance(1e18, 0, math.nan, steps)  # run_from's loop on the device (swe_cuda_advance)
    else:
        dt = st.compute_dt(math.inf)
        for k in range(steps):
            dt = st.step(dt, k).dt_next
    t2 = time.perf_counter()
    st.state_rows(*[o.numpy() for o in outs])
    el = time.perf_counter() - t0
    if dist:
        t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    phases = {"load_ms": round((t1 - t0) * 1e3, 2), "steps_ms": round((t2 - t1) * 1e3, 2),
              "state_ms": round((t0 + el - t2) * 1e3, 2)}
    st.close()
    cells = spec.cell_count()
    ctl = 2 * 256 * kind.nranks  # control block H2D + D2H per step() call and rank
    return {"value": cells * steps / el, "unit": "cell-steps/s",
            "h2d_bytes_per_step": (4 * cells * 8) // steps + ctl, "d2h_bytes_per_step": (3 * cells * 8) // steps + ctl,
            "steps": steps, "seconds": round(el, 4), "phases": phases,
            "api": ("Stepper.load(host, pinned) + K x Stepper.step() (dt_next read back each step) + "
                    "Stepper.state() (host); C-ABI swe_cuda_load/step/state" if api == "step" else
                    "Stepper.load(host, pinned) + Stepper.advance(K) (run_from's loop on the device, CUDA graphs) + "
                    "Stepper.state() (host); C-ABI swe_cuda_load/advance/state") +
                   ("; every rank moves its own strip, max over ranks" if kind.nranks > 1 else "")}


def parity_run(sc, exact, steps, local=0):
    """max |d| and max |d| / max |ref| of h, u = qx/h, v = qy/h between this
    build (headline mode) and the unmodified reference (oracle/_ref,
    decomposed:<cores>) after `steps` steps from the same initial state."""
    from oracle import oracle as O
    from paper_1309_1230_b200 import ExecutorKind, Stepper
    if not O.ref_available():
        return {"unavailable": "oracle/_ref/libswe_ref.so not built"}
    fs = sc.build()
    g = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, ExecutorKind(exact=exact, device=local))
    g.load(fs)
    rg = g.advance(1e18, 0, math.nan, steps)
    a = g.state()
    g.close()
    cores = os.cpu_count() or 1
    r = _ref_stepper(sc, cores)
    r.load(fs)
    del fs
    dt = r.compute_dt(math.inf)
    for k in range(steps):
        dt = r.step(dt, k).dt_next
    b = r.state()
    del r
    out = {"steps": steps, "against": f"reference decomposed:{cores} (oracle/_ref)",
           "mode": "exact" if exact else "fast", "t_gpu": rg.t_final, "t_ref": b.t,
           "dt_next_rel": abs(rg.dt_next - dt) / dt}
    for name, x, y in (("h", a.h, b.h), ("u", a.qx / a.h, b.qx / b.h), ("v", a.qy / a.h, b.qy / b.h)):
        d = float(np.abs(x - y).max())
        m = float(np.abs(y).max())
        out[f"max_abs_{name}"] = d
        out[f"max_rel_{name}"] = d / m if m > 0 else (0.0 if d == 0 else math.inf)
    out["definition"] = "max_rel = max |gpu - ref| / max |ref| per field"
    return out


def strong_scaling_c4(args, world, rank, local, dist, new_id, peak):
    """C4 (32768^2 dam break): rank 0 alone on one GPU, then N row strips."""
    import torch
    from paper_1309_1230_b200 import ExecutorKind
    sc, bpc = scenario_for("c4", 1)
    t1 = None
    if rank == 0:
        k1 = ExecutorKind(exact=False, device=local)
        d1, _, _, _ = timed_run(sc, k1, None, args, None, local)
        t1 = d1 / args.steps
    dist.barrier()
    kn = ExecutorKind(exact=False, device=local, rank=rank, nranks=world)
    dn, launches, cells_local, _ = timed_run(sc, kn, new_id(), args, dist, local)
    tn = dn / args.steps
    if rank != 0:
        return None
    cells = sc.spec.cell_count()
    return {"config": CONFIGS["c4"], "grid": [sc.spec.nx, sc.spec.ny], "n_gpus": world, "scaling": "strong",
            "ms_per_step_1gpu": t1 * 1e3, "ms_per_step": tn * 1e3, "value": cells / tn, "unit": "cell-steps/s",
            "efficiency": t1 / (world * tn),
            "roofline_frac_per_gpu": round(bpc * cells_local / tn / 1e9 / peak, 4), "gpu_launches": launches}


def dry_run(args):
    """CPU check of the multi-rank plumbing (gloo): no kernel is launched."""
    import torch.distributed as dist
    from paper_1309_1230_b200.stepper import partition_scanlines
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    ids = [os.urandom(128) if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(ids, src=0)
    sc, bpc = scenario_for(args.config, world)
    j0, j1 = partition_scanlines(sc.spec.ny, world)[rank]
    import torch
    mine = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(mine, op=dist.ReduceOp.MAX)
    got = [None] * world
    if world > 1:
        dist.all_gather_object(got, (rank, j0, j1, ids[0][:8].hex()))
    else:
        got = [(0, j0, j1, ids[0][:8].hex())]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "metric": METRIC, "config":
                          config_dict(args.config, sc.spec, world, args.exact, args.config == "c5"),
                          "strips": [list(g[1:3]) for g in got], "id_prefixes": sorted({g[3] for g in got}),
                          "max_over_ranks": float(mine.item()), "bytes_per_cell": bpc}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--fast", action="store_true", help="headline in FAST mode only (skip the exact-mode line)")
    ap.add_argument("--exact", action="store_true", help="headline in EXACT (-fmad=false, bit-identical) mode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--parity-steps", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=1000,
                    help="steps of the end-to-end run (load from host, K x step(), state to host); "
                         "1000 = the reference run length of config C1")
    ap.add_argument("--dry-run", action="store_true")
    args = ap.parse_args()
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("bench: --steps >= 1 and --warmup >= 0")
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    from paper_1309_1230_b200 import ExecutorKind

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    args.gpus = world
    dist = None
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    sc, bpc = scenario_for(args.config, world)
    spec = sc.spec

    comm_id = []

    def new_id():
        # one NCCL unique id per process group: every Stepper of this rank shares
        # one communicator (the library caches it by id)
        if world == 1:
            return None
        if not comm_id:
            from paper_1309_1230_b200 import abi
            import ctypes as C
            buf = C.create_string_buffer(abi.SWE_NCCL_ID_BYTES)
            if rank == 0:
                st = abi.swe_status()
                abi.load_library().swe_cuda_nccl_unique_id(buf, C.byref(st))
            obj = [bytes(buf.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            comm_id.append(obj[0])
        return comm_id[0]

    head_exact = bool(args.exact)
    early = args.config == "c5"  # wet/dry early-exit tiles (SWE_EXEC_EARLY_EXIT)
    clk = ClockSampler(local)
    kind = ExecutorKind(exact=head_exact, device=local, rank=rank, nranks=world, early_exit=early)
    dev_s, launches, cells_local, skipped = timed_run(sc, kind, new_id(), args, dist, local, clk)
    total_cells = spec.cell_count()
    value = total_cells * args.steps / dev_s
    ms = dev_s / args.steps * 1e3
    peak, peak_src = load_peaks()

    other = None
    if not args.fast and not args.exact:  # also report the other arithmetic mode
        k2 = ExecutorKind(exact=not head_exact, device=local, rank=rank, nranks=world, early_exit=early)
        d2, _, _, _ = timed_run(sc, k2, new_id(), args, dist, local)
        other = {"mode": EXACT_MODE if not head_exact else "fast",
                 "value": total_cells * args.steps / d2, "ms_per_step": d2 / args.steps * 1e3,
                 "roofline_frac": round(bpc * cells_local / (d2 / args.steps) / 1e9 / peak, 4)}

    # e2e moves the whole state through pinned host memory: skipped when one
    # rank would hold more than a 16384^2 strip (32768^2 on one GPU: 60 GB pinned)
    e2e = None
    if spec.cell_count() // world <= 16384 * 16384:
        ke = ExecutorKind(exact=head_exact, device=local, rank=rank, nranks=world, early_exit=early)
        e2e = e2e_run(sc, ke, args.e2e_steps, new_id(), dist, local)
        # the same through the device-resident loop (no per-step host round trip)
        e2e["advance_api"] = e2e_run(sc, ke, args.e2e_steps, new_id(), dist, local, api="advance")

    strong = None
    if world > 1:
        try:
            strong = strong_scaling_c4(args, world, rank, local, dist, new_id, peak)
        except Exception as e:  # the strong-scaling block must not cost the main line
            strong = {"error": str(e)}

    achieved = bpc * cells_local / (ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(args.config + ("_exact" if head_exact else "_fast"))
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
            "bytes_per_cell": bpc, "kernel": "swe_step_kernel (fused K1-K6, one launch per step)",
            "achieved_definition": f"{bpc} B/cell-step x {cells_local} cells per launch / mean launch time "
                                   "(device events over the timed region)"}
    activity = None
    if early:
        # roofline of the cells the kernels actually computed; the effective rate
        # (every interior cell counted, skipped ones included) is `value`
        active = 1.0 - skipped / float(cells_local * args.steps)
        roof["frac"] = round(achieved * active / peak, 4)
        roof["achieved"] = round(achieved * active, 1)
        roof["achieved_definition"] += " x active-cell fraction (skipped early-exit items are not counted)"
        roof["effective_frac_all_cells"] = round(achieved / peak, 4)
        activity = {"early_exit": True, "active_fraction": round(active, 5), "skipped_cells": skipped,
                    "active_cell_steps_per_s": value * active}

    cpu = par = None
    if world == 1 and rank == 0:
        if not args.no_parity:
            try:
                par = parity_run(sc, head_exact, args.parity_steps, local)
            except Exception as e:  # the parity leg must never kill the GPU bench
                par = {"error": str(e)}
        if not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline_sample(sc, args.config, steps=10)
            except Exception as e:
                cpu = {"value": None, "error": str(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "cell-steps/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_dict(args.config, spec, world, head_exact, early),
                "other_mode": other, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "parity": par,
                "gpu_launches": launches, "clocks": clk.summary()}
        if strong:
            line["strong_scaling"] = strong
        if activity:
            line["activity"] = activity
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
