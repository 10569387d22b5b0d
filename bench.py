#!/usr/bin/env python3
"""Throughput of the fused MacCormack step on B200 (cell-steps/s, % of HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c3f|c1|c2|c4|c5]

N=1 runs BASELINE.json's headline workload: the 8192^2 synthetic channel flood
(gen_channel_flood(8192), scenarios.hpp:237-256; Manning 0.035, inflow west,
fixed elevation east, walls N/S).  N>1 (torchrun, one rank per GPU) runs the
same channel with 8192 rows per GPU as NCCL-exchanged row strips (weak
scaling).  One JSON line is printed by rank 0.

--impl reference times the unmodified reference solver (oracle/_ref: the
reference headers compiled in place, decomposed:<host cores> executor) on the
same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

EXACT_MODE = ("exact (-fmad=false IEEE expression trees: bit-identical to the reference without Manning "
              "friction; within 1e-12 with it, std::pow not being reproducible on CUDA)")

CONFIGS = {
    # name: (description, builder)
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
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def scenario_for(cfg: str, nranks: int):
    from paper_1309_1230_b200 import scenarios as S
    if cfg in ("c3", "c3f"):
        sc = S.gen_channel_flood(8192, manning_n=0.035 if cfg == "c3" else 0.0)
        if nranks > 1:  # weak scaling: 8192 rows per GPU, same physics per strip
            from paper_1309_1230_b200.stepper import GridSpec
            sc.spec = GridSpec(8192, 8192 * nranks, 1.0, 1.0)
        return sc, 56  # algorithmic bytes/cell-step: read h,qx,qy,z + write h,qx,qy (fp64)
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


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_baseline_sample(sc, cfg, steps=2):
    """Time the reference itself (oracle/_ref, decomposed:<cores>) on a bounded sample.
    Grids above 8192^2 are sampled on the same scenario at 8192^2 (per-cell rate):
    the reference needs ~192 B/cell of host memory."""
    from oracle import oracle as O
    if sc.spec.cell_count() > 8192 * 8192:
        from paper_1309_1230_b200 import scenarios as S
        sc = S.gen_floodplain(8192) if cfg == "c5" else S.gen_square_dam(8192)
    cores = os.cpu_count() or 1
    if O.ref_available():
        kind = "reference"
        mk = lambda: O.RefStepper(sc.spec, sc.phys, sc.pol, sc.bounds, O.REF_DECOMPOSED, cores)  # noqa: E731
    else:
        kind, cores = "port", 1
        mk = lambda: O.OracleStepper(sc.spec, sc.phys, sc.pol, sc.bounds)  # noqa: E731
    fs = sc.build()
    st = mk()
    st.load(fs)
    dt = st.compute_dt(math.inf)
    dt = st.step(dt, 0).dt_next  # warm-up
    t0 = time.perf_counter()
    for k in range(1, steps + 1):
        dt = st.step(dt, k).dt_next
    el = time.perf_counter() - t0
    cells = sc.spec.cell_count()
    return {"value": cells * steps / el, "unit": "cell-steps/s", "cores": cores, "kind": kind,
            "sample": f"{sc.spec.nx}x{sc.spec.ny} {cfg}, {steps} timed steps after 1 warm-up, "
                      f"{'decomposed:%d' % cores if kind == 'reference' else 'naive C port'} executor",
            "seconds": el}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sc, bpc = scenario_for(args.config, 1)
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libswe_ref.so not built"}))
        return 0
    cores = os.cpu_count() or 1
    fs = sc.build()
    st = O.RefStepper(sc.spec, sc.phys, sc.pol, sc.bounds, O.REF_DECOMPOSED, cores)
    st.load(fs)
    dt = st.compute_dt(math.inf)
    k = 0
    # bounded: each step is ~1-3 s at 8192^2 on the host, so cap the sample
    warm = min(args.warmup, 1)
    steps = max(1, min(args.steps, int(os.environ.get("SWE_REF_MAX_STEPS", "10"))))
    for _ in range(warm):
        dt = st.step(dt, k).dt_next
        k += 1
    t0 = time.perf_counter()
    for _ in range(steps):
        dt = st.step(dt, k).dt_next
        k += 1
    el = time.perf_counter() - t0
    cells = sc.spec.cell_count()
    v = cells * steps / el
    line = {"metric": "cell-steps/sec (full 16-substep step) at 8192² and % of HBM roofline",
            "value": v, "unit": "cell-steps/s", "impl": "reference", "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": el / steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIGS[args.config], "grid": [sc.spec.nx, sc.spec.ny],
                       "executor": f"reference decomposed:{cores} (oracle/_ref, -O3 -ffp-contract=off)"},
            "cpu_baseline": {"value": v, "unit": "cell-steps/s", "cores": cores, "kind": "reference",
                             "sample": f"{steps} steps of the full {sc.spec.nx}x{sc.spec.ny} grid"},
            "e2e": {"value": v, "unit": "cell-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def timed_run(sc, kind, nccl_id, args, dist, local, sampler=None):
    """W untimed warm-up steps, then exactly K device-resident steps timed with
    CUDA events on the library's stream (max over ranks)."""
    import torch
    from paper_1309_1230_b200 import Stepper
    world = kind.nranks
    stp = Stepper(sc.spec, sc.phys, sc.pol, sc.bounds, kind, nccl_id=nccl_id)
    r0, r1 = stp.row_begin, stp.row_end
    if sc.initial is not None:  # generated on the device (swe_cuda_load_initial), bit-identical to the host build
        stp.load_initial(sc.initial)
    elif world == 1:
        stp.load(sc.build())
    else:
        fsr = sc.build_rows(r0, r1)
        stp.load_rows(fsr.z, fsr.h, fsr.qx, fsr.qy, 0.0)
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
        res = stp.advance(1e18, step0, dt_next, args.steps)
    finally:
        if sampler:
            sampler.__exit__()
    torch.cuda.synchronize()
    act = stp.activity()
    skipped = act["skipped_cells"] - a0
    n1, s1 = stp.timing()
    launches = stp.launch_count() - l0
    dev_s = s1 - s0
    if res.steps != args.steps:
        raise SystemExit(f"bench: only {res.steps} of {args.steps} steps committed")
    if dist:
        t = torch.tensor([dev_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
        dist.barrier()
    stp.close()
    timed_run.skipped_cells = skipped
    return dev_s, launches, (r1 - r0) * sc.spec.nx


def e2e_run(sc, kind, steps, nccl_id=None, dist=None, local=0):
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
    ctl = 2 * 200 * kind.nranks  # control block H2D + D2H per step() call and rank
    return {"value": cells * steps / el, "unit": "cell-steps/s",
            "h2d_bytes_per_step": (4 * cells * 8) // steps + ctl, "d2h_bytes_per_step": (3 * cells * 8) // steps + ctl,
            "steps": steps, "seconds": el, "phases": phases,
            "api": "Stepper.load(host, pinned) + K x Stepper.step() (dt_next read back each step) + "
                   "Stepper.state() (host); C-ABI swe_cuda_load/step/state" +
                   ("; every rank moves its own strip, max over ranks" if kind.nranks > 1 else "")}


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
    ap.add_argument("--e2e-steps", type=int, default=1000,
                    help="steps of the end-to-end run (load from host, K x step(), state to host); "
                         "1000 = the reference run length of config C1")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    from paper_1309_1230_b200 import ExecutorKind

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    args.gpus = world
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    sc, bpc = scenario_for(args.config, world)
    spec = sc.spec

    def new_id():
        if world == 1:
            return None
        from paper_1309_1230_b200 import abi
        import ctypes as C
        buf = C.create_string_buffer(abi.SWE_NCCL_ID_BYTES)
        if rank == 0:
            st = abi.swe_status()
            abi.load_library().swe_cuda_nccl_unique_id(buf, C.byref(st))
        obj = [bytes(buf.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    head_exact = bool(args.exact)
    clk = ClockSampler(local)
    early = args.config == "c5"  # wet/dry early-exit tiles (SWE_EXEC_EARLY_EXIT)
    kind = ExecutorKind(exact=head_exact, device=local, rank=rank, nranks=world, early_exit=early)
    dev_s, launches, cells_local = timed_run(sc, kind, new_id(), args, dist, local, clk)
    skipped = timed_run.skipped_cells
    total_cells = spec.cell_count()
    value = total_cells * args.steps / dev_s
    ms = dev_s / args.steps * 1e3

    other = None
    if not args.fast and not args.exact:  # also report the other arithmetic mode
        k2 = ExecutorKind(exact=not head_exact, device=local, rank=rank, nranks=world, early_exit=early)
        d2, l2, _ = timed_run(sc, k2, new_id(), args, dist, local)
        other = {"mode": EXACT_MODE if not head_exact else "fast",
                 "value": total_cells * args.steps / d2, "ms_per_step": d2 / args.steps * 1e3,
                 "roofline_frac": round(bpc * cells_local / (d2 / args.steps) / 1e9 / load_peaks()[0], 4)}

    # e2e moves the whole state through pinned host memory: skipped when one
    # rank would hold more than a 16384^2 strip (32768^2 on one GPU: 60 GB pinned)
    e2e = None
    if spec.cell_count() // world <= 16384 * 16384:
        ke = ExecutorKind(exact=head_exact, device=local, rank=rank, nranks=world, early_exit=early)
        e2e = e2e_run(sc, ke, args.e2e_steps, new_id(), dist, local)

    peak, peak_src = load_peaks()
    achieved = bpc * cells_local / (ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get(args.config + ("_exact" if head_exact else "_fast"))
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
            "bytes_per_cell": bpc, "kernel": "swe_step_kernel (fused K1-K6, one launch per step)",
            "achieved_definition": f"{bpc} B/cell-step x {cells_local} cells per launch / mean launch time"}
    activity = None
    if early:
        active = 1.0 - skipped / float(cells_local * args.steps)
        activity = {"early_exit": True, "active_fraction": round(active, 5),
                    "skipped_cells": skipped,
                    "active_cell_steps_per_s": value * active,
                    "active_roofline_frac": round(achieved * active / peak, 4),
                    "note": "value/roofline count every interior cell (effective); the active_* figures "
                            "count only computed (non-skipped) cells"}

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(sc, args.config, steps=10)
        except Exception as e:  # the baseline must never kill the GPU bench
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        line = {"metric": "cell-steps/sec (full 16-substep step) at 8192² and % of HBM roofline",
                "value": value, "unit": "cell-steps/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": CONFIGS[args.config], "grid": [spec.nx, spec.ny],
                           "rows_per_gpu": cells_local // spec.nx, "parallelism": f"row-strips{world}",
                           "mode": EXACT_MODE if head_exact else
                           "fast (FMA + shared reciprocals; max |dh|,|du|,|dv| <= 1e-10 vs reference, "
                           "measured ~1e-14)",
                           "l2": "inputs (2 x 24 B/cell state + 16 B/cell slopes) >> 126 MB L2; no flush needed",
                           "timing": "CUDA events on the library stream around device-resident advance() "
                                     "(CUDA graphs of 64 steps), max over ranks"},
                "other_mode": other, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary()}
        if activity:
            line["activity"] = activity
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
