"""The C++ command-line driver (paper_1309_1230_b200/bin/swe_cuda) against the
reference's own `run` (parse_config + run, run.hpp:101-179; oracle/_ref):
the same config text must produce byte-identical SWS1 snapshots (with the
dt_next / step_index resume trailers) at every snapshot mark, in exact mode.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1309_1230_b200 import io as sio

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1309_1230_b200", "bin", "swe_cuda")

FIVE_DROPS_64 = """
[grid]
nx = 64
ny = 64
[policy]
cfl = 0.45
[executor]
kind = naive
[initial]
kind = drops
depth = 1
drop = 31.5 31.5 3.2 0.3
drop = 15.5 15.5 3.2 0.3
drop = 47.5 20 3.2 0.3
[run]
name = drops64
t_end = 9
snapshot_every = 2.5
"""

CHANNEL_72x50 = """
[grid]
nx = 72
ny = 50
[policy]
cfl = 0.45
[boundaries]
north = wall
south = wall
east = fixed_eta 1
west = inflow 0.1 1
[initial]
kind = channel_slope
depth = 1
slope = 0.007
[run]
name = channel
t_end = 14
snapshot_every = 4
"""

DAM_CHANNEL = """
[grid]
nx = 200
ny = 3
[physics]
nu_art = 0.05
[policy]
cfl = 0.45
[boundaries]
north = transmissive
south = transmissive
east = wall
west = wall
[initial]
kind = dam_break
split_x = 100
h_left = 1
h_right = 0.5
[run]
name = dam
t_end = 15.96
"""

CASES = {"drops64": FIVE_DROPS_64, "channel": CHANNEL_72x50, "dam": DAM_CHANNEL}


def run_ref(text, out):
    return O.ref_run_config(text, out)


def run_cli(text, out, tmp_path, *extra):
    cfg = tmp_path / "case.cfg"
    cfg.write_text(text)
    return subprocess.run([CLI, "run", "--config", str(cfg), "--out", str(out), *extra],
                          capture_output=True, text=True, timeout=300)


def sws_files(d):
    return sorted(f for f in os.listdir(d) if f.endswith(".sws"))


@pytest.mark.parametrize("name", sorted(CASES))
def test_cli_run_matches_reference_run_bytes(name, tmp_path):
    text = CASES[name]
    ref, got = tmp_path / "ref", tmp_path / "got"
    assert run_ref(text, str(ref)) == 0
    r = run_cli(text, got, tmp_path)
    assert r.returncode == 0, r.stderr
    assert sws_files(ref) == sws_files(got) and len(sws_files(got)) >= 1
    for f in sws_files(ref):
        assert (ref / f).read_bytes() == (got / f).read_bytes(), f
    rep_ref = dict(l.split(": ", 1) for l in (ref / f"{name}_report.txt").read_text().splitlines() if ": " in l)
    rep_got = dict(l.split(": ", 1) for l in (got / f"{name}_report.txt").read_text().splitlines() if ": " in l)
    for k in ("scenario", "cells", "steps", "t_final", "snapshots_written"):
        assert rep_ref[k] == rep_got[k], k
    assert rep_got["executor"] == "cuda"
    assert "final_snapshot:" in r.stdout


def test_cli_strips_local_group_bytes_equal_single(tmp_path):
    a, b = tmp_path / "one", tmp_path / "three"
    assert run_cli(CHANNEL_72x50, a, tmp_path).returncode == 0
    r = run_cli(CHANNEL_72x50, b, tmp_path, "--executor", "cuda:3:local")
    assert r.returncode == 0, r.stderr
    assert sws_files(a) == sws_files(b)
    for f in sws_files(a):
        assert (a / f).read_bytes() == (b / f).read_bytes(), f


def test_cli_fast_mode_within_tolerance(tmp_path):
    a, b = tmp_path / "exact", tmp_path / "fast"
    assert run_cli(FIVE_DROPS_64, a, tmp_path).returncode == 0
    r = run_cli(FIVE_DROPS_64, b, tmp_path, "--executor", "cuda:fast", "--snapshot-every", "0")
    assert r.returncode == 0, r.stderr
    fa, _, ea = sio.parse_snapshot((a / "drops64_final.sws").read_bytes())
    fb, _, eb = sio.parse_snapshot((b / "drops64_final.sws").read_bytes())
    assert ea["step_index"] == eb["step_index"]
    assert np.abs(fa.h - fb.h).max() <= 1e-12 and np.abs(fa.qx - fb.qx).max() <= 1e-12


def test_cli_set_override_and_error_exit_codes(tmp_path):
    # thin film without smoothing collapses: exit code 3 like the reference's
    bad = DAM_CHANNEL.replace("h_right = 0.5", "h_right = 0.001").replace("nu_art = 0.05", "nu_art = 0")
    ref = tmp_path / "ref"
    assert run_ref(bad, str(ref)) == 3
    r = run_cli(bad, tmp_path / "got", tmp_path)
    assert r.returncode == 3 and "error [instability]" in r.stderr
    # --set goes through the parser: an out-of-range value is a config error (2)
    r = run_cli(DAM_CHANNEL, tmp_path / "x", tmp_path, "--set", "physics.nu_art=0.7")
    assert r.returncode == 2 and "nu_art" in r.stderr
    r = run_cli(DAM_CHANNEL, tmp_path / "y", tmp_path, "--set", "run.t_end=1")
    assert r.returncode == 0
    rep = (tmp_path / "y" / "dam_report.txt").read_text()
    assert "t_final: 1\n" in rep


def test_cli_bench_writes_csv(tmp_path):
    csv = tmp_path / "b.csv"
    r = subprocess.run([CLI, "bench", "--sizes", "64,96", "--steps", "5", "--reps", "2", "--executors",
                        "cuda,cuda:fast", "--csv", str(csv)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = csv.read_text().splitlines()
    assert rows[0] == "size,executor,steps,reps,median_sec_per_step,cells_per_second"
    assert [l.split(",")[:2] for l in rows[1:]] == [["64", "cuda"], ["64", "cuda:fast"], ["96", "cuda"],
                                                    ["96", "cuda:fast"]]


DROPS48_CKPT = """
[grid]
nx = 48
ny = 48
[policy]
cfl = 0.45
[initial]
kind = drops
depth = 1
drop = 23.5 23.5 2.4 0.3
drop = 11.5 11.5 2.4 0.3
drop = 35.5 11.5 2.4 0.3
[run]
name = ckpt
t_end = 6
snapshot_every = 2
"""


@pytest.mark.parametrize("text,which", [(DROPS48_CKPT, 0),
                                        (DAM_CHANNEL.replace("t_end = 15.96", "t_end = 15.96\nsnapshot_every = 3.99"),
                                         1)])
def test_cli_checkpoint_resume_is_bit_exact(text, which, tmp_path):
    """test_io.cpp:268-315: resuming from an intermediate snapshot (its dt_next
    and step_index records) reproduces the unsplit run's final state bytes."""
    full, res = tmp_path / "full", tmp_path / "resumed"
    r = run_cli(text, full, tmp_path)
    assert r.returncode == 0, r.stderr
    mids = [f for f in sws_files(full) if not f.endswith("_final.sws")]
    assert len(mids) > which
    r = run_cli(text, res, tmp_path, "--resume", str(full / mids[which]))
    assert r.returncode == 0, r.stderr
    name = [f for f in sws_files(full) if f.endswith("_final.sws")][0]
    assert (full / name).read_bytes() == (res / name).read_bytes()
    steps = lambda d: int(dict(l.split(": ", 1) for l in (d / name.replace("_final.sws", "_report.txt"))
                               .read_text().splitlines() if ": " in l)["steps"])
    _, _, ex = sio.parse_snapshot((full / mids[which]).read_bytes())
    assert steps(full) == ex["step_index"] + steps(res)
