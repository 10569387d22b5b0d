"""The C++ CLI's config front end on the CPU: the reference's grammar
(io.hpp:363-486) and error contract (ConfigError -> exit 2, with the line
number), checked before any device work starts."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1309_1230_b200", "bin", "swe_cuda")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="swe_cuda not built (__graft_entry__.build)")


def run(tmp_path, text, *args):
    cfg = tmp_path / "c.cfg"
    cfg.write_text(text)
    return subprocess.run([CLI, "run", "--config", str(cfg), "--out", str(tmp_path / "o"), *args],
                          capture_output=True, text=True, timeout=60)


@pytest.mark.parametrize("text,needle", [
    ("[grid]\nnx = 40\n[bogus]\n", "config line 3: unknown section 'bogus'"),
    ("nx = 40\n", "config line 1: key 'nx' outside any section"),
    ("[grid]\nnx = forty\n", "config line 2: expected an integer"),
    ("[physics]\nnu_art = 0.5\n", "config line 2: nu_art must lie in [0, 0.5)"),
    ("[policy]\ncfl = 1.5\n", "config line 2: cfl must lie in (0, 1]"),
    ("[boundaries]\nnorth = inflow 0.1\n", "config line 2: wrong parameter count"),
    ("[executor]\nkind = gpu\n", "config line 2: unknown executor kind 'gpu'"),
    ("[initial]\nkind = tsunami\n", "config line 2: unknown initial kind 'tsunami'"),
    ("[grid]\nnx = 2\n", "GridSpec: nx and ny must be at least 3"),
    ("[grid\n", "config line 1: malformed section header"),
])
def test_config_errors_exit_2_with_line(tmp_path, text, needle):
    r = run(tmp_path, text)
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert "error [config]" in r.stderr and needle in r.stderr, r.stderr


def test_bad_executor_flag_and_set_syntax(tmp_path):
    r = run(tmp_path, "[grid]\nnx = 40\n", "--executor", "cuda:fastest")
    assert r.returncode == 2 and "bad cuda option" in r.stderr
    r = run(tmp_path, "[grid]\nnx = 40\n", "--set", "gridnx=4")
    assert r.returncode == 2 and "--set expects section.key=value" in r.stderr


def test_missing_config_is_io_error(tmp_path):
    r = subprocess.run([CLI, "run", "--config", str(tmp_path / "nope.cfg")], capture_output=True, text=True,
                       timeout=60)
    assert r.returncode == 5 and "error [io]" in r.stderr
