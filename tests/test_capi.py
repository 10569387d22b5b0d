"""The drop-in boundary: libswe_cuda.so loads without a GPU and exports every
entry point include/swe_cuda.h declares (and the ctypes mirror binds exactly
those).  No compute calls here."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1309_1230_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "swe_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(swe_cuda_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = abi.load_library()
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (swe_cuda_\w+)", out))
    assert set(names) <= exported
    # nothing else with the public prefix leaks out
    assert exported == set(names)


def test_ctypes_mirror_binds_exactly_the_header():
    assert sorted(abi.SIGNATURES) == declared_symbols()


def test_struct_layouts_match_header():
    # sizes computed by the C compiler from include/swe_cuda.h
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "swe_cuda.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(swe_status), sizeof(swe_grid),
 sizeof(swe_physics), sizeof(swe_policy), sizeof(swe_boundary), sizeof(swe_boundary_set), sizeof(swe_exec),
 sizeof(swe_step_result), sizeof(swe_run_result), offsetof(swe_status, msg));return 0;}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(abi.swe_status), C.sizeof(abi.swe_grid), C.sizeof(abi.swe_physics), C.sizeof(abi.swe_policy),
            C.sizeof(abi.swe_boundary), C.sizeof(abi.swe_boundary_set), C.sizeof(abi.swe_exec),
            C.sizeof(abi.swe_step_result), C.sizeof(abi.swe_run_result), abi.swe_status.msg.offset]
    assert got == want


def test_version_string():
    lib = abi.load_library()
    assert b"sm_100a" in lib.swe_cuda_version()


def test_create_validates_like_the_reference_without_a_gpu():
    # validation (scheme.hpp:22-32, timestep.hpp:26-39, grid.hpp:28-37) precedes any device call
    lib = abi.load_library()
    st = abi.swe_status()
    ctx = C.c_void_p()
    bad_grid = abi.swe_grid(2, 5, 1.0, 1.0)
    p = abi.swe_physics(9.81, 0.0, 0.0)
    po = abi.swe_policy(0.45, float("inf"), 1e-9, 1e-6)
    b = abi.swe_boundary_set()
    ex = abi.swe_exec(0, abi.SWE_EXEC_EXACT, 0, 1, None)
    assert lib.swe_cuda_create(C.byref(bad_grid), C.byref(p), C.byref(po), C.byref(b), C.byref(ex), C.byref(ctx),
                               C.byref(st)) == abi.SWE_ERR_CONFIG
    assert b"at least 3" in st.msg
    g = abi.swe_grid(8, 8, 1.0, 1.0)
    bad_p = abi.swe_physics(9.81, 0.0, 0.5)  # nu_art must lie in [0, 0.5)
    assert lib.swe_cuda_create(C.byref(g), C.byref(bad_p), C.byref(po), C.byref(b), C.byref(ex), C.byref(ctx),
                               C.byref(st)) == abi.SWE_ERR_CONFIG
    bad_po = abi.swe_policy(1.5, float("inf"), 1e-9, 1e-6)
    assert lib.swe_cuda_create(C.byref(g), C.byref(p), C.byref(bad_po), C.byref(b), C.byref(ex), C.byref(ctx),
                               C.byref(st)) == abi.SWE_ERR_CONFIG
    inflow = abi.swe_boundary_set()
    inflow.west = abi.swe_boundary(abi.SWE_BC_INFLOW, 0.1, 0.0, 0.0)  # h_in < h_min
    assert lib.swe_cuda_create(C.byref(g), C.byref(p), C.byref(po), C.byref(inflow), C.byref(ex), C.byref(ctx),
                               C.byref(st)) == abi.SWE_ERR_CONFIG
    strips = abi.swe_exec(0, 0, 0, 4, None)  # 10 rows over 4 ranks leaves 2-row bands
    g10 = abi.swe_grid(16, 10, 1.0, 1.0)
    assert lib.swe_cuda_create(C.byref(g10), C.byref(p), C.byref(po), C.byref(b), C.byref(strips), C.byref(ctx),
                               C.byref(st)) == abi.SWE_ERR_CONFIG
    assert b"at least 4 rows" in st.msg


def test_strip_rows_match_partition_scanlines_and_create_errors():
    # host-only C-ABI entry (no GPU): the strips swe_cuda_create assigns
    from paper_1309_1230_b200.stepper import ConfigError, partition_scanlines, strip_rows
    for ny, n in [(10, 1), (10, 2), (17, 3), (8192, 8), (35, 4), (32768, 8)]:
        assert [strip_rows(ny, n, r) for r in range(n)] == partition_scanlines(ny, n)
    for args, msg in [((3, 4, 0), "need at least as many rows"), ((10, 3, 0), "at least 4 rows"),
                      ((10, 2, 2), "outside"), ((10, 0, 0), "workers must be >= 1")]:
        with pytest.raises(ConfigError, match=msg):
            strip_rows(*args)
