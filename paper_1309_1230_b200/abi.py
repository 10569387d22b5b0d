"""ctypes mirror of include/swe_cuda.h and the loader for libswe_cuda.so.

The loader fails loudly: there is no CPU fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWE_CUDA_LIB") or os.path.join(HERE, "lib", "libswe_cuda.so")

SWE_OK = 0
SWE_ERR_CONFIG = 2
SWE_ERR_INSTABILITY = 3
SWE_ERR_STEP_COLLAPSE = 4
SWE_ERR_IO = 5
SWE_ERR_RUNTIME = 6

SWE_BC_WALL = 0
SWE_BC_TRANSMISSIVE = 1
SWE_BC_INFLOW = 2
SWE_BC_FIXED_ETA = 3

SWE_EXEC_EXACT = 1 << 0
SWE_EXEC_NO_GRAPH = 1 << 1
SWE_EXEC_EARLY_EXIT = 1 << 2
SWE_EXEC_LOCAL_GROUP = 1 << 3

SWE_NCCL_ID_BYTES = 128


class swe_status(C.Structure):
    _fields_ = [("code", C.c_int32), ("i", C.c_int32), ("j", C.c_int32), ("t", C.c_double),
                ("dt", C.c_double), ("h", C.c_double), ("qx", C.c_double), ("qy", C.c_double),
                ("msg", C.c_char * 256)]


class swe_grid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("dx", C.c_double), ("dy", C.c_double)]


class swe_physics(C.Structure):
    _fields_ = [("g", C.c_double), ("manning_n", C.c_double), ("nu_art", C.c_double)]


class swe_policy(C.Structure):
    _fields_ = [("cfl", C.c_double), ("dt_max", C.c_double), ("dt_min", C.c_double),
                ("h_min", C.c_double)]


class swe_boundary(C.Structure):
    _fields_ = [("type", C.c_int32), ("q_n", C.c_double), ("h_in", C.c_double),
                ("eta_out", C.c_double)]


class swe_boundary_set(C.Structure):
    _fields_ = [("north", swe_boundary), ("south", swe_boundary), ("east", swe_boundary),
                ("west", swe_boundary)]


class swe_exec(C.Structure):
    _fields_ = [("device", C.c_int32), ("flags", C.c_uint32), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("nccl_id", C.c_void_p)]


class swe_step_result(C.Structure):
    _fields_ = [("dt_used", C.c_double), ("dt_next", C.c_double), ("guard_warnings", C.c_int32)]


SWE_IC_FLAT_POOL = 0
SWE_IC_CHANNEL_SLOPE = 2
SWE_IC_DAM_BREAK = 4


class swe_initial(C.Structure):
    _fields_ = [("kind", C.c_int32), ("depth", C.c_double), ("slope", C.c_double), ("split_x", C.c_double),
                ("h_left", C.c_double), ("h_right", C.c_double)]


class swe_run_result(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("step_index", C.c_uint64), ("t_final", C.c_double),
                ("dt_next", C.c_double), ("guard_warnings", C.c_int32)]


class swe_activity(C.Structure):
    _fields_ = [("cells_per_step", C.c_uint64), ("items_per_step", C.c_uint64),
                ("eligible_items", C.c_uint64), ("skipped_cells", C.c_uint64)]


class swe_accounting(C.Structure):
    _fields_ = [("halo_values_exchanged", C.c_int64), ("redundant_star_rows", C.c_int32),
                ("redundant_corrector_rows", C.c_int32)]


class swe_timing(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("step_seconds", C.c_double), ("exchange_steps", C.c_uint64),
                ("exchange_seconds", C.c_double), ("allreduce_seconds", C.c_double)]


DP = C.POINTER(C.c_double)
ST = C.POINTER(swe_status)

# name -> (restype, argtypes); exactly the symbols include/swe_cuda.h declares
SIGNATURES = {
    "swe_cuda_create": (C.c_int, [C.POINTER(swe_grid), C.POINTER(swe_physics), C.POINTER(swe_policy),
                                  C.POINTER(swe_boundary_set), C.POINTER(swe_exec),
                                  C.POINTER(C.c_void_p), ST]),
    "swe_cuda_destroy": (None, [C.c_void_p]),
    "swe_cuda_load": (C.c_int, [C.c_void_p, DP, DP, DP, DP, C.c_double, ST]),
    "swe_cuda_load_initial": (C.c_int, [C.c_void_p, C.POINTER(swe_initial), C.c_double, ST]),
    "swe_cuda_state": (C.c_int, [C.c_void_p, DP, DP, DP, DP, DP, ST]),
    "swe_cuda_step": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64, C.c_double,
                                C.POINTER(swe_step_result), ST]),
    "swe_cuda_compute_dt": (C.c_int, [C.c_void_p, C.c_double, DP, ST]),
    "swe_cuda_guard": (C.c_int, [C.c_void_p, ST]),
    "swe_cuda_advance": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64, C.c_double, C.c_uint64,
                                   C.POINTER(swe_run_result), ST]),
    "swe_cuda_advance_marked": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_uint64, C.c_double, C.c_uint64,
                                          C.POINTER(swe_run_result), ST]),
    "swe_cuda_time": (C.c_double, [C.c_void_p]),
    "swe_cuda_guard_warnings": (C.c_int32, [C.c_void_p]),
    "swe_cuda_timing": (C.c_int, [C.c_void_p, C.POINTER(swe_timing)]),
    "swe_cuda_accounting": (C.c_int, [C.c_void_p, C.POINTER(swe_accounting)]),
    "swe_cuda_activity": (C.c_int, [C.c_void_p, C.POINTER(swe_activity)]),
    "swe_cuda_rows": (None, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "swe_cuda_halo_rows": (C.c_int32, [C.c_void_p]),
    "swe_cuda_state_digest": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(swe_status)]),
    "swe_cuda_debug_guard_check": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(swe_status)]),
    "swe_cuda_nccl_unique_id": (C.c_int, [C.c_void_p, ST]),
    "swe_cuda_strip_rows": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      ST]),
    "swe_cuda_version": (C.c_char_p, []),
    "swe_cuda_launch_count": (C.c_uint64, [C.c_void_p]),
    "swe_cuda_selftest_div": (C.c_int, [DP, DP, C.c_size_t, C.c_int, DP, ST]),
}

_lib = None


def load_library(path: str | None = None) -> C.CDLL:
    """Load libswe_cuda.so (built in-tree by __graft_entry__.build()).

    Raises RuntimeError when the library is missing: the product path has no
    CPU fallback.
    """
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"libswe_cuda.so not built at {p}; run __graft_entry__.build()")
    lib = C.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("SWE_ABI_LENIENT") and not hasattr(lib, name):
            continue  # tools/ A/B runs against older library builds
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(DP)
