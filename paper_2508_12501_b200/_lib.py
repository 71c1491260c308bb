"""ctypes binding of libdecmg_gpu.so (the C ABI in include/decmg_gpu.h).

The product has exactly one implementation: the sm_100a CUDA library. There
is no CPU fallback -- if the library is missing or no CUDA device is present,
every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("DECMG_GPU_LIB", PKG_DIR / "libdecmg_gpu.so"))

DECMG_OK = 0
DECMG_INVALID_ARGUMENT = 1
DECMG_RUNTIME = 2
DECMG_CUDA = 3
DECMG_NCCL = 4
DECMG_OOM = 5

DECMG_PROJECT_SPHERE = 1
DECMG_DIRICHLET = 2
DECMG_CUBIC = 4
DECMG_CLAMP_DUAL_AREAS = 8


class DecmgError(RuntimeError):
    """Base class of errors raised through the C ABI."""


class CudaError(DecmgError):
    pass


class decmg_gpu_config(C.Structure):
    _fields_ = [("device", C.c_int), ("max_nrhs", C.c_int)]


class decmg_gpu_plan(C.Structure):
    _fields_ = [("walk", C.c_char_p), ("pre", C.POINTER(C.c_int)), ("post", C.POINTER(C.c_int)),
                ("pre_all", C.c_int), ("post_all", C.c_int), ("smoother", C.c_int),
                ("jacobi_omega", C.c_double)]


class decmg_gpu_dist_transport(C.Structure):
    _fields_ = [("kind", C.c_int), ("nccl_id", C.c_void_p), ("shm_path", C.c_char_p)]


DECMG_DIST_EMULATE = 0
DECMG_DIST_NCCL = 1
DECMG_DIST_SHM = 2


class decmg_gpu_level_desc(C.Structure):
    _fields_ = [("nv", C.c_int),
                ("L_row_ptr", C.c_void_p), ("L_col_idx", C.c_void_p), ("L_values", C.c_void_p),
                ("L_nnz", C.c_int64), ("dual_areas", C.c_void_p), ("boundary", C.c_void_p),
                ("P_row_ptr", C.c_void_p), ("P_col_idx", C.c_void_p), ("P_values", C.c_void_p),
                ("P_nnz", C.c_int64),
                ("R_row_ptr", C.c_void_p), ("R_col_idx", C.c_void_p), ("R_values", C.c_void_p),
                ("R_nnz", C.c_int64)]


# name -> (restype, argtypes); the list is also the set of exported symbols
# tests/test_cabi.py checks against include/decmg_gpu.h.
SIGNATURES = {
    "decmg_gpu_create_from_base": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_uint,
                                             C.POINTER(decmg_gpu_config), C.POINTER(C.c_void_p)]),
    "decmg_gpu_create_from_base_ex": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                C.c_uint, C.POINTER(decmg_gpu_config), C.POINTER(C.c_void_p)]),
    "decmg_gpu_create_from_levels": (C.c_int, [C.POINTER(decmg_gpu_level_desc), C.c_int, C.c_uint,
                                               C.POINTER(decmg_gpu_config), C.POINTER(C.c_void_p)]),
    "decmg_gpu_destroy": (None, [C.c_void_p]),
    "decmg_gpu_last_error": (C.c_char_p, [C.c_void_p]),
    "decmg_gpu_run_cycles": (C.c_int, [C.c_void_p, C.POINTER(decmg_gpu_plan), C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_int, C.c_void_p, C.c_void_p]),
    "decmg_gpu_solve": (C.c_int, [C.c_void_p, C.POINTER(decmg_gpu_plan), C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "decmg_gpu_solve_batches": (C.c_int, [C.c_void_p, C.POINTER(decmg_gpu_plan), C.c_int, C.c_int, C.c_void_p, C.c_double, C.c_int,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "decmg_gpu_pcg": (C.c_int, [C.c_void_p, C.POINTER(decmg_gpu_plan), C.c_int, C.c_int, C.c_void_p, C.c_double,
                                C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "decmg_gpu_run_cycles_dev": (C.c_int, [C.c_void_p, C.POINTER(decmg_gpu_plan), C.c_int, C.c_void_p,
                                           C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "decmg_gpu_stream": (C.c_void_p, [C.c_void_p]),
    "decmg_gpu_project_compatible": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "decmg_gpu_apply": (C.c_int, [C.c_void_p, C.c_int, C.c_char, C.c_void_p, C.c_void_p]),
    "decmg_gpu_levels": (C.c_int, [C.c_void_p]),
    "decmg_gpu_level_info": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int64)]),
    "decmg_gpu_export": (C.c_int64, [C.c_void_p, C.c_int, C.c_char_p, C.c_void_p]),
    "decmg_gpu_mesh_hash": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64)]),
    "decmg_gpu_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "decmg_gpu_get_timing": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "decmg_gpu_launch_count": (C.c_int64, [C.c_void_p]),
    "decmg_gpu_projection_fallbacks": (C.c_int64, [C.c_void_p]),
    "decmg_base_mesh": (C.c_int, [C.c_char_p, C.c_void_p, C.POINTER(C.c_int), C.c_void_p, C.POINTER(C.c_int)]),
    "decmg_io_last_error": (C.c_char_p, []),
    "decmg_read_obj": (C.c_int, [C.c_char_p, C.c_void_p, C.POINTER(C.c_int), C.c_void_p, C.POINTER(C.c_int)]),
    "decmg_gpu_write_obj": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p]),
    "decmg_gpu_write_matrix_market": (C.c_int, [C.c_void_p, C.c_int, C.c_char, C.c_char_p]),
    "decmg_gpu_make_rhs": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_int, C.c_void_p]),
    "decmg_gpu_smooth": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_int]),
    "decmg_gpu_last_times": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "decmg_gpu_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_int]),
    "decmg_gpu_dist_create": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_uint,
                                        C.POINTER(decmg_gpu_config), C.c_int, C.c_int, C.c_void_p, C.c_int,
                                        C.POINTER(C.c_void_p)]),
    "decmg_gpu_dist_create_ex": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_uint,
                                           C.POINTER(decmg_gpu_config), C.c_int, C.c_int,
                                           C.POINTER(decmg_gpu_dist_transport), C.c_int, C.POINTER(C.c_void_p)]),
    "decmg_gpu_dist_destroy": (None, [C.c_void_p]),
    "decmg_gpu_dist_last_error": (C.c_char_p, [C.c_void_p]),
    "decmg_gpu_dist_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]),
    "decmg_gpu_dist_context": (C.c_void_p, [C.c_void_p]),
    "decmg_gpu_dist_last_cycle_ms": (C.c_double, [C.c_void_p]),
    "decmg_gpu_dist_launch_count": (C.c_int64, [C.c_void_p]),
    "decmg_gpu_dist_run": (C.c_int, [C.c_void_p, C.POINTER(decmg_gpu_plan), C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
}

_lib = None


def load() -> C.CDLL:
    """Load libdecmg_gpu.so; raises (no fallback) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA library is the only implementation; there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_EXC = {DECMG_INVALID_ARGUMENT: ValueError, DECMG_RUNTIME: RuntimeError, DECMG_CUDA: CudaError,
        DECMG_NCCL: DecmgError, DECMG_OOM: MemoryError}


def check(rc: int, ctx=None, dist=False) -> None:
    if rc == DECMG_OK:
        return
    msg = (load().decmg_gpu_dist_last_error if dist else load().decmg_gpu_last_error)(ctx)
    msg = msg.decode() if msg else f"decmg_gpu error {rc}"
    raise _EXC.get(rc, DecmgError)(msg)
