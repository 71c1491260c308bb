"""ctypes view of the CPU oracle (oracle/liboracle.so) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module. The oracle is the checker, never the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"
LIB_PATH = ORACLE_DIR / "liboracle.so"

_lib = None


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "oracle"], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        src = ORACLE_DIR / "decmg_oracle.c"
        if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
            build_oracle()
        L = C.CDLL(str(LIB_PATH))
        L.orc_build.restype = C.c_void_p
        L.orc_build.argtypes = [C.c_char_p, C.c_int, C.c_int]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_levels.argtypes = [C.c_void_p]
        L.orc_level_info.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        L.orc_get.restype = C.c_int64
        L.orc_get.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_void_p]
        L.orc_level_nnz.restype = C.c_int64
        L.orc_level_nnz.argtypes = [C.c_void_p, C.c_int, C.c_char_p]
        L.orc_rhs.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_void_p]
        L.orc_project.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_spmv.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_void_p, C.c_void_p]
        L.orc_norm2.restype = C.c_double
        L.orc_norm2.argtypes = [C.c_void_p, C.c_int64]
        L.orc_fnv.restype = C.c_uint64
        L.orc_fnv.argtypes = [C.c_void_p, C.c_int64]
        L.orc_run_cycles.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                     C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p,
                                C.c_double, C.c_int, C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.orc_coarse_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_smooth.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_pcg.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                              C.c_void_p, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def fnv(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().orc_fnv(_p(a), a.nbytes))


class OracleHierarchy:
    """Finest-first level hierarchy built by the oracle (build_hierarchy)."""

    def __init__(self, base: str, nsub: int, dirichlet: bool = False):
        self.h = lib().orc_build(base.encode(), nsub, int(dirichlet))
        if not self.h:
            raise RuntimeError(lib().orc_last_error().decode())
        self.dirichlet = dirichlet
        self.levels = lib().orc_levels(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_free(self.h)
            self.h = None

    def info(self, k: int):
        counts = (C.c_int64 * 4)()
        h = C.c_uint64()
        lib().orc_level_info(self.h, k, counts, C.byref(h))
        return dict(nv=counts[0], ne=counts[1], nt=counts[2], nnz=counts[3], hash=h.value)

    def n(self, k: int = 0) -> int:
        return self.info(k)["nv"]

    _DT = {"positions": np.float64, "dual_areas": np.float64, "L_v": np.float64,
           "P_v": np.float64, "R_v": np.float64}

    def get(self, k: int, name: str) -> np.ndarray:
        cnt = lib().orc_get(self.h, k, name.encode(), None)
        if cnt < 0:
            raise KeyError(name)
        out = np.empty(cnt, dtype=self._DT.get(name, np.int32))
        lib().orc_get(self.h, k, name.encode(), _p(out))
        return out

    def rhs(self, kind: str, seed: int) -> np.ndarray:
        b = np.empty(self.n(), dtype=np.float64)
        if lib().orc_rhs(self.h, kind.encode(), seed, _p(b)):
            raise RuntimeError(lib().orc_last_error().decode())
        return b

    def project(self, b: np.ndarray) -> np.ndarray:
        b = np.array(b, dtype=np.float64, copy=True)
        lib().orc_project(self.h, _p(b))
        return b

    def spmv(self, k: int, op: str, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if op == "R":
            ny = self.n(k + 1)
        else:
            ny = self.n(k)
        y = np.empty(ny, dtype=np.float64)
        lib().orc_spmv(self.h, k, op.encode(), _p(x), _p(y))
        return y

    def run_cycles(self, b, x0=None, ncycles=1, pre=2, post=2, smoother=0, omega=2.0 / 3.0, walk=None):
        n = self.n()
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        x = np.empty(n)
        hist = np.empty(max(ncycles, 1))
        rc = lib().orc_run_cycles(self.h, None if walk is None else walk.encode(), pre, post, smoother,
                                  omega, _p(b), _p(x0), ncycles, _p(x), _p(hist))
        if rc:
            raise RuntimeError(lib().orc_last_error().decode())
        return x, hist[:ncycles]

    def solve(self, b, tol=1e-8, max_cycles=200, pre=2, post=2, smoother=0, omega=2.0 / 3.0):
        n = self.n()
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(n)
        hist = np.empty(max(max_cycles, 1))
        it = C.c_int()
        fin = C.c_double()
        rc = lib().orc_solve(self.h, pre, post, smoother, omega, _p(b), tol, max_cycles, _p(x), _p(hist),
                             C.byref(it), C.byref(fin))
        if rc:
            raise RuntimeError(lib().orc_last_error().decode())
        return x, hist[: it.value], it.value, fin.value

    def pcg(self, b, tol, maxiter, walk=None, pre=2, post=2, smoother=0, omega=2.0 / 3.0, cycles=1):
        """gmg_preconditioned_cg (solvers.cpp:118-130): (x, history[iters+1], iters, final)."""
        n = self.n()
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(n)
        hist = np.empty(maxiter + 1)
        it = C.c_int()
        fin = C.c_double()
        rc = lib().orc_pcg(self.h, None if walk is None else walk.encode(), pre, post, smoother, omega, cycles,
                           _p(b), tol, maxiter, _p(x), _p(hist), C.byref(it), C.byref(fin))
        if rc:
            raise RuntimeError(lib().orc_last_error().decode())
        return x, hist[: it.value + 1], it.value, fin.value

    def smooth(self, k, b, x, iters, smoother=1, omega=2.0 / 3.0):
        """smooth (multigrid.cpp:95-120) on level k's Laplacian; returns the new x."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x, dtype=np.float64, copy=True)
        if lib().orc_smooth(self.h, k, smoother, omega, iters, _p(b), _p(x)):
            raise RuntimeError(lib().orc_last_error().decode())
        return x

    def coarse_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        lib().orc_coarse_solve(self.h, _p(b), _p(x))
        return x
