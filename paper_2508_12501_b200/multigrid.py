"""Host-side mirror of the reference's multigrid API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/decmg/multigrid.hpp, solvers.hpp):

  Smoother / SmootherConfig / Transition / CyclePlan / CycleKind / standard_plan
                                             multigrid.hpp:55-89, multigrid.cpp:122-194
  MultigridHierarchy (+ build_hierarchy)     multigrid.hpp:106-143, multigrid.cpp:196-341
      .project_compatible / .run_cycle       multigrid.cpp:240-323
  gmg_solve / SolveReport                    solvers.hpp:17-59, solvers.cpp:251-279

std::invalid_argument surfaces as ValueError and std::runtime_error as
RuntimeError. Everything numerical runs in libdecmg_gpu.so on the GPU.
Right-hand sides may be a vector [n] or a batch [n, nrhs] (extension x4).
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, decmg_gpu_config, decmg_gpu_level_desc, decmg_gpu_plan


class Smoother(enum.Enum):
    GaussSeidel = 0
    SymmetricGaussSeidel = 1
    WeightedJacobi = 2
    Cg = 3


@dataclass
class SmootherConfig:
    # Default = the reference's GaussSeidel (multigrid.hpp:58): the forward
    # lexicographic sweep (multigrid.cpp:13-34), run on the device as a level
    # schedule bit-identical to the sequential sweep.
    # WeightedJacobi (multigrid.cpp:36-56) is the BASELINE configs' smoother and
    # is selected explicitly there. Cg = cg_fixed (multigrid.cpp:63-91) with
    # tree dots (within rounding).
    method: Smoother = Smoother.GaussSeidel
    jacobi_omega: float = 2.0 / 3.0


class Transition(enum.Enum):
    Down = "d"
    Up = "u"


class CycleKind(enum.Enum):
    V = 0
    W = 1
    F = 2


@dataclass
class CyclePlan:
    walk: List[Transition] = field(default_factory=list)
    pre: List[int] = field(default_factory=list)
    post: List[int] = field(default_factory=list)
    smoother: SmootherConfig = field(default_factory=SmootherConfig)
    cycles: int = 1

    def depth(self) -> int:  # multigrid.cpp:122-129
        level = deepest = 0
        for t in self.walk:
            level += 1 if t == Transition.Down else -1
            deepest = max(deepest, level)
        return deepest + 1

    def validate(self, levels: int) -> None:  # multigrid.cpp:131-143
        level = 0
        for t in self.walk:
            level += 1 if t == Transition.Down else -1
            if level < 0:
                raise ValueError("CyclePlan: walk rises above the finest level")
            if level > levels - 1:
                raise ValueError("CyclePlan: walk descends below the coarsest level")
        if level != 0:
            raise ValueError("CyclePlan: walk does not return to the finest level")
        if len(self.pre) < levels or len(self.post) < levels:
            raise ValueError("CyclePlan: missing per-level smoothing counts")
        if self.cycles < 0:
            raise ValueError("CyclePlan: negative cycle count")

    def walk_string(self) -> str:
        return "".join(t.value for t in self.walk)


def _emit_solve(out, k, levels, gamma):  # multigrid.cpp:149-156
    if k == levels - 1:
        return
    for _ in range(gamma):
        out.append(Transition.Down)
        _emit_solve(out, k + 1, levels, gamma)
        out.append(Transition.Up)


def _emit_f(out, k, levels):  # multigrid.cpp:159-167
    if k == levels - 1:
        return
    out.append(Transition.Down)
    _emit_f(out, k + 1, levels)
    out.append(Transition.Up)
    out.append(Transition.Down)
    _emit_solve(out, k + 1, levels, 1)
    out.append(Transition.Up)


def standard_plan(levels: int, kind: CycleKind = CycleKind.V, pre: int = 3, post: int = 3,
                  smoother: Optional[SmootherConfig] = None) -> CyclePlan:
    """Canonical V/W/F walk (multigrid.cpp:171-194)."""
    if levels < 1:
        raise ValueError("standard_plan: levels >= 1")
    plan = CyclePlan(pre=[pre] * levels, post=[post] * levels,
                     smoother=smoother if smoother is not None else SmootherConfig())
    if levels > 1:
        if kind == CycleKind.V:
            _emit_solve(plan.walk, 0, levels, 1)
        else:
            plan.walk.append(Transition.Down)
            if kind == CycleKind.W:
                _emit_solve(plan.walk, 1, levels, 2)
            else:
                _emit_f(plan.walk, 1, levels)
            plan.walk.append(Transition.Up)
    plan.validate(levels)
    return plan


@dataclass
class CycleResult:
    x: np.ndarray
    residual_history: np.ndarray  # [cycles] or [cycles, nrhs]


@dataclass
class SolveReport:  # solvers.hpp:17-30
    solution: np.ndarray
    residual_history: list
    cumulative_seconds: list
    iterations: object
    converged: object
    final_relative_residual: object
    wall_seconds: float
    stagnated: bool = False
    config_echo: dict = field(default_factory=lambda: {"solver": "gmg"})

    def to_json(self, include_solution: bool = False) -> dict:  # solvers.cpp:31-43
        j = {"iterations": self.iterations, "converged": self.converged, "stagnated": self.stagnated,
             "final_relative_residual": self.final_relative_residual, "wall_seconds": self.wall_seconds,
             "residual_history": self.residual_history, "cumulative_seconds": self.cumulative_seconds,
             "config": self.config_echo}
        if include_solution:
            j["solution"] = np.asarray(self.solution).tolist()
        return j

    def write_residual_csv(self, path: str) -> None:  # solvers.cpp:45-54
        with open(path, "w") as f:
            f.write("cycle,rel_residual,cumulative_seconds\n")
            for i, r in enumerate(self.residual_history):
                t = self.cumulative_seconds[i] if i < len(self.cumulative_seconds) else 0.0
                f.write(f"{i + 1},{r:.17g},{t:.17g}\n")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


_SMOOTHER_C = {Smoother.WeightedJacobi: 0, Smoother.GaussSeidel: 1, Smoother.SymmetricGaussSeidel: 2,
               Smoother.Cg: 3}


def _plan_struct(plan: CyclePlan, levels: int):
    if plan.smoother.method not in _SMOOTHER_C:
        raise ValueError("smoother: unknown smoother")
    plan.validate(levels)
    pre = (C.c_int * levels)(*plan.pre[:levels])
    post = (C.c_int * levels)(*plan.post[:levels])
    walk = plan.walk_string().encode()
    s = decmg_gpu_plan(walk=walk, pre=C.cast(pre, C.POINTER(C.c_int)), post=C.cast(post, C.POINTER(C.c_int)),
                       pre_all=0, post_all=0, smoother=_SMOOTHER_C[plan.smoother.method],
                       jacobi_omega=float(plan.smoother.jacobi_omega))
    return s, (pre, post, walk)  # keep buffers alive


def base_mesh(spec: str):
    """(positions [nv,3], corner triples [nt,3]) of a named base complex."""
    lib = _lib.load()
    nv, nt = C.c_int(), C.c_int()
    check(lib.decmg_base_mesh(spec.encode(), None, C.byref(nv), None, C.byref(nt)))
    pos = np.empty((nv.value, 3), dtype=np.float64)
    tri = np.empty((nt.value, 3), dtype=np.int32)
    check(lib.decmg_base_mesh(spec.encode(), _ptr(pos), C.byref(nv), _ptr(tri), C.byref(nt)))
    return pos, tri


def read_obj(path) -> tuple:
    """read_obj (mesh_io.cpp:19-69): (positions [nv,3], corner triples [nt,3]);
    RuntimeError with the reference's message on a malformed file."""
    lib = _lib.load()
    nv, nt = C.c_int(), C.c_int()
    p = str(path).encode()
    if lib.decmg_read_obj(p, None, C.byref(nv), None, C.byref(nt)) != _lib.DECMG_OK:
        raise RuntimeError(lib.decmg_io_last_error().decode())
    pos = np.empty((nv.value, 3), dtype=np.float64)
    tri = np.empty((nt.value, 3), dtype=np.int32)
    check(lib.decmg_read_obj(p, _ptr(pos), C.byref(nv), _ptr(tri), C.byref(nt)))
    return pos, tri


class MultigridHierarchy:
    """Device-resident level hierarchy (finest level = 0)."""

    _DT = {"positions": np.float64, "dual_areas": np.float64, "diag": np.float64, "L_values": np.float64,
           "P_values": np.float64, "R_values": np.float64}

    def __init__(self, ctx: int, dirichlet: bool, max_nrhs: int, owned: bool = True):
        self._ctx = C.c_void_p(ctx)
        self.dirichlet = dirichlet
        self.max_nrhs = max_nrhs
        self._owned = owned
        self._lib = _lib.load()

    # -- construction ------------------------------------------------------
    @classmethod
    def from_base(cls, base, nsub: int, dirichlet: bool = False, project_sphere: Optional[bool] = None,
                  device: int = 0, max_nrhs: int = 1, cubic: bool = False, use_levels: int = 0,
                  clamp_dual_areas: bool = False) -> "MultigridHierarchy":
        """build_hierarchy(base, subdivision_tower(base, Binary|Cubic, nsub), use_levels,
        HierarchyOptions{hodge.clamp_dual_areas}) on the GPU (multigrid.cpp:325-341).

        base: a spec string for base_mesh() -- with the suffix "+cubic" for
        SubdivisionScheme::Cubic, as in the reference harness -- or a
        (positions, corner_triples) pair. use_levels > 0 keeps only the finest
        use_levels meshes (the coarse solve runs on a finer mesh).
        """
        lib = _lib.load()
        if isinstance(base, str):
            if base.endswith("+cubic"):
                cubic, base = True, base[: -len("+cubic")]
            if project_sphere is None:
                project_sphere = base == "ico"
            pos, tri = base_mesh(base)
        else:
            pos, tri = base
            project_sphere = bool(project_sphere)
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        flags = ((_lib.DECMG_PROJECT_SPHERE if project_sphere else 0) | (_lib.DECMG_DIRICHLET if dirichlet else 0)
                 | (_lib.DECMG_CUBIC if cubic else 0) | (_lib.DECMG_CLAMP_DUAL_AREAS if clamp_dual_areas else 0))
        cfg = decmg_gpu_config(device=device, max_nrhs=max_nrhs)
        out = C.c_void_p()
        check(lib.decmg_gpu_create_from_base_ex(_ptr(pos), pos.shape[0], _ptr(tri), tri.shape[0], nsub, use_levels,
                                                flags, C.byref(cfg), C.byref(out)))
        return cls(out.value, dirichlet, max_nrhs)

    @classmethod
    def from_levels(cls, levels: Sequence[dict], dirichlet: bool = False, device: int = 0,
                    max_nrhs: int = 1) -> "MultigridHierarchy":
        """MultigridHierarchy from assembled per-level CSR (reference layout)."""
        lib = _lib.load()
        keep = []
        descs = (decmg_gpu_level_desc * len(levels))()
        for k, lv in enumerate(levels):
            d = descs[k]

            def arr(name, dt):
                a = lv.get(name)
                if a is None:
                    return None
                a = np.ascontiguousarray(a, dtype=dt)
                keep.append(a)
                return _ptr(a)

            d.nv = int(lv["nv"])
            d.L_row_ptr = arr("L_row_ptr", np.int32)
            d.L_col_idx = arr("L_col_idx", np.int32)
            d.L_values = arr("L_values", np.float64)
            d.L_nnz = len(lv["L_values"])
            d.dual_areas = arr("dual_areas", np.float64)
            d.boundary = arr("boundary", np.int32)
            if "P_row_ptr" in lv:
                d.P_row_ptr = arr("P_row_ptr", np.int32)
                d.P_col_idx = arr("P_col_idx", np.int32)
                d.P_values = arr("P_values", np.float64)
                d.P_nnz = len(lv["P_values"])
                d.R_row_ptr = arr("R_row_ptr", np.int32)
                d.R_col_idx = arr("R_col_idx", np.int32)
                d.R_values = arr("R_values", np.float64)
                d.R_nnz = len(lv["R_values"])
        cfg = decmg_gpu_config(device=device, max_nrhs=max_nrhs)
        out = C.c_void_p()
        flags = _lib.DECMG_DIRICHLET if dirichlet else 0
        check(lib.decmg_gpu_create_from_levels(descs, len(levels), flags, C.byref(cfg), C.byref(out)))
        return cls(out.value, dirichlet, max_nrhs)

    def close(self) -> None:
        if self._ctx and self._ctx.value and self._owned:
            self._lib.decmg_gpu_destroy(self._ctx)
        self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- structure ---------------------------------------------------------
    @property
    def ctx(self):
        return self._ctx

    def levels(self) -> int:
        return self._lib.decmg_gpu_levels(self._ctx)

    def level_info(self, k: int) -> dict:
        c = (C.c_int64 * 6)()
        check(self._lib.decmg_gpu_level_info(self._ctx, k, c), self._ctx)
        return dict(nv=c[0], ne=c[1], nt=c[2], nnz_L=c[3], nnz_P=c[4], nnz_R=c[5])

    def n(self, k: int = 0) -> int:
        return self.level_info(k)["nv"]

    def export(self, k: int, name: str) -> np.ndarray:
        cnt = self._lib.decmg_gpu_export(self._ctx, k, name.encode(), None)
        if cnt < 0:
            raise KeyError(f"{name} not available on level {k}")
        out = np.empty(cnt, dtype=self._DT.get(name, np.int32))
        if self._lib.decmg_gpu_export(self._ctx, k, name.encode(), _ptr(out)) < 0:
            raise _lib.CudaError("export failed")
        return out

    def write_obj(self, k: int, path) -> None:
        """write_obj (mesh_io.cpp:71-82) of level k's complex."""
        check(self._lib.decmg_gpu_write_obj(self._ctx, k, str(path).encode()), self._ctx)

    def write_matrix_market(self, k: int, op: str, path) -> None:
        """SparseOperator::write_matrix_market (sparse.cpp:247-259) of level k's
        L, P or R ('L' / 'P' / 'R')."""
        check(self._lib.decmg_gpu_write_matrix_market(self._ctx, k, op.encode(), str(path).encode()), self._ctx)

    def mesh_hash(self, k: int) -> int:
        h = C.c_uint64()
        check(self._lib.decmg_gpu_mesh_hash(self._ctx, k, C.byref(h)), self._ctx)
        return h.value

    # -- numerics ----------------------------------------------------------
    def _vec(self, b, n):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.ndim == 1:
            nrhs = 1
        elif b.ndim == 2:
            nrhs = b.shape[1]
        else:
            raise ValueError("rhs must be [n] or [n, nrhs]")
        if b.shape[0] != n:
            raise ValueError("run_cycle: rhs size mismatch")
        return b, nrhs

    def apply(self, k: int, op: str, x: np.ndarray) -> np.ndarray:
        """SparseOperator::apply of level k's L, P or R (sparse.cpp:209-218)."""
        info = self.level_info(k)
        nc = self.level_info(k + 1)["nv"] if op in "PR" and k + 1 < self.levels() else 0
        nin = nc if op == "P" else info["nv"]
        nout = nc if op == "R" else info["nv"]
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (nin,):
            raise ValueError("apply: length mismatch")
        y = np.empty(nout)
        check(self._lib.decmg_gpu_apply(self._ctx, k, op.encode(), _ptr(x), _ptr(y)), self._ctx)
        return y

    def project_compatible(self, b: np.ndarray) -> np.ndarray:
        b, nrhs = self._vec(b, self.n())
        out = np.array(b, copy=True)
        check(self._lib.decmg_gpu_project_compatible(self._ctx, nrhs, _ptr(out)), self._ctx)
        return out

    def run_cycle(self, plan: CyclePlan, b: np.ndarray, x0: Optional[np.ndarray] = None) -> CycleResult:
        n = self.n()
        b, nrhs = self._vec(b, n)
        ps, keep = _plan_struct(plan, self.levels())
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=np.float64)
            if x0.shape != b.shape:
                raise ValueError("run_cycle: rhs size mismatch")
        x = np.empty_like(b)
        hist = np.empty((max(plan.cycles, 1), nrhs))
        check(self._lib.decmg_gpu_run_cycles(self._ctx, C.byref(ps), nrhs, _ptr(b),
                                             None if x0 is None else _ptr(x0), plan.cycles, _ptr(x),
                                             _ptr(hist)), self._ctx)
        hist = hist[: plan.cycles]
        return CycleResult(x=x, residual_history=hist[:, 0] if b.ndim == 1 else hist)

    def make_rhs(self, kind: str, seed: int, nrhs: int = 1) -> np.ndarray:
        b = np.empty((self.n(), nrhs))
        check(self._lib.decmg_gpu_make_rhs(self._ctx, kind.encode(), seed, nrhs, _ptr(b)), self._ctx)
        return b[:, 0].copy() if nrhs == 1 else b

    def set_timing(self, enable: bool) -> None:
        check(self._lib.decmg_gpu_set_timing(self._ctx, int(enable)), self._ctx)

    def timing(self, cls: int):
        n, ms, by = C.c_int64(), C.c_double(), C.c_double()
        check(self._lib.decmg_gpu_get_timing(self._ctx, cls, C.byref(n), C.byref(ms), C.byref(by)), self._ctx)
        return n.value, ms.value, by.value

    def launch_count(self) -> int:
        return self._lib.decmg_gpu_launch_count(self._ctx)

    def projection_fallbacks(self) -> int:
        """(segment, RHS) pairs of the exact projection chain that ran the literal add chain."""
        return self._lib.decmg_gpu_projection_fallbacks(self._ctx)

    def stream(self) -> int:
        return self._lib.decmg_gpu_stream(self._ctx)


def _last_times(h) -> list:
    """SolveReport::cumulative_seconds of the last solve / pcg on h (decmg_gpu_last_times)."""
    n = h._lib.decmg_gpu_last_times(h.ctx, None, 0)
    t = np.zeros(max(n, 0))
    if n > 0:
        h._lib.decmg_gpu_last_times(h.ctx, _ptr(t), n)
    return t.tolist()


def smooth(h: "MultigridHierarchy", k: int, x: np.ndarray, b: np.ndarray, cfg: "SmootherConfig", iters: int,
           weighted: bool = False) -> np.ndarray:
    """smooth(A = level k's Laplacian, x, b, cfg, iters, weights) (multigrid.hpp:66-68,
    multigrid.cpp:95-120) on the device; returns the smoothed x. weighted: the CG
    smoother's inner product uses the level's dual areas (cycle_once's call),
    else plain dots (the reference's default weights = {})."""
    n = h.level_info(k)["nv"]
    xx = np.array(x, dtype=np.float64, copy=True, order="C")
    bb = np.ascontiguousarray(b, dtype=np.float64)
    if xx.shape[0] != n or bb.shape != xx.shape:
        raise ValueError("smooth: shape mismatch")
    nrhs = 1 if xx.ndim == 1 else xx.shape[1]
    check(h._lib.decmg_gpu_smooth(h.ctx, k, _SMOOTHER_C[cfg.method], cfg.jacobi_omega, iters, nrhs, _ptr(xx),
                                  _ptr(bb), int(weighted)), h.ctx)
    return xx


def build_hierarchy(base, nsub: int, **kw) -> MultigridHierarchy:
    """build_hierarchy(base, subdivision_tower(base, Binary, nsub)) (multigrid.cpp:325-341)."""
    return MultigridHierarchy.from_base(base, nsub, **kw)


def gmg_solve(h: MultigridHierarchy, plan: CyclePlan, b: np.ndarray, tol: float, max_cycles: int,
              x0: Optional[np.ndarray] = None) -> SolveReport:
    """Standalone multigrid solve (solvers.cpp:251-279); batched RHS stop independently."""
    t0 = time.perf_counter()
    n = h.n()
    b, nrhs = h._vec(b, n)
    ps, keep = _plan_struct(plan, h.levels())
    if x0 is not None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
    x = np.empty_like(b)
    hist = np.zeros((max(max_cycles, 1), nrhs))
    done = np.zeros(nrhs, dtype=np.int32)
    final = np.zeros(nrhs)
    check(h._lib.decmg_gpu_solve(h.ctx, C.byref(ps), nrhs, _ptr(b), None if x0 is None else _ptr(x0), tol,
                                 max_cycles, _ptr(x), _ptr(hist), _ptr(done), _ptr(final)), h.ctx)
    wall = time.perf_counter() - t0
    times = _last_times(h)
    if b.ndim == 1:
        it = int(done[0])
        hl = hist[:it, 0].tolist()
        return SolveReport(solution=x, residual_history=hl, cumulative_seconds=times[:it],
                           iterations=it, converged=bool((hl[-1] if it else final[0]) <= tol),
                           final_relative_residual=float(final[0]), wall_seconds=wall)
    hl = [hist[: done[j], j].tolist() for j in range(nrhs)]
    return SolveReport(solution=x, residual_history=hl, cumulative_seconds=[times[: done[j]] for j in range(nrhs)],
                       iterations=done.tolist(),
                       converged=[bool((hl[j][-1] if done[j] else final[j]) <= tol) for j in range(nrhs)],
                       final_relative_residual=final.tolist(), wall_seconds=wall)


def gmg_solve_batches(h: MultigridHierarchy, plan: CyclePlan, batches, tol: float, max_cycles: int,
                      out=None) -> list:
    """A stream of independent gmg_solve batches (extension x6, decmg_gpu_solve_batches):
    batch k+1's upload and projection and batch k-1's download overlap batch
    k's cycles; every batch equals its own gmg_solve bit for bit. batches: list
    of [n] or [n, nrhs] arrays of one shape (pinned, e.g. torch pin_memory
    views, for the copies to overlap); out: optional list of result arrays."""
    nb = len(batches)
    n = h.n()
    arrs = [h._vec(b, n)[0] for b in batches]
    nrhs = 1 if arrs and arrs[0].ndim == 1 else (arrs[0].shape[1] if arrs else 1)
    if any(a.shape != arrs[0].shape for a in arrs):
        raise ValueError("gmg_solve_batches: batches differ in shape")
    outs = out if out is not None else [np.empty_like(a) for a in arrs]
    ps, keep = _plan_struct(plan, h.levels())
    bptrs = (C.c_void_p * max(nb, 1))(*[a.ctypes.data for a in arrs])
    xptrs = (C.c_void_p * max(nb, 1))(*[o.ctypes.data for o in outs])
    mc = max(max_cycles, 1)
    hist = np.zeros((max(nb, 1), mc, nrhs))
    done = np.zeros((max(nb, 1), nrhs), dtype=np.int32)
    final = np.zeros((max(nb, 1), nrhs))
    t0 = time.perf_counter()
    check(h._lib.decmg_gpu_solve_batches(h.ctx, C.byref(ps), nrhs, nb, bptrs, tol, max_cycles, xptrs, _ptr(hist),
                                         _ptr(done), _ptr(final)), h.ctx)
    wall = time.perf_counter() - t0
    reps = []
    for k in range(nb):
        if arrs[k].ndim == 1:
            it = int(done[k, 0])
            reps.append(SolveReport(solution=outs[k], residual_history=hist[k, :it, 0].tolist(), cumulative_seconds=[],
                                    iterations=it, converged=bool(final[k, 0] <= tol),
                                    final_relative_residual=float(final[k, 0]), wall_seconds=wall))
        else:
            reps.append(SolveReport(solution=outs[k], residual_history=[hist[k, : done[k, j], j].tolist()
                                                                        for j in range(nrhs)],
                                    cumulative_seconds=[], iterations=done[k].tolist(),
                                    converged=(final[k] <= tol).tolist(), final_relative_residual=final[k].tolist(),
                                    wall_seconds=wall))
    return reps


def gmg_preconditioned_cg(h: MultigridHierarchy, inner_plan: CyclePlan, b: np.ndarray, tol: float,
                          maxiter: int) -> SolveReport:
    """gmg_preconditioned_cg (solvers.cpp:118-130): weighted CG on the fine
    operator (dual-area inner product) preconditioned by inner_plan.cycles
    cycles of inner_plan from zero; b is projected first (Neumann only).
    residual_history has iterations + 1 entries (the initial residual first);
    final_relative_residual is recomputed from the solution. A CG breakdown
    raises RuntimeError with the reference's message."""
    t0 = time.perf_counter()
    n = h.n()
    b, nrhs = h._vec(b, n)
    ps, keep = _plan_struct(inner_plan, h.levels())
    x = np.empty_like(b)
    hist = np.zeros((maxiter + 1, nrhs))
    its = np.zeros(nrhs, dtype=np.int32)
    conv = np.zeros(nrhs, dtype=np.int32)
    final = np.zeros(nrhs)
    check(h._lib.decmg_gpu_pcg(h.ctx, C.byref(ps), int(inner_plan.cycles), nrhs, _ptr(b), tol, maxiter, _ptr(x),
                               _ptr(hist), _ptr(its), _ptr(conv), _ptr(final)), h.ctx)
    wall = time.perf_counter() - t0
    times = _last_times(h)
    if b.ndim == 1:
        it = int(its[0])
        return SolveReport(solution=x, residual_history=hist[: it + 1, 0].tolist(), cumulative_seconds=times[: it + 1],
                           iterations=it, converged=bool(conv[0]), final_relative_residual=float(final[0]),
                           wall_seconds=wall, config_echo={"solver": "gmg_pcg"})
    return SolveReport(solution=x, residual_history=[hist[: its[j] + 1, j].tolist() for j in range(nrhs)],
                       cumulative_seconds=[times[: its[j] + 1] for j in range(nrhs)], iterations=its.tolist(),
                       converged=[bool(v) for v in conv], final_relative_residual=final.tolist(), wall_seconds=wall,
                       config_echo={"solver": "gmg_pcg"})


class DistributedHierarchy:
    """Vertex-partitioned multi-GPU hierarchy.

    world_size ranks. Transports (include/decmg_gpu.h):
      * nccl_id=None, shm_path=None: all ranks emulated in this process on one
        device (device copies instead of NCCL);
      * nccl_id: this process is `rank` of a one-process-per-GPU job and
        nccl_id is the 128-byte id from `nccl_unique_id()` on rank 0;
      * shm_path: this process is `rank`, halos host-staged through the shared
        file shm_path (several ranks may share one GPU: the multi-process test).
    """

    def __init__(self, base, nsub: int, world_size: int, rank: int = 0, nccl_id: Optional[bytes] = None,
                 dirichlet: bool = False, project_sphere: Optional[bool] = None, device: int = 0, max_nrhs: int = 1,
                 agglomerate_below: int = 65536, shm_path: Optional[str] = None):
        self._lib = _lib.load()
        if isinstance(base, str):
            if project_sphere is None:
                project_sphere = base == "ico"
            pos, tri = base_mesh(base)
        else:
            pos, tri = base
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        flags = (_lib.DECMG_PROJECT_SPHERE if project_sphere else 0) | (_lib.DECMG_DIRICHLET if dirichlet else 0)
        cfg = decmg_gpu_config(device=device, max_nrhs=max_nrhs)
        out = C.c_void_p()
        idbuf = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), len(nccl_id))
        if nccl_id is not None:
            tr = _lib.decmg_gpu_dist_transport(_lib.DECMG_DIST_NCCL, C.cast(idbuf, C.c_void_p), None)
        elif shm_path is not None:
            tr = _lib.decmg_gpu_dist_transport(_lib.DECMG_DIST_SHM, None, str(shm_path).encode())
        else:
            tr = _lib.decmg_gpu_dist_transport(_lib.DECMG_DIST_EMULATE, None, None)
        check(self._lib.decmg_gpu_dist_create_ex(_ptr(pos), pos.shape[0], _ptr(tri), tri.shape[0], nsub, flags,
                                                 C.byref(cfg), world_size, rank, C.byref(tr), agglomerate_below,
                                                 C.byref(out)), None, dist=True)
        self._d = out
        self.world_size = world_size
        self.dirichlet = dirichlet
        self.max_nrhs = max_nrhs
        ka, lv, own, halo = C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        self._lib.decmg_gpu_dist_info(self._d, C.byref(ka), C.byref(lv), C.byref(own), C.byref(halo))
        self.agglomeration_level, self.nlevels = ka.value, lv.value
        self.owned0, self.halo0 = own.value, halo.value

    def close(self):
        if getattr(self, "_d", None) and self._d.value:
            self._lib.decmg_gpu_dist_destroy(self._d)
            self._d = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def levels(self) -> int:
        return self.nlevels

    def last_cycle_ms(self) -> float:
        return self._lib.decmg_gpu_dist_last_cycle_ms(self._d)

    def context(self) -> "MultigridHierarchy":
        """Non-owning view of this rank's full (replicated) hierarchy."""
        return MultigridHierarchy(self._lib.decmg_gpu_dist_context(self._d), self.dirichlet, self.max_nrhs,
                                  owned=False)

    def launch_count(self) -> int:
        return self._lib.decmg_gpu_dist_launch_count(self._d)

    def _run(self, plan, b, x0, cycles, solve, tol):
        b = np.ascontiguousarray(b, dtype=np.float64)
        nrhs = 1 if b.ndim == 1 else b.shape[1]
        ps, keep = _plan_struct(plan, self.nlevels)
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=np.float64)
        x = np.empty_like(b)
        hist = np.zeros((max(cycles, 1), nrhs))
        done = np.zeros(nrhs, dtype=np.int32)
        fin = np.zeros(nrhs)
        check(self._lib.decmg_gpu_dist_run(self._d, C.byref(ps), nrhs, _ptr(b), None if x0 is None else _ptr(x0),
                                           cycles, int(solve), tol, _ptr(x), _ptr(hist), _ptr(done), _ptr(fin)),
              self._d, dist=True)
        return x, hist, done, fin

    def run_cycle(self, plan: CyclePlan, b, x0=None) -> CycleResult:
        x, hist, done, fin = self._run(plan, b, x0, plan.cycles, False, 0.0)
        hist = hist[: plan.cycles]
        return CycleResult(x=x, residual_history=hist[:, 0] if np.ndim(b) == 1 else hist)

    def gmg_solve(self, plan: CyclePlan, b, tol: float, max_cycles: int, x0=None) -> SolveReport:
        t0 = time.perf_counter()
        x, hist, done, fin = self._run(plan, b, x0, max_cycles, True, tol)
        wall = time.perf_counter() - t0
        if np.ndim(b) == 1:
            it = int(done[0])
            return SolveReport(solution=x, residual_history=hist[:it, 0].tolist(), cumulative_seconds=[],
                               iterations=it, converged=bool(fin[0] <= tol), final_relative_residual=float(fin[0]),
                               wall_seconds=wall)
        return SolveReport(solution=x, residual_history=[hist[: done[j], j].tolist() for j in range(len(done))],
                           cumulative_seconds=[], iterations=done.tolist(), converged=(fin <= tol).tolist(),
                           final_relative_residual=fin.tolist(), wall_seconds=wall)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_lib.load().decmg_gpu_nccl_unique_id(buf, 128))
    return buf.raw
