"""Time to 1e-8 on config 4 (16 RHS) through the public host-pointer API
(pinned buffers, H2D of b and D2H of x inside the timing): gmg_solve with
weighted Jacobi, Gauss-Seidel and symmetric GS V(2,2) cycles, and
gmg_preconditioned_cg with a V(2,2) Jacobi preconditioner."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402
from paper_2508_12501_b200 import _lib  # noqa: E402
from paper_2508_12501_b200.multigrid import _plan_struct  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nrhs = 16
h = d.MultigridHierarchy.from_base("ico", nsub, max_nrhs=nrhs)
lib = _lib.load()
hb = torch.from_numpy(h.make_rhs("uniform", 1, nrhs)).pin_memory()
hx = torch.empty_like(hb).pin_memory()
n = h.n()
hist = np.zeros((201, nrhs))
its = np.zeros(nrhs, dtype=np.int32)
conv = np.zeros(nrhs, dtype=np.int32)
fin = np.zeros(nrhs)
for name, m in [("jacobi", d.Smoother.WeightedJacobi), ("gs", d.Smoother.GaussSeidel),
                ("sgs", d.Smoother.SymmetricGaussSeidel)]:
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, d.SmootherConfig(method=m))
    ps, keep = _plan_struct(plan, h.levels())
    for rep in range(2):
        t0 = time.perf_counter()
        _lib.check(lib.decmg_gpu_solve(h.ctx, C.byref(ps), nrhs, C.c_void_p(hb.data_ptr()), None, 1e-8, 200,
                                       C.c_void_p(hx.data_ptr()), hist.ctypes.data_as(C.c_void_p),
                                       its.ctypes.data_as(C.c_void_p), fin.ctypes.data_as(C.c_void_p)), h.ctx)
        t = time.perf_counter() - t0
    print(f"gmg_solve {name:7s} cycles {its.max():3d}  time to 1e-8 {1e3 * t:7.1f} ms  "
          f"final {fin.max():.2e}  {n * nrhs * its.max() / t / 1e9:.2f} G unknowns*cycles/s")
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
ps, keep = _plan_struct(plan, h.levels())
for rep in range(2):
    t0 = time.perf_counter()
    _lib.check(lib.decmg_gpu_pcg(h.ctx, C.byref(ps), 1, nrhs, C.c_void_p(hb.data_ptr()), 1e-8, 200,
                                 C.c_void_p(hx.data_ptr()), hist.ctypes.data_as(C.c_void_p),
                                 its.ctypes.data_as(C.c_void_p), conv.ctypes.data_as(C.c_void_p),
                                 fin.ctypes.data_as(C.c_void_p)), h.ctx)
    t = time.perf_counter() - t0
print(f"gmg_pcg  V(2,2) jacobi iters {its.max():3d}  time to 1e-8 {1e3 * t:7.1f} ms  final {fin.max():.2e}")
