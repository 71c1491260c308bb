"""Jacobi vs Gauss-Seidel vs symmetric GS on config 4 (16 RHS): device time
per V(2,2) cycle (CUDA events around one run_cycles_dev call of K cycles,
inputs resident in HBM) and the cycles gmg_solve needs to reach 1e-8."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402
from paper_2508_12501_b200 import _lib  # noqa: E402
from paper_2508_12501_b200.multigrid import _plan_struct  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
K = 10
nrhs = 16
h = d.MultigridHierarchy.from_base("ico", nsub, max_nrhs=nrhs)
lib = _lib.load()
B = h.project_compatible(h.make_rhs("uniform", 1, nrhs))
db = torch.from_numpy(B).cuda()
dx = torch.zeros_like(db)
dh = torch.zeros((K, nrhs), dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(h.stream())
for name, m in [("jacobi", d.Smoother.WeightedJacobi), ("gs", d.Smoother.GaussSeidel),
                ("sgs", d.Smoother.SymmetricGaussSeidel)]:
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, d.SmootherConfig(method=m))
    ps, keep = _plan_struct(plan, h.levels())

    def run(k):
        _lib.check(lib.decmg_gpu_run_cycles_dev(h.ctx, C.byref(ps), nrhs, C.c_void_p(db.data_ptr()), None, k,
                                                C.c_void_p(dx.data_ptr()), C.c_void_p(dh.data_ptr())), h.ctx)

    run(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(K)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    rep = d.gmg_solve(h, plan, B, 1e-8, 200)
    it = max(rep.iterations)
    print(f"{name:7s} {ms:7.3f} ms per V(2,2) cycle  cycles to 1e-8: {it}  "
          f"device time to 1e-8 ~ {ms * it:6.1f} ms  hist[{K - 1}] {dh[K - 1].max().item():.3e}")
