"""A small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the library on BASELINE configs 1-2 sizes --
the pipelined TMA ring (16-RHS and single-RHS tiles), the bottom-of-V
cooperative kernel, the graph-driven solve loop, exact Gauss-Seidel phases,
the exact projection chain, the tree-sum grid coarse CG (use_levels), the CG
smoother, GMG-PCG and the partitioned cycle (2 ranks emulated).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

jac = d.SmootherConfig(d.Smoother.WeightedJacobi)
# config 1: Dirichlet square x4, sin*sin
h = d.MultigridHierarchy.from_base("square", 4, dirichlet=True)
rep = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, jac), h.make_rhs("sinsin", 0), 1e-8, 50)
print("config1", rep.iterations, rep.final_relative_residual)
# config 2 size, 16-RHS batch (pipelined ring, 4 RHS per thread) and single RHS
h = d.MultigridHierarchy.from_base("ico", 6, max_nrhs=16)
B = h.make_rhs("ylm", 1, 16)
rep = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, jac), B, 1e-8, 50)
print("config2 batch", rep.iterations[:2])
b = h.make_rhs("ylm", 1)
rep = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, jac), b, 1e-8, 50)
print("config2", rep.iterations)
plan = d.standard_plan(h.levels(), d.CycleKind.W, 1, 1)  # Gauss-Seidel (reference default)
plan.cycles = 2
print("gs W", h.run_cycle(plan, h.project_compatible(b)).residual_history)
cg = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, d.SmootherConfig(d.Smoother.Cg))
cg.cycles = 1
print("cg smoother", h.run_cycle(cg, h.project_compatible(b)).residual_history)
pcg = d.gmg_preconditioned_cg(h, d.standard_plan(h.levels(), d.CycleKind.V, 1, 1, jac), b, 1e-8, 20)
print("pcg", pcg.iterations)
# use_levels: coarse solve of 2,401 unknowns on the grid CG
hu = d.MultigridHierarchy.from_base("equi:24:48:1.0", 2, use_levels=2)
rep = d.gmg_solve(hu, d.standard_plan(hu.levels(), d.CycleKind.W, 2, 2), hu.make_rhs("uniform", 7), 1e-8, 10)
print("levels used", rep.iterations)
# partitioned, 2 ranks emulated
dh = d.DistributedHierarchy("ico", 5, 2, agglomerate_below=100)
rep = dh.gmg_solve(d.standard_plan(dh.levels(), d.CycleKind.V, 2, 2, jac), dh.context().make_rhs("uniform", 3),
                   1e-8, 30)
print("dist", rep.iterations)
