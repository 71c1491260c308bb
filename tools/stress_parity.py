"""Repeated bitwise check of run_cycle against the oracle on the larger single-RHS meshes (square x11/x12
Dirichlet, icosphere x10): the stress test that exposed the stage-release race fixed in k_rowop_pipe."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2508_12501_b200 as d
from oracle_ctypes import OracleHierarchy
for base, dirich, nsub in (("square", True, 11), ("square", True, 12), ("ico", False, 10)):
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirich)
    o = OracleHierarchy(base, nsub, dirichlet=dirich)
    b = o.rhs("uniform", 3)
    if not dirich: b = o.project(b)
    for cyc in (1, 2):
        plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi)); plan.cycles = cyc
        x = h.run_cycle(plan, b).x
        ox, oh = o.run_cycles(b, ncycles=cyc)
        diff = np.flatnonzero(x != ox)
        print(base, nsub, dirich, "cycles", cyc, "n", h.n(), "mismatches", diff.size, "first", diff[:5], flush=True)
