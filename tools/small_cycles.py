"""K V(2,2) Jacobi cycles of a small BASELINE config through run_cycles (for
launch lists / profiles): python tools/small_cycles.py config2 [K]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

CONFIGS = {"config1": ("square", 4, True, "sinsin"), "config2": ("ico", 6, False, "ylm"),
           "config3": ("ico", 8, False, "uniform")}
base, nsub, dirichlet, kind = CONFIGS[sys.argv[1]]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet)
b = h.make_rhs(kind, 1)
if not dirichlet:
    b = h.project_compatible(b)
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
plan.cycles = K
for _ in range(3):
    res = h.run_cycle(plan, b)
print(sys.argv[1], res.residual_history[-1])
