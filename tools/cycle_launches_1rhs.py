"""One V(2,2) cycle of a single-RHS config (default config 5b) between
cudaProfilerStart/Stop for an in-order ncu launch list or a --set full capture.
Usage: python tools/cycle_launches_1rhs.py [base] [nsub]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

base = sys.argv[1] if len(sys.argv) > 1 else "ico"
nsub = int(sys.argv[2]) if len(sys.argv) > 2 else 11
h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=(base == "square"))
b = h.make_rhs("uniform", 1)
if base != "square":
    b = h.project_compatible(b)
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
plan.cycles = 2
h.run_cycle(plan, b)
cudart = C.CDLL("libcudart.so.12")
plan.cycles = 1
cudart.cudaProfilerStart()
h.run_cycle(plan, b)
cudart.cudaProfilerStop()
