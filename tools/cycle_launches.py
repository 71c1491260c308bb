"""Three batched V(2,2) cycles at config 4 (16 RHS) bracketed by cudaProfilerStart/Stop,
for an in-order ncu launch list:
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/cycle_launches.py"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nrhs = 16
h = d.MultigridHierarchy.from_base("ico", nsub, max_nrhs=nrhs)
B = h.project_compatible(h.make_rhs("uniform", 1, nrhs))
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
plan.cycles = 2
h.run_cycle(plan, B)
cudart = C.CDLL("libcudart.so.12")
plan.cycles = 3  # the last one is a steady-state cycle (the first starts from x = 0)
cudart.cudaProfilerStart()
h.run_cycle(plan, B)
cudart.cudaProfilerStop()
print("levels", [h.level_info(k)["nv"] for k in range(h.levels())])
