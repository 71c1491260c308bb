"""Per-pass time of the bottom-of-V kernel (DECMG_VTAIL_TRACE=1): the
%globaltimer stamps CTA 0 writes after every barrier of the last cycle.
    DECMG_VTAIL_TRACE=1 python tools/vtail_trace.py config3"""
import os
import sys
from pathlib import Path

import numpy as np

os.environ["DECMG_VTAIL_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

CONFIGS = {"config1": ("square", 4, True, "sinsin", 1), "config2": ("ico", 6, False, "ylm", 1),
           "config3": ("ico", 8, False, "uniform", 1), "config4": ("ico", 10, False, "uniform", 16)}
base, nsub, dirichlet, kind, nrhs = CONFIGS[sys.argv[1]]
h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
b = h.make_rhs(kind, 1, nrhs) if nrhs > 1 else h.make_rhs(kind, 1)
if not dirichlet:
    b = h.project_compatible(b)
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
plan.cycles = 2
for _ in range(3):
    h.run_cycle(plan, b)
t = np.zeros(256, dtype=np.uint64)
h._lib.decmg_gpu_export(h.ctx, 0, b"vtail_trace", t.ctypes.data_as(__import__("ctypes").c_void_p))
n = int(np.argmax(t[1:] == 0)) + 1 if np.any(t[1:] == 0) else 256
dt = np.diff(t[:n].astype(np.int64)) / 1000.0
print(sys.argv[1], "levels", [h.n(k) for k in range(h.levels())])
print("passes (us):", " ".join(f"{x:.1f}" for x in dt))
print("total us", dt.sum())
