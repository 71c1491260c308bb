"""Where the time of one 16-RHS gmg_solve (host -> host) goes on config 4."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402
from paper_2508_12501_b200 import _lib  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nrhs = 16
h = d.MultigridHierarchy.from_base("ico", nsub, max_nrhs=nrhs)
B = h.make_rhs("uniform", 1, nrhs)
hb = torch.from_numpy(B).pin_memory()
hx = torch.empty_like(hb).pin_memory()
db = torch.empty(hb.shape, dtype=torch.float64, device="cuda")
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    db.copy_(hb, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    hx.copy_(db, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    h.set_timing(True)
    h.timing(-1)
    t3 = time.perf_counter()
    rep_ = d.gmg_solve(h, plan, hb.numpy(), 1e-8, 200)
    t4 = time.perf_counter()
    cls = {c: h.timing(c) for c in range(8)}
    h.set_timing(False)
    print(f"H2D {1e3*(t1-t0):.1f} ms  D2H {1e3*(t2-t1):.1f} ms  solve(host API) {1e3*(t4-t3):.1f} ms  "
          f"cycles {rep_.iterations[0]}")
    print("  classes ms:", {k: round(v[1], 2) for k, v in cls.items()}, "launches", sum(v[0] for v in cls.values()))
