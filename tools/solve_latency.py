"""Host-to-host latency of one 16-RHS gmg_solve at config 4 (pinned buffers), best and median of 7.
Usage: [DECMG_GRAPH=0] python tools/solve_latency.py [nsub]"""
import os
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
h = d.MultigridHierarchy.from_base("ico", nsub, max_nrhs=16)
B = torch.from_numpy(h.make_rhs("uniform", 1, 16)).pin_memory().numpy()
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
ts = []
for _ in range(8):
    t0 = time.perf_counter()
    r = d.gmg_solve(h, plan, B, 1e-8, 200)
    ts.append(time.perf_counter() - t0)
ts = ts[1:]
print(f"DECMG_GRAPH={os.environ.get('DECMG_GRAPH', '1')}: gmg_solve best {1e3 * min(ts):.2f} ms, "
      f"median {1e3 * statistics.median(ts):.2f} ms, cycles {r.iterations[0]}")
