"""Bitwise check of the wavefront sweep pairs (DECMG_PAIR=1) against separate
sweeps: run with both settings and compare the printed hashes.
Usage: DECMG_PAIR=1 python tools/pair_check.py [nsub] [nrhs] [cycles]"""
import hashlib
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

nsub = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cyc = int(sys.argv[3]) if len(sys.argv) > 3 else 3
h = d.MultigridHierarchy.from_base("ico", nsub, max_nrhs=nrhs)
B = h.project_compatible(h.make_rhs("uniform", 1, nrhs))
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2)
plan.cycles = cyc
t0 = time.perf_counter()
res = h.run_cycle(plan, B)
t1 = time.perf_counter()
print(f"DECMG_PAIR={os.environ.get('DECMG_PAIR', '0')} n={h.n()} nrhs={nrhs} cycles={cyc} "
      f"x={hashlib.sha1(res.x.tobytes()).hexdigest()[:16]} hist={np.asarray(res.residual_history).ravel()[:4]} "
      f"wall={t1 - t0:.3f}s")
