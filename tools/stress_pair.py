"""Stress test of the two-sweep pass's inter-CTA hand-over (k_sweep_pair): the same V(2,2) cycles run
REPS times with the pass on, at several group sizes and horizons, each compared bit for bit with one
sweep per launch (DECMG_PAIR=0). A missed dependency (a sweep-2 row gathering a neighbour whose sweep-1
value is not yet published) would show up as a mismatch in some repetition.
    python tools/stress_pair.py [REPS]"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2508_12501_b200 as d  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 20
JAC = d.SmootherConfig(d.Smoother.WeightedJacobi)


def make(env, *a, **kw):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return d.MultigridHierarchy.from_base(*a, **kw)
    finally:
        for k, v in old.items():
            os.environ.pop(k, None) if v is None else os.environ.__setitem__(k, v)


total = 0
for base, nsub, dirich, nrhs in (("ico", 9, False, 16), ("ico", 10, False, 1), ("square", 11, True, 1)):
    h0 = make({"DECMG_PAIR": "0"}, base, nsub, dirichlet=dirich, max_nrhs=nrhs)
    b = h0.make_rhs("uniform", 3, nrhs) if nrhs > 1 else h0.make_rhs("uniform", 3)
    if not dirich:
        b = h0.project_compatible(b)
    plan = d.standard_plan(h0.levels(), d.CycleKind.V, 2, 2, smoother=JAC)
    plan.cycles = 2
    ref = h0.run_cycle(plan, b).x
    del h0
    for env in ({"DECMG_PAIR": "1"}, {"DECMG_PAIR": "1", "DECMG_PAIR_GROUP": "1"},
                {"DECMG_PAIR": "1", "DECMG_PAIR_GROUP": "1", "DECMG_PAIR_MIN_ROUNDS": "2"},
                {"DECMG_PAIR": "1", "DECMG_PAIR_AHEAD": "1"}):
        h = make(env, base, nsub, dirichlet=dirich, max_nrhs=nrhs)
        bad = 0
        for _ in range(REPS):
            x = h.run_cycle(plan, b).x
            bad += int(np.count_nonzero(x.view(np.uint64) != ref.view(np.uint64)))
        total += bad
        print(base, nsub, "nrhs", nrhs, env, "reps", REPS, "mismatching values", bad, flush=True)
        del h
print("TOTAL mismatches", total)
sys.exit(1 if total else 0)
