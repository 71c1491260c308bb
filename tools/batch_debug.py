import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2508_12501_b200 as d
h = d.MultigridHierarchy.from_base("ico", 10, max_nrhs=16)
B = h.make_rhs("uniform", 1, 16)
hb = torch.from_numpy(B).pin_memory().numpy()
outs = [torch.empty_like(torch.from_numpy(B)).pin_memory().numpy() for _ in range(6)]
plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
d.gmg_solve_batches(h, plan, [hb, hb], 1e-8, 200, out=outs[:2])
t0 = time.perf_counter(); r = d.gmg_solve_batches(h, plan, [hb] * 6, float(sys.argv[1]) if len(sys.argv) > 1 else 1e-8, int(sys.argv[2]) if len(sys.argv) > 2 else 200, out=outs); t1 = time.perf_counter()
print("6 batches", (t1 - t0) / 6 * 1e3, "ms per batch")
t0 = time.perf_counter(); d.gmg_solve(h, plan, hb, 1e-8, 200); t1 = time.perf_counter()
print("single", (t1 - t0) * 1e3, "ms")
