"""One rank of a multi-process partitioned solve (tests/test_gpu_dist.py).

  python tests/dist_worker.py SHM_PATH WORLD RANK BASE NSUB NRHS DIRICHLET AGGL OUT.npz

Each process builds its own context and partition (decmg_gpu_dist_create_ex
with the host-staged transport) on cuda:0, runs run_cycle (4
V(2,2) Jacobi cycles) and gmg_solve (tol 1e-8), and saves what it got.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2508_12501_b200 as d  # noqa: E402


def main():
    shm, world, rank, base, nsub, nrhs, dirichlet, aggl, out = sys.argv[1:10]
    world, rank, nsub, nrhs, aggl = int(world), int(rank), int(nsub), int(nrhs), int(aggl)
    dirichlet = dirichlet == "1"
    dh = d.DistributedHierarchy(base, nsub, world, rank=rank, shm_path=shm, dirichlet=dirichlet, max_nrhs=nrhs,
                                agglomerate_below=aggl)
    g = dh.context()
    kind = "sinsin" if dirichlet else "uniform"
    b = g.make_rhs(kind, 7, nrhs) if nrhs > 1 else g.make_rhs(kind, 7)
    plan = d.standard_plan(dh.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 4
    bp = b if dirichlet else g.project_compatible(b)
    res = dh.run_cycle(plan, bp)
    rep = dh.gmg_solve(plan, b, 1e-8, 100)
    np.savez(out, x=res.x, hist=np.asarray(res.residual_history), sx=rep.solution,
             shist=np.asarray(rep.residual_history, dtype=object) if nrhs > 1 else np.asarray(rep.residual_history),
             it=np.asarray(rep.iterations), b=b, ka=dh.agglomeration_level, halo=dh.halo0,
             launches=dh.launch_count())


if __name__ == "__main__":
    main()
