"""Vertex-partitioned multi-GPU V-cycle, emulated on one GPU.

All ranks of the world run inside this process on cuda:0 with device copies
in place of NCCL (no kernel ever waits on another rank's kernel). The
partitioned solve must give the single-GPU (= reference) iterate bit for bit
for every rank count, residual histories within 1e-10 relative and the same
cycle count.
"""
import numpy as np
import pytest

import paper_2508_12501_b200 as d
from oracle_ctypes import OracleHierarchy

pytestmark = pytest.mark.gpu
RTOL = 1e-10


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_partitioned_run_cycle_bitwise(world):
    base, nsub = "ico", 6
    o = OracleHierarchy(base, nsub)
    b = o.project(o.rhs("uniform", 3))
    dh = d.DistributedHierarchy(base, nsub, world, agglomerate_below=200)
    assert dh.agglomeration_level >= 2  # several distributed levels
    assert dh.halo0 > 0
    plan = d.standard_plan(dh.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 5
    res = dh.run_cycle(plan, b)
    ox, oh = o.run_cycles(b, ncycles=5)
    np.testing.assert_array_equal(res.x, ox)
    assert np.all(np.abs(res.residual_history - oh) <= RTOL * oh)


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_gmg_solve_matches_single_gpu(world):
    base, nsub = "ico", 7
    h = d.MultigridHierarchy.from_base(base, nsub)
    b = h.make_rhs("ylm", 1)
    rep1 = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi)), b, 1e-8, 200)
    dh = d.DistributedHierarchy(base, nsub, world, agglomerate_below=500)
    rep = dh.gmg_solve(d.standard_plan(dh.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi)), b, 1e-8, 200)
    assert rep.iterations == rep1.iterations
    np.testing.assert_array_equal(rep.solution, rep1.solution)
    np.testing.assert_allclose(rep.residual_history, rep1.residual_history, rtol=RTOL)


def test_partitioned_dirichlet_and_batch():
    """Config-1 family (Dirichlet square) and a 16-RHS batch across 4 ranks."""
    o = OracleHierarchy("square", 7, True)
    b = o.rhs("sinsin", 0)
    dh = d.DistributedHierarchy("square", 7, 4, dirichlet=True, agglomerate_below=100)
    plan = d.standard_plan(dh.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 4
    res = dh.run_cycle(plan, b)
    ox, oh = o.run_cycles(b, ncycles=4)
    np.testing.assert_array_equal(res.x, ox)

    nrhs = 16
    h = d.MultigridHierarchy.from_base("ico", 6, max_nrhs=nrhs)
    B = h.project_compatible(h.make_rhs("uniform", 9, nrhs))
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 3
    r1 = h.run_cycle(plan, B)
    dh = d.DistributedHierarchy("ico", 6, 4, max_nrhs=nrhs, agglomerate_below=300)
    r4 = dh.run_cycle(plan, B)
    np.testing.assert_array_equal(r4.x, r1.x)
    np.testing.assert_allclose(r4.residual_history, r1.residual_history, rtol=RTOL)


def test_nccl_single_rank_world():
    """The NCCL transport path with a world of one rank (the only GPU we get):
    communicator init, no peers, rank-ordered norm all-gather."""
    uid = d.nccl_unique_id()
    dh = d.DistributedHierarchy("ico", 5, 1, rank=0, nccl_id=uid)
    h = d.MultigridHierarchy.from_base("ico", 5)
    b = h.project_compatible(h.make_rhs("uniform", 2))
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 3
    np.testing.assert_array_equal(dh.run_cycle(plan, b).x, h.run_cycle(plan, b).x)
