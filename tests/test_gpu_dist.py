"""Vertex-partitioned multi-GPU V-cycle on one GPU.

Emulation: all ranks of the world run inside this process on cuda:0 with
device copies in place of NCCL (no kernel ever waits on another rank's
kernel). Multi-process: world_size processes on cuda:0, each with its own
context and partition, exchanging halos through host staging with a host
barrier (no kernel waits on another process). The partitioned solve must give
the single-GPU (= reference) iterate bit for bit for every rank count,
residual histories within 1e-10 relative and the same cycle count.
"""
import os
import subprocess
import sys
import tempfile
from pathlib import Path

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


@pytest.mark.parametrize("graph", ["0", "1"])
@pytest.mark.parametrize("pre,post", [(2, 2), (2, 1), (1, 1)])
def test_partitioned_graph_and_host_loops_agree(monkeypatch, graph, pre, post):
    """Cycles replayed as a CUDA graph (DECMG_GRAPH=1, parity-preserving walks)
    and the eager loop give the oracle's iterates, cycle counts and histories."""
    monkeypatch.setenv("DECMG_GRAPH", graph)
    o = OracleHierarchy("ico", 6)
    b = o.rhs("uniform", 11)
    dh = d.DistributedHierarchy("ico", 6, 3, agglomerate_below=300)
    plan = d.standard_plan(dh.levels(), d.CycleKind.V, pre, post,
                           smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    for _ in range(2):  # second call: cached graph
        rep = dh.gmg_solve(plan, b, 1e-8, 100)
        ox, ohist, oit, _ = o.solve(b, tol=1e-8, max_cycles=100, pre=pre, post=post)
        assert rep.iterations == oit
        np.testing.assert_array_equal(rep.solution, ox)
        np.testing.assert_allclose(rep.residual_history, ohist, rtol=RTOL)
    plan.cycles = 6
    bp = o.project(b)
    res = dh.run_cycle(plan, bp)
    ox, oh = o.run_cycles(bp, ncycles=6, pre=pre, post=post)
    np.testing.assert_array_equal(res.x, ox)
    np.testing.assert_allclose(res.residual_history, oh, rtol=RTOL)


def test_partitioned_max_cycles_edges():
    """max_cycles 0 (the solution is x0) and 1, and a cap below convergence."""
    h = d.MultigridHierarchy.from_base("ico", 5)
    dh = d.DistributedHierarchy("ico", 5, 2, agglomerate_below=100)
    b = h.make_rhs("uniform", 4)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    for maxc in (0, 1, 3):
        r1 = d.gmg_solve(h, plan, b, 1e-8, maxc)
        r2 = dh.gmg_solve(plan, b, 1e-8, maxc)
        assert r2.iterations == r1.iterations == maxc
        np.testing.assert_array_equal(r2.solution, r1.solution)
        np.testing.assert_allclose(r2.residual_history, r1.residual_history, rtol=RTOL)
        np.testing.assert_allclose(r2.final_relative_residual, r1.final_relative_residual, rtol=RTOL)


def _run_processes(world, base, nsub, nrhs, dirichlet, aggl):
    worker = Path(__file__).resolve().parent / "dist_worker.py"
    with tempfile.TemporaryDirectory(dir="/dev/shm" if os.path.isdir("/dev/shm") else None) as tmp:
        shm = os.path.join(tmp, "halo")
        outs = [os.path.join(tmp, f"r{r}.npz") for r in range(world)]
        procs = [subprocess.Popen([sys.executable, str(worker), shm, str(world), str(r), base, str(nsub), str(nrhs),
                                   "1" if dirichlet else "0", str(aggl), outs[r]],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for r in range(world)]
        logs = []
        for p in procs:
            try:
                logs.append(p.communicate(timeout=600)[0])
            except subprocess.TimeoutExpired:
                for q in procs:
                    q.kill()
                raise
        for p, log in zip(procs, logs):
            assert p.returncode == 0, log
        return [dict(np.load(o, allow_pickle=True)) for o in outs]


@pytest.mark.parametrize("world,base,nsub,nrhs,dirichlet,aggl", [(2, "ico", 6, 1, False, 300),
                                                                  (3, "square", 6, 1, True, 100),
                                                                  (2, "ico", 5, 4, False, 100)])
def test_multiprocess_ranks_bitwise(world, base, nsub, nrhs, dirichlet, aggl):
    """world_size processes, each with its own context and partition on the
    one GPU, host-staged halos: every rank returns the single-GPU iterate
    bit for bit (run_cycle and gmg_solve) and the same cycle counts."""
    outs = _run_processes(world, base, nsub, nrhs, dirichlet, aggl)
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    b = outs[0]["b"]
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 4
    bp = b if dirichlet else h.project_compatible(b)
    r1 = h.run_cycle(plan, bp)
    rep1 = d.gmg_solve(h, plan, b, 1e-8, 100)
    for o in outs:
        assert int(o["ka"]) >= 2 and int(o["halo"]) > 0
        np.testing.assert_array_equal(o["b"], b)
        np.testing.assert_array_equal(o["x"], r1.x)
        np.testing.assert_allclose(o["hist"], r1.residual_history, rtol=RTOL)
        np.testing.assert_array_equal(o["sx"], rep1.solution)
        assert np.asarray(o["it"]).tolist() == rep1.iterations
