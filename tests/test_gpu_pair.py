"""Two Jacobi sweeps per pass (csrc/rowkernels.cuh k_sweep_pair; smooth =
jacobi_sweep twice, proj/src/multigrid.cpp:36-56,95-120): the pass hands the
intermediate iterate from sweep 1 to sweep 2 through L2, round by round, with
the rows whose neighbours lie past their round's horizon deferred to the end.
Every row is the arithmetic of a separate sweep, so iterates must be
bit-identical to a context that runs one sweep per launch (DECMG_PAIR=0) -- on
meshes small enough that rounds are ragged (CTAs without tiles in the last
round), with one and with sixteen right-hand sides, for walks that mix paired
and single sweeps, with the residual norm fused into the first pair, and
through gmg_solve's device loop. Residual histories agree to rounding (the
norm partials are summed per CTA, and the tile-to-CTA map differs)."""
import os

import numpy as np
import pytest

import paper_2508_12501_b200 as d

pytestmark = pytest.mark.gpu

JAC = d.SmootherConfig(d.Smoother.WeightedJacobi)


def hierarchy(env, *a, **kw):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return d.MultigridHierarchy.from_base(*a, **kw)  # the switches are read at context creation
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


PAIRED = [
    {"DECMG_PAIR": "1", "DECMG_PAIR_MIN_ROUNDS": "2", "DECMG_PAIR_GROUP": "1"},
    {"DECMG_PAIR": "1", "DECMG_PAIR_MIN_ROUNDS": "2", "DECMG_PAIR_GROUP": "1", "DECMG_PAIR_AHEAD": "1"},
    {"DECMG_PAIR": "1", "DECMG_PAIR_MIN_ROUNDS": "2", "DECMG_PAIR_GROUP": "3"},
]


@pytest.mark.parametrize("base,nsub,dirichlet,nrhs", [("ico", 6, False, 16), ("ico", 7, False, 16),
                                                      ("ico", 8, False, 1), ("square", 9, True, 1),
                                                      ("square", 8, True, 4), ("ico", 7, False, 5),
                                                      ("ico", 6, False, 32), ("equi:24:48:1.0", 4, False, 2)])
@pytest.mark.parametrize("pre,post", [(2, 2), (3, 2), (2, 1), (4, 5)])
def test_pair_iterates_bitwise(base, nsub, dirichlet, nrhs, pre, post):
    h0 = hierarchy({"DECMG_PAIR": "0"}, base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    kind = "sinsin" if dirichlet else "uniform"
    b = h0.make_rhs(kind, 3, nrhs) if nrhs > 1 else h0.make_rhs(kind, 3)
    if not dirichlet:
        b = h0.project_compatible(b)
    plan = d.standard_plan(h0.levels(), d.CycleKind.V, pre, post, smoother=JAC)
    plan.cycles = 3
    ref = h0.run_cycle(plan, b)
    for env in PAIRED:
        h1 = hierarchy(env, base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
        got = h1.run_cycle(plan, b)
        np.testing.assert_array_equal(got.x.view(np.uint64), ref.x.view(np.uint64), err_msg=str(env))
        np.testing.assert_allclose(got.residual_history, ref.residual_history, rtol=1e-12, err_msg=str(env))
        del h1


@pytest.mark.parametrize("kindc", [d.CycleKind.W, d.CycleKind.F])
def test_pair_w_f_walks_bitwise(kindc):
    h0 = hierarchy({"DECMG_PAIR": "0"}, "ico", 6, max_nrhs=16)
    b = h0.project_compatible(h0.make_rhs("uniform", 5, 16))
    plan = d.standard_plan(h0.levels(), kindc, 2, 2, smoother=JAC)
    plan.cycles = 2
    ref = h0.run_cycle(plan, b)
    h1 = hierarchy(PAIRED[0], "ico", 6, max_nrhs=16)
    got = h1.run_cycle(plan, b)
    np.testing.assert_array_equal(got.x.view(np.uint64), ref.x.view(np.uint64))


@pytest.mark.parametrize("pre,post", [(2, 2), (2, 1), (3, 3)])
@pytest.mark.parametrize("base,nsub,dirichlet,nrhs", [("ico", 7, False, 16), ("square", 9, True, 1)])
def test_pair_gmg_solve(base, nsub, dirichlet, nrhs, pre, post):
    """gmg_solve (solvers.cpp:251-279) with the fused norm inside the first pair: same cycle counts, bit-identical
    solutions, histories to rounding; graph replays included (two solves per context). V(2,1) flips level 0's
    ping-pong parity every cycle, so it runs the host-driven loop with its early exit after the pair."""
    h0 = hierarchy({"DECMG_PAIR": "0"}, base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    h1 = hierarchy(PAIRED[0], base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    kind = "sinsin" if dirichlet else "uniform"
    b = h0.make_rhs(kind, 11, nrhs) if nrhs > 1 else h0.make_rhs(kind, 11)
    plan = d.standard_plan(h0.levels(), d.CycleKind.V, pre, post, smoother=JAC)
    for _ in range(2):
        r0 = d.gmg_solve(h0, plan, b, 1e-8, 100)
        r1 = d.gmg_solve(h1, plan, b, 1e-8, 100)
        assert np.array_equal(np.asarray(r0.iterations), np.asarray(r1.iterations))
        np.testing.assert_array_equal(r1.solution.view(np.uint64), r0.solution.view(np.uint64))
        if nrhs == 1:
            np.testing.assert_allclose(r1.residual_history, r0.residual_history, rtol=1e-10)
        else:
            for a, bb in zip(r1.residual_history, r0.residual_history):
                np.testing.assert_allclose(a, bb, rtol=1e-10)
