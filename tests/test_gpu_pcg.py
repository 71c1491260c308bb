"""GMG-preconditioned CG (gmg_preconditioned_cg, proj/src/solvers.cpp:118-130)
on the GPU against the reference's own PCG runs (tests/golden/pcg_*.json) and
the oracle restatement (oracle/decmg_oracle.c orc_pcg).

The weighted dots are deterministic trees on the device but sequential sums
in the reference. That perturbs alpha and beta at ~1e-16 relative, and the
recursively updated residual carries the perturbation as an absolute error of
~1e-16 ||b||, which is a larger *relative* error once ||r_k|| << ||b||. The
bar: same iteration count (within 1); per-iteration relative residuals within
1e-10 relative or 1e-14 absolute (in units of ||b||, the history's scale);
the solution equal to rounding."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2508_12501_b200 as d
from oracle_ctypes import OracleHierarchy

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
RTOL_HIST = 1e-10
ATOL_HIST = 1e-14
SMOOTHERS = {"jacobi": d.Smoother.WeightedJacobi, "gs": d.Smoother.GaussSeidel,
             "sgs": d.Smoother.SymmetricGaussSeidel}
ORC = {d.Smoother.WeightedJacobi: 0, d.Smoother.GaussSeidel: 1, d.Smoother.SymmetricGaussSeidel: 2}


def inner_plan(levels, kind, pre, post, cycles, smoother="jacobi"):
    plan = d.standard_plan(levels, d.CycleKind.W if kind == "W" else d.CycleKind.V, pre, post,
                           d.SmootherConfig(method=SMOOTHERS[smoother]))
    plan.cycles = cycles
    return plan


def check_history(hist, ref, iters, ref_iters):
    assert abs(iters - ref_iters) <= 1
    m = min(len(hist), len(ref))
    hist, ref = np.asarray(hist[:m]), np.asarray(ref[:m])
    assert np.all(np.abs(hist - ref) <= RTOL_HIST * np.abs(ref) + ATOL_HIST), (hist, ref)


@pytest.mark.parametrize("stem", sorted(p.stem for p in GOLDEN.glob("pcg_*.json")))
def test_pcg_vs_reference(stem):
    g = json.loads((GOLDEN / f"{stem}.json").read_text())
    argv = g["_argv"]
    base, k = argv[1], int(argv[2])
    kind, seed, ck, pre, post, cyc, tol, maxit = (argv[4], int(argv[5]), argv[6], int(argv[7]), int(argv[8]),
                                                  int(argv[9]), float(argv[10]), int(argv[11]))
    smoother = argv[12] if len(argv) > 12 else "jacobi"
    h = d.MultigridHierarchy.from_base(base, k)
    b = h.make_rhs(kind, seed)
    plan = inner_plan(h.levels(), ck, pre, post, cyc, smoother)
    rep = d.gmg_preconditioned_cg(h, plan, b, tol, maxit)
    check_history(rep.residual_history, g["history"], rep.iterations, g["iterations"])
    assert rep.converged == g["converged"]
    if g["converged"]:
        assert rep.final_relative_residual <= 10 * tol
    o = OracleHierarchy(base, k)
    ox, oh, oit, ofin = o.pcg(b, tol, maxit, walk=plan.walk_string() if ck == "W" else None, pre=pre, post=post,
                              smoother=ORC[plan.smoother.method], cycles=cyc)
    if oit == rep.iterations:
        assert np.max(np.abs(rep.solution - ox)) <= 1e-9 * np.max(np.abs(ox))


def test_pcg_batched_lanes_match_single_rhs_oracle():
    base, k, nrhs = "ico", 6, 16
    h = d.MultigridHierarchy.from_base(base, k, max_nrhs=nrhs)
    o = OracleHierarchy(base, k)
    B = h.make_rhs("uniform", 500, nrhs)
    plan = inner_plan(h.levels(), "V", 2, 2, 1)
    rep = d.gmg_preconditioned_cg(h, plan, B, 1e-9, 60)
    for j in range(nrhs):
        ox, oh, oit, _ = o.pcg(B[:, j], 1e-9, 60)
        check_history(rep.residual_history[j], oh, rep.iterations[j], oit)
        assert rep.converged[j]
        if oit == rep.iterations[j]:
            assert np.max(np.abs(rep.solution[:, j] - ox)) <= 1e-9 * np.max(np.abs(ox))


def test_pcg_config3_and_gauss_seidel_inner():
    """config 3 (655 k vertices) with the V(2,2) Jacobi preconditioner, and a
    symmetric Gauss-Seidel W-cycle preconditioner on a smaller sphere."""
    for base, k, ck, sm in [("ico", 8, "V", "jacobi"), ("ico", 5, "W", "sgs")]:
        h = d.MultigridHierarchy.from_base(base, k)
        o = OracleHierarchy(base, k)
        b = h.make_rhs("uniform", 1)
        plan = inner_plan(h.levels(), ck, 2, 2, 1, sm)
        rep = d.gmg_preconditioned_cg(h, plan, b, 1e-8, 100)
        ox, oh, oit, _ = o.pcg(b, 1e-8, 100, walk=plan.walk_string() if ck == "W" else None,
                               smoother=ORC[plan.smoother.method])
        check_history(rep.residual_history, oh, rep.iterations, oit)
        assert rep.converged


def test_pcg_edges():
    h = d.MultigridHierarchy.from_base("ico", 4, max_nrhs=2)
    plan = inner_plan(h.levels(), "V", 2, 2, 1)
    b = h.make_rhs("uniform", 3)
    rep = d.gmg_preconditioned_cg(h, plan, b, 1e-9, 0)  # maxiter 0: initial residual only
    assert rep.iterations == 0 and len(rep.residual_history) == 1 and not rep.converged
    z = d.gmg_preconditioned_cg(h, plan, np.zeros_like(b), 1e-9, 10)  # r0 = 0: converged at once
    assert z.iterations == 0 and z.converged and np.all(z.solution == 0.0)
    hd = d.MultigridHierarchy.from_base("square", 4, dirichlet=True)
    with pytest.raises(ValueError, match="Neumann"):
        d.gmg_preconditioned_cg(hd, inner_plan(hd.levels(), "V", 2, 2, 1), hd.make_rhs("sinsin", 0), 1e-8, 10)
