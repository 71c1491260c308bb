"""GPU parity: the CUDA path (through the C ABI) against the reference goldens
and the CPU oracle.

Bars (BASELINE.json north_star): bit-exact integer mesh/connectivity/sparsity;
per-cycle residual norms within 1e-10 relative; same cycle count to 1e-8
(within 1). In addition every row-local kernel (sweep, residual, restriction,
prolongation, SpMV, coarse CG) is bit-identical to the reference, so iterates
from run_cycle on an identical right-hand side must match bit for bit.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2508_12501_b200 as d
from oracle_ctypes import OracleHierarchy, fnv

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
RTOL_HIST = 1e-10


def load(stem):
    return json.loads((GOLDEN / f"{stem}.json").read_text())


def gpu_from_argv(argv, max_nrhs=1):
    base, k, bc = argv[1], int(argv[2]), argv[3]
    return d.MultigridHierarchy.from_base(base, k, dirichlet=(bc == "dirichlet"), max_nrhs=max_nrhs)


EXPORT = {"L": ("L_row_ptr", "L_col_idx", "L_values"), "P": ("P_row_ptr", "P_col_idx", "P_values"),
          "R": ("R_row_ptr", "R_col_idx", "R_values")}


@pytest.mark.parametrize("stem", sorted(p.stem for p in GOLDEN.glob("struct_*.json")))
def test_structure_bit_exact_vs_reference(stem):
    """Mesh hash, edges, triangles, positions, dual areas and the CSR arrays of
    L, P, R built on the device equal the reference's (proj/src/mesh.cpp:112-119,
    operators.cpp:102-122, geometric_map.cpp:205-223)."""
    g = load(stem)
    h = gpu_from_argv(g["_argv"])
    assert h.levels() == len(g["levels"])
    for k, lv in enumerate(g["levels"]):
        info = h.level_info(k)
        assert (info["nv"], info["ne"], info["nt"]) == (lv["nv"], lv["ne"], lv["nt"])
        assert str(h.mesh_hash(k)) == lv["hash"]
        assert str(fnv(h.export(k, "edges"))) == lv["fnv_edges"]
        assert str(fnv(h.export(k, "triangles"))) == lv["fnv_triangles"]
        assert str(fnv(h.export(k, "positions"))) == lv["fnv_positions"]
        assert str(fnv(h.export(k, "dual_areas"))) == lv["fnv_dual_areas"]
        for key in ["L"] + (["P", "R"] if "P" in lv else []):
            rp, ci, v = (h.export(k, n) for n in EXPORT[key])
            assert str(fnv(rp)) == lv[key]["fnv_row_ptr"], (key, k)
            assert str(fnv(ci)) == lv[key]["fnv_col_idx"], (key, k)
            if "values" in lv[key]:
                np.testing.assert_array_equal(v, np.array(lv[key]["values"]))
            assert str(fnv(v)) == lv[key]["fnv_values"], (key, k)


@pytest.mark.parametrize("base,nsub,dirichlet", [("ico", 7, False), ("square", 7, True), ("equi:4:8:1.0", 4, False)])
def test_structure_bit_exact_vs_oracle(base, nsub, dirichlet):
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet)
    o = OracleHierarchy(base, nsub, dirichlet)
    for k in range(h.levels()):
        assert h.mesh_hash(k) == o.info(k)["hash"]
        for ours, theirs in [("edges", "edges"), ("triangles", "triangles"), ("positions", "positions"),
                             ("dual_areas", "dual_areas"), ("boundary", "boundary"), ("L_row_ptr", "L_rp"),
                             ("L_col_idx", "L_ci"), ("L_values", "L_v")]:
            np.testing.assert_array_equal(h.export(k, ours), o.get(k, theirs), err_msg=f"{ours} level {k}")
        if k + 1 < h.levels():
            for ours, theirs in [("P_row_ptr", "P_rp"), ("P_col_idx", "P_ci"), ("P_values", "P_v"),
                                 ("R_row_ptr", "R_rp"), ("R_col_idx", "R_ci"), ("R_values", "R_v")]:
                np.testing.assert_array_equal(h.export(k, ours), o.get(k, theirs), err_msg=f"{ours} level {k}")


def test_spmv_bitwise_equal_to_reference_apply():
    """Mirrors proj/tests/test_kernels.cpp:99-111 (CSR SpMV bitwise-equal)."""
    h = d.MultigridHierarchy.from_base("ico", 6)
    o = OracleHierarchy("ico", 6)
    rng = np.random.default_rng(7)
    for k in range(h.levels()):
        x = rng.random(h.n(k))
        np.testing.assert_array_equal(h.apply(k, "L", x), o.spmv(k, "L", x))
        if k + 1 < h.levels():
            xc = rng.random(h.n(k + 1))
            np.testing.assert_array_equal(h.apply(k, "P", xc), o.spmv(k, "P", xc))
            np.testing.assert_array_equal(h.apply(k, "R", x), o.spmv(k, "R", x))


SMOOTHERS = {"jacobi": d.Smoother.WeightedJacobi, "gs": d.Smoother.GaussSeidel,
             "sgs": d.Smoother.SymmetricGaussSeidel, "cg": d.Smoother.Cg}
ORC_SMOOTHER = {d.Smoother.WeightedJacobi: 0, d.Smoother.GaussSeidel: 1, d.Smoother.SymmetricGaussSeidel: 2,
                d.Smoother.Cg: 3}


def smoother_cfg(name):
    return d.SmootherConfig(method=SMOOTHERS[name])


@pytest.mark.parametrize("stem", sorted(p.stem for p in GOLDEN.glob("cycles_*.json") if not p.stem.endswith("_cg")))
def test_run_cycle_iterates_bitwise_vs_reference(stem):
    """run_cycle (multigrid.cpp:287-323) from the reference's own projected RHS:
    bit-identical iterate, residual history within 1e-10 relative -- weighted
    Jacobi, and (suffix _gs / _sgs) the reference's sequential Gauss-Seidel
    sweeps reproduced by the level-scheduled device sweep."""
    g = load(stem)
    argv = g["_argv"]
    h = gpu_from_argv(argv)
    o = OracleHierarchy(argv[1], int(argv[2]), argv[3] == "dirichlet")
    b = o.rhs(argv[4], int(argv[5]))
    if argv[3] != "dirichlet":
        b = o.project(b)
    assert str(fnv(b)) == g["fnv_b"]
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother_cfg(argv[7] if len(argv) > 7 else "jacobi"))
    plan.cycles = int(argv[6])
    res = h.run_cycle(plan, b, np.zeros_like(b))
    ref = np.array(g["history"])
    assert np.all(np.abs(res.residual_history - ref) <= RTOL_HIST * np.abs(ref))
    assert str(fnv(res.x)) == g["fnv_x"], "iterate not bit-identical to the reference"


@pytest.mark.parametrize("stem", ["solve_config1", "solve_config2", "solve_config3", "solve_equi_4_8_3_lr",
                                  "solve_square_6_uniform", "solve_config2_gs", "solve_config1_sgs",
                                  "solve_ico_cubic_3_ylm", "solve_square_cubic_4_uniform", "solve_levels_used_2",
                                  "solve_levels_used_3", "solve_levels_used_all", "solve_square_dirichlet_levels_used",
                                  "solve_ico_5_clamp", "solve_square_5_gs"])
def test_gmg_solve_vs_reference(stem):
    """gmg_solve (solvers.cpp:251-279) against the reference's own solve: the
    same cycle count to tol, per-cycle residuals within 1e-10 relative and a
    bit-identical solution -- BASELINE configs 1-3, the reference's
    Gauss-Seidel / symmetric Gauss-Seidel smoothers, cubic towers,
    build_hierarchy's use_levels (coarse solves of 625 to 9,409 unknowns on
    the tree-sum grid CG, W-cycles: the paper's levels-used experiment) and
    HierarchyOptions::hodge.clamp_dual_areas."""
    g = load(stem)
    argv = g["_argv"]
    use_levels = int(argv[9]) if len(argv) > 9 else 0
    opt = argv[10] if len(argv) > 10 else "rediscretize"
    kind = {"V": d.CycleKind.V, "W": d.CycleKind.W, "F": d.CycleKind.F}[argv[11] if len(argv) > 11 else "V"]
    pre, post = (int(argv[12]), int(argv[13])) if len(argv) > 13 else (2, 2)
    h = d.MultigridHierarchy.from_base(argv[1], int(argv[2]), dirichlet=argv[3] == "dirichlet",
                                       use_levels=use_levels, clamp_dual_areas="clamp" in opt)
    rhs, seed, tol, maxc = argv[4], int(argv[5]), float(argv[6]), int(argv[7])
    b = h.make_rhs(rhs, seed)
    o = OracleHierarchy(argv[1], int(argv[2]), argv[3] == "dirichlet")
    np.testing.assert_array_equal(b, o.rhs(rhs, seed))
    plan = d.standard_plan(h.levels(), kind, pre, post, smoother_cfg(argv[8] if len(argv) > 8 else "jacobi"))
    rep = d.gmg_solve(h, plan, b, tol, maxc)
    ref = np.array(g["history"])
    assert rep.iterations == g["iterations"]
    hist = np.array(rep.residual_history)
    assert np.all(np.abs(hist - ref) <= RTOL_HIST * np.abs(ref)), (hist, ref)
    assert rep.converged
    assert str(fnv(rep.solution)) == g["fnv_x"], "solution not bit-identical to the reference's"


def test_batched_rhs_match_single_rhs_oracle():
    """16 right-hand sides in one [n][16] batch (config 4 layout) give each
    RHS's single-vector reference history and iterate."""
    base, nsub, nrhs = "ico", 5, 16
    h = d.MultigridHierarchy.from_base(base, nsub, max_nrhs=nrhs)
    o = OracleHierarchy(base, nsub)
    B = h.make_rhs("uniform", 100, nrhs)
    Bp = np.stack([o.project(B[:, j]) for j in range(nrhs)], axis=1)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 6
    res = h.run_cycle(plan, Bp, np.zeros_like(Bp))
    for j in range(nrhs):
        ox, oh = o.run_cycles(Bp[:, j], ncycles=6)
        np.testing.assert_array_equal(res.x[:, j], ox)
        assert np.all(np.abs(res.residual_history[:, j] - oh) <= RTOL_HIST * oh)
    rep = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi)), B, 1e-8, 100)
    for j in range(nrhs):
        ox, oh, oit, _ = o.solve(B[:, j], tol=1e-8, max_cycles=100)
        assert abs(rep.iterations[j] - oit) <= 1
        m = min(oit, rep.iterations[j])
        assert np.all(np.abs(np.array(rep.residual_history[j][:m]) - oh[:m]) <= RTOL_HIST * oh[:m])


def test_w_and_f_walks_bitwise():
    h = d.MultigridHierarchy.from_base("equi:4:8:1.0", 3)
    o = OracleHierarchy("equi:4:8:1.0", 3)
    b = o.project(o.rhs("lr", 11))
    for kind in (d.CycleKind.W, d.CycleKind.F):
        plan = d.standard_plan(h.levels(), kind, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
        plan.cycles = 4
        res = h.run_cycle(plan, b)
        ox, oh = o.run_cycles(b, ncycles=4, walk=plan.walk_string())
        np.testing.assert_array_equal(res.x, ox)
        assert np.all(np.abs(res.residual_history - oh) <= RTOL_HIST * oh)
    # truncated walk that bottoms out above the coarsest level (multigrid.cpp:271-275)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.walk = [d.Transition.Down, d.Transition.Down, d.Transition.Up, d.Transition.Up]
    plan.cycles = 3
    res = h.run_cycle(plan, b)
    ox, oh = o.run_cycles(b, ncycles=3, walk="dduu")
    np.testing.assert_array_equal(res.x, ox)


def test_reference_unit_semantics():
    """Mirrors proj/tests/test_multigrid.cpp: hierarchy shapes (113-131),
    transfers preserve constants (133-149), zero data stays zero (151-164),
    contraction <= 0.5 per cycle for 5 seeds (195-212), bit-identical reruns
    (214-227), one-level hierarchy = coarse solve (183-193)."""
    h = d.MultigridHierarchy.from_base("equi:4:8:1.0", 3)
    assert [h.n(k) for k in range(4)] == [1089, 289, 81, 25]
    for k in range(3):
        np.testing.assert_allclose(h.apply(k, "P", np.ones(h.n(k + 1))), 1.0, rtol=1e-12)
        np.testing.assert_allclose(h.apply(k, "R", np.ones(h.n(k))), 1.0, rtol=1e-12)
    for k in range(4):
        lap = h.apply(k, "L", np.ones(h.n(k)))
        assert np.max(np.abs(lap)) <= 1e-12 * np.max(np.abs(h.export(k, "L_values")))
    plan = d.standard_plan(4, d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 3
    z = np.zeros(h.n())
    res = h.run_cycle(plan, z, z)
    assert np.all(res.x == 0.0) and np.all(res.residual_history == 0.0)
    plan.cycles = 10
    for seed in range(1, 6):
        b = h.project_compatible(h.make_rhs("lr", seed))
        r = h.run_cycle(plan, b).residual_history
        for k in range(len(r) - 1):
            if r[k] > 1e-10:
                assert r[k + 1] <= 0.5 * r[k]
        assert r[-1] <= 1e-6
        r2 = h.run_cycle(plan, b).residual_history
        np.testing.assert_array_equal(r, r2)
    one = d.MultigridHierarchy.from_base("equi:4:8:1.0", 0)
    b = one.project_compatible(one.make_rhs("lr", 5))
    p1 = d.standard_plan(1, d.CycleKind.V, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    r = one.run_cycle(p1, b, np.zeros_like(b)).residual_history
    assert r[-1] <= 1e-12


def test_errors_surface_like_the_reference():
    h = d.MultigridHierarchy.from_base("square", 2)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    bad = d.CyclePlan(walk=[d.Transition.Down, d.Transition.Down, d.Transition.Up], pre=[1] * 3, post=[1] * 3)
    with pytest.raises(ValueError, match="does not return"):
        h.run_cycle(bad, np.zeros(h.n()))
    with pytest.raises(ValueError, match="size mismatch"):
        h.run_cycle(plan, np.zeros(h.n() + 1))
    # zero diagonal -> runtime_error "jacobi: zero diagonal at row i" (multigrid.cpp:47-51)
    lv = [dict(nv=2, L_row_ptr=[0, 1, 2], L_col_idx=[0, 1], L_values=[1.0, 0.0], dual_areas=[1.0, 1.0])]
    lv2 = [dict(nv=2, L_row_ptr=[0, 1, 2], L_col_idx=[0, 1], L_values=[1.0, 0.0], dual_areas=[1.0, 1.0],
                P_row_ptr=[0, 1, 2], P_col_idx=[0, 0], P_values=[1.0, 1.0], R_row_ptr=[0, 2],
                R_col_idx=[0, 1], R_values=[0.5, 0.5]),
           dict(nv=1, L_row_ptr=[0, 1], L_col_idx=[0], L_values=[1.0], dual_areas=[1.0])]
    hz = d.MultigridHierarchy.from_levels(lv2)
    with pytest.raises(RuntimeError, match="jacobi: zero diagonal at row 1"):
        hz.run_cycle(d.standard_plan(2, d.CycleKind.V, 1, 1, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi)), np.ones(2))
    # the default smoother is the reference's Gauss-Seidel (multigrid.hpp:58, multigrid.cpp:29-31)
    with pytest.raises(RuntimeError, match="gauss_seidel: zero diagonal at row 1"):
        hz.run_cycle(d.standard_plan(2, d.CycleKind.V, 1, 1), np.ones(2))
    assert d.MultigridHierarchy.from_levels(lv).levels() == 1
    with pytest.raises(RuntimeError, match="bad corner triple"):
        d.MultigridHierarchy.from_base((np.zeros((3, 3)), np.array([[0, 1, 1]])), 1)


def test_from_levels_matches_from_base():
    """create_from_levels (host-assembled reference layout) runs the same cycles."""
    o = OracleHierarchy("ico", 4)
    levels = []
    for k in range(o.levels):
        lv = dict(nv=o.n(k), L_row_ptr=o.get(k, "L_rp"), L_col_idx=o.get(k, "L_ci"), L_values=o.get(k, "L_v"),
                  dual_areas=o.get(k, "dual_areas"))
        if k + 1 < o.levels:
            lv.update(P_row_ptr=o.get(k, "P_rp"), P_col_idx=o.get(k, "P_ci"), P_values=o.get(k, "P_v"),
                      R_row_ptr=o.get(k, "R_rp"), R_col_idx=o.get(k, "R_ci"), R_values=o.get(k, "R_v"))
        levels.append(lv)
    h = d.MultigridHierarchy.from_levels(levels)
    b = o.project(o.rhs("uniform", 3))
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 5
    res = h.run_cycle(plan, b)
    ox, oh = o.run_cycles(b, ncycles=5)
    np.testing.assert_array_equal(res.x, ox)


@pytest.mark.parametrize("stem,base,nsub,dirichlet", [("fullstruct_config4", "ico", 10, False),
                                                       ("fullstruct_config5a", "square", 12, True),
                                                       ("fullstruct_config5b", "ico", 11, False)])
def test_full_size_structure_bitwise(stem, base, nsub, dirichlet):
    """BASELINE configs 4, 5a, 5b at full size (10.5 M / 16.8 M / 41.9 M
    vertices): every level's mesh hash (EmbeddedComplex2D::hash), dual areas
    and the CSR arrays of L, P, R bit-identical to the oracle's (fixtures from
    tests/golden/make_fullsize.py; the oracle is pinned to the reference), plus
    size-independent properties: L 1 = 0 and P 1 = R 1 = 1 on the finest level."""
    g = json.loads((GOLDEN / f"{stem}.json").read_text())
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet)
    assert h.levels() == len(g["levels"])
    names = {"rp": "row_ptr", "ci": "col_idx", "v": "values"}
    for k, lv in enumerate(g["levels"]):
        info = h.level_info(k)
        assert (info["nv"], info["ne"], info["nt"]) == (lv["nv"], lv["ne"], lv["nt"])
        assert h.mesh_hash(k) == int(lv["hash"])
        assert fnv(h.export(k, "dual_areas")) == int(lv["dual_areas"])
        for key, want in lv.items():
            if key[:2] in ("L_", "P_", "R_"):
                assert fnv(h.export(k, f"{key[0]}_{names[key[2:]]}")) == int(want), (k, key)
    n = h.n()
    one = np.ones(n)
    lap = h.apply(0, "L", one)
    if not dirichlet:
        assert np.max(np.abs(lap)) <= 1e-9 * np.max(np.abs(h.export(0, "L_values")))
    np.testing.assert_allclose(h.apply(0, "P", np.ones(h.n(1))), 1.0, rtol=1e-15)
    np.testing.assert_allclose(h.apply(0, "R", one), 1.0, rtol=1e-13)


@pytest.mark.parametrize("nrhs", [2, 3, 5, 32])
def test_odd_batch_widths_bitwise(nrhs):
    """Every thread mapping (scalar lanes for non-power-of-two batches, 2- and
    4-wide vector lanes) gives each RHS its single-vector reference iterate."""
    base, nsub = "ico", 4
    h = d.MultigridHierarchy.from_base(base, nsub, max_nrhs=nrhs)
    o = OracleHierarchy(base, nsub)
    B = np.stack([o.project(o.rhs("uniform", 40 + j)) for j in range(nrhs)], axis=1)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 3
    res = h.run_cycle(plan, B)
    for j in range(nrhs):
        ox, oh = o.run_cycles(B[:, j], ncycles=3)
        np.testing.assert_array_equal(res.x[:, j], ox)
        assert np.all(np.abs(res.residual_history[:, j] - oh) <= RTOL_HIST * oh)


def test_warm_start_and_cycle_cap():
    """x0 warm start (gmg_solve's optional x0, solvers.cpp:251-258), the cycle
    cap (max_cycles hit: not converged) and max_cycles = 0 (the solution is x0)."""
    base, nsub = "ico", 5
    h = d.MultigridHierarchy.from_base(base, nsub)
    o = OracleHierarchy(base, nsub)
    b = o.rhs("uniform", 8)
    x0 = np.random.default_rng(1).uniform(-1, 1, h.n())
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    bp = o.project(b)
    plan.cycles = 3
    res = h.run_cycle(plan, bp, x0)
    ox, oh = o.run_cycles(bp, x0=x0, ncycles=3)
    np.testing.assert_array_equal(res.x, ox)
    rep = d.gmg_solve(h, plan, b, 1e-30, 4)
    assert rep.iterations == 4 and not rep.converged
    rep0 = d.gmg_solve(h, plan, b, 1e-8, 0, x0=x0)
    assert rep0.iterations == 0
    np.testing.assert_array_equal(rep0.solution, x0)


def test_w_cycle_solve_and_one_level_solve():
    """gmg_solve with a W-cycle plan and on a one-level hierarchy (the coarse
    CG alone, multigrid.cpp:312-313)."""
    h = d.MultigridHierarchy.from_base("equi:4:8:1.0", 3)
    o = OracleHierarchy("equi:4:8:1.0", 3)
    b = o.rhs("lr", 23)
    plan = d.standard_plan(h.levels(), d.CycleKind.W, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    rep = d.gmg_solve(h, plan, b, 1e-10, 50)
    assert rep.converged
    bp = o.project(b)
    ox, oh = o.run_cycles(bp, ncycles=rep.iterations, walk=plan.walk_string())
    np.testing.assert_array_equal(rep.solution, ox)
    one = d.MultigridHierarchy.from_base("equi:4:8:1.0", 0)
    rep1 = d.gmg_solve(one, d.standard_plan(1, d.CycleKind.V, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi)), one.make_rhs("lr", 5), 1e-12, 3)
    assert rep1.iterations == 1 and rep1.final_relative_residual <= 1e-12


def test_setup_errors_match_reference_messages():
    """Non-well-centred dual cell (operators.cpp:88-98) and degenerate triangle
    (geometry.cpp:11-13) raise runtime_error with the reference's message."""
    P = np.array([[0, 0, 0], [1, 0, 0], [0.5, 0.1, 0], [0.5, -0.1, 0]], float)
    with pytest.raises(RuntimeError, match="non-well-centered dual cell at vertex 0"):
        d.MultigridHierarchy.from_base((P, np.array([[0, 1, 2], [0, 3, 1]])), 0)
    Q = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
    with pytest.raises(RuntimeError, match="circumcenter: degenerate triangle"):
        d.MultigridHierarchy.from_base((Q, np.array([[0, 1, 2]])), 0)


@pytest.mark.parametrize("env", [{"DECMG_KERNEL": "ell"}, {"DECMG_KERNEL": "pipe"}, {"DECMG_PF": "0"},
                                 {"DECMG_RPT": "2"}, {"DECMG_VTAIL": "0"}])
@pytest.mark.parametrize("base,nsub,dirichlet,nrhs", [("ico", 6, False, 16), ("square", 6, True, 1)])
def test_kernel_variants_bitwise(monkeypatch, env, base, nsub, dirichlet, nrhs):
    """Every kernel switch (high-occupancy or pipelined row kernel for every
    operator, no prefetch, 2 RHS per thread, per-pass kernels instead of the
    bottom-of-V kernel) gives the reference iterate bit for bit. The switches
    are read at context creation."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    o = OracleHierarchy(base, nsub, dirichlet)
    if nrhs == 1:
        B = o.rhs("sinsin" if dirichlet else "uniform", 5)[:, None]
    else:
        B = h.make_rhs("uniform", 40, nrhs)
    if not dirichlet:
        B = np.stack([o.project(B[:, j]) for j in range(nrhs)], axis=1)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 3
    res = h.run_cycle(plan, B if nrhs > 1 else B[:, 0])
    x = res.x if nrhs > 1 else res.x[:, None]
    for j in range(nrhs):
        ox, oh = o.run_cycles(B[:, j], ncycles=3)
        np.testing.assert_array_equal(x[:, j], ox)


@pytest.mark.parametrize("smoother", ["gs", "sgs"])
@pytest.mark.parametrize("base,nsub,dirichlet,nrhs", [("ico", 7, False, 16), ("square", 7, True, 1),
                                                      ("equi:4:8:1.0", 4, False, 3)])
def test_gauss_seidel_bitwise_vs_oracle(smoother, base, nsub, dirichlet, nrhs):
    """Level-scheduled Gauss-Seidel (forward and symmetric) against the
    oracle's sequential sweep at 164 k vertices, batched and Dirichlet; the
    schedule has a handful of phases per level (setup.cu build_gs_schedule)."""
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    o = OracleHierarchy(base, nsub, dirichlet)
    if nrhs == 1:
        B = o.rhs("sinsin" if dirichlet else "uniform", 3)[:, None]
    else:
        B = h.make_rhs("uniform", 70, nrhs)
    if not dirichlet:
        B = np.stack([o.project(B[:, j]) for j in range(nrhs)], axis=1)
    cfg = smoother_cfg(smoother)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 1, 1, cfg)
    plan.cycles = 3
    res = h.run_cycle(plan, B if nrhs > 1 else B[:, 0])
    x = res.x if nrhs > 1 else res.x[:, None]
    hist = res.residual_history if nrhs > 1 else res.residual_history[:, None]
    for j in range(nrhs):
        ox, oh = o.run_cycles(B[:, j], ncycles=3, pre=1, post=1, smoother=ORC_SMOOTHER[cfg.method])
        np.testing.assert_array_equal(x[:, j], ox)
        assert np.all(np.abs(hist[:, j] - oh) <= RTOL_HIST * oh)
    # W walk with Gauss-Seidel on every level
    plan = d.standard_plan(h.levels(), d.CycleKind.W, 2, 1, cfg)
    plan.cycles = 2
    res = h.run_cycle(plan, B[:, 0] if nrhs == 1 else B)
    x = res.x if nrhs > 1 else res.x[:, None]
    ox, _ = o.run_cycles(B[:, 0], ncycles=2, pre=2, post=1, smoother=ORC_SMOOTHER[cfg.method],
                         walk=plan.walk_string())
    np.testing.assert_array_equal(x[:, 0], ox)


def test_partitioned_solve_rejects_gauss_seidel():
    dh = d.DistributedHierarchy("ico", 4, 2)
    plan = d.standard_plan(dh.levels(), d.CycleKind.V, 2, 2, smoother_cfg("gs"))
    plan.cycles = 1
    b = np.zeros(dh.context().n())
    with pytest.raises(ValueError, match="only the weighted Jacobi"):
        dh.run_cycle(plan, b)


@pytest.mark.parametrize("base,nsub,dirichlet", [("ico+cubic", 4, False), ("square+cubic", 5, True),
                                                  ("equi:4:8:1.0+cubic", 3, False)])
def test_cubic_hierarchy_vs_oracle(base, nsub, dirichlet):
    """SubdivisionScheme::Cubic (1 -> 9) towers up to 66 k vertices: structure,
    transfers and V(2,2) iterates bit-identical to the oracle (which is pinned
    to the reference's cubic goldens)."""
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet)
    o = OracleHierarchy(base, nsub, dirichlet)
    assert h.levels() == o.levels
    for k in range(h.levels()):
        assert h.mesh_hash(k) == o.info(k)["hash"]
        for op, names in EXPORT.items():
            if op != "L" and k == h.levels() - 1:
                continue
            oname = {"L": ("L_rp", "L_ci", "L_v"), "P": ("P_rp", "P_ci", "P_v"), "R": ("R_rp", "R_ci", "R_v")}[op]
            for gn, on in zip(names, oname):
                np.testing.assert_array_equal(h.export(k, gn), o.get(k, on))
    b = o.rhs("sinsin" if dirichlet else "uniform", 9)
    if not dirichlet:
        b = o.project(b)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 3
    res = h.run_cycle(plan, b)
    ox, oh = o.run_cycles(b, ncycles=3)
    np.testing.assert_array_equal(res.x, ox)
    assert np.all(np.abs(res.residual_history - oh) <= RTOL_HIST * oh)


@pytest.mark.parametrize("stem", sorted(p.stem for p in GOLDEN.glob("*_cg.json")))
def test_cg_smoother_vs_reference(stem):
    """Smoother::Cg (cg_fixed, multigrid.cpp:63-91): its weighted dots are
    trees on the device and sequential sums in the reference, so iterates agree
    to rounding, not bit for bit: histories within 1e-10 relative (or 1e-14
    absolute, in units of ||b||), same cycle count, solutions to 1e-9."""
    g = load(stem)
    argv = g["_argv"]
    h = gpu_from_argv(argv)
    o = OracleHierarchy(argv[1], int(argv[2]), argv[3] == "dirichlet")
    cfg = smoother_cfg("cg")
    if argv[0] == "cycles":
        b = o.rhs(argv[4], int(argv[5]))
        if argv[3] != "dirichlet":
            b = o.project(b)
        plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, cfg)
        plan.cycles = int(argv[6])
        res = h.run_cycle(plan, b)
        hist, x = res.residual_history, res.x
        ox, _ = o.run_cycles(b, ncycles=plan.cycles, smoother=3)
    else:
        kind, seed, tol, maxc = argv[4], int(argv[5]), float(argv[6]), int(argv[7])
        b = h.make_rhs(kind, seed)
        rep = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, cfg), b, tol, maxc)
        assert abs(rep.iterations - g["iterations"]) <= 1
        hist, x = np.array(rep.residual_history), rep.solution
        ox, _, oit, _ = o.solve(b, tol=tol, max_cycles=maxc, smoother=3)
        if oit != rep.iterations:
            ox = None
    ref = np.array(g["history"])
    m = min(len(ref), len(hist))
    assert np.all(np.abs(hist[:m] - ref[:m]) <= RTOL_HIST * np.abs(ref[:m]) + 1e-14), (hist, ref)
    if ox is not None:
        assert np.max(np.abs(x - ox)) <= 1e-9 * np.max(np.abs(ox))


@pytest.mark.parametrize("graph", ["1", "0"])
def test_nonfinite_residual_guard(monkeypatch, graph):
    """A NaN/Inf residual stops gmg_solve with DECMG_RUNTIME after the first
    cycle (single-GPU graph and host loops, and the partitioned solve);
    run_cycle just reports it in the history, like the reference."""
    monkeypatch.setenv("DECMG_GRAPH", graph)
    h = d.MultigridHierarchy.from_base("ico", 4)
    jac = d.SmootherConfig(d.Smoother.WeightedJacobi)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=jac)
    for bad in (np.nan, np.inf):
        b = h.make_rhs("uniform", 1)
        b[17] = bad
        with pytest.raises(RuntimeError, match="non-finite residual"):
            d.gmg_solve(h, plan, b, 1e-8, 50)
        plan.cycles = 2
        res = h.run_cycle(plan, b)
        assert not np.all(np.isfinite(res.residual_history))
    dh = d.DistributedHierarchy("ico", 4, 2, agglomerate_below=100)
    b = h.make_rhs("uniform", 1)
    b[3] = np.nan
    with pytest.raises(RuntimeError, match="non-finite residual"):
        dh.gmg_solve(plan, b, 1e-8, 50)
    # a healthy lane of a batch still converges; the batch call reports the bad lane
    h2 = d.MultigridHierarchy.from_base("ico", 4, max_nrhs=2)
    B = h2.make_rhs("uniform", 1, 2)
    B[5, 1] = np.inf
    with pytest.raises(RuntimeError, match="right-hand side 1"):
        d.gmg_solve(h2, plan, B, 1e-8, 50)
