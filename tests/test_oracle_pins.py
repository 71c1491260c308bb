"""Pin the CPU oracle (oracle/decmg_oracle.c) to the reference itself.

Every fixture in tests/golden/ was produced by the UNMODIFIED reference
library (oracle/_ref/ref_harness, generator tests/golden/make_golden.py).
The oracle must reproduce the reference bit for bit: mesh hashes
(EmbeddedComplex2D::hash, proj/src/mesh.cpp:112-119), CSR structure and
values of L/P/R (proj/src/operators.cpp:102-122, geometric_map.cpp:205-223,
multigrid.cpp:215), residual histories of run_cycle / gmg_solve
(proj/src/multigrid.cpp:287-323, solvers.cpp:251-279) and the iterates.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle_ctypes import OracleHierarchy, fnv

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(stem):
    return json.loads((GOLDEN / f"{stem}.json").read_text())


def hier_from_argv(argv):
    base, k, bc = argv[1], int(argv[2]), argv[3]
    return OracleHierarchy(base, k, dirichlet=(bc == "dirichlet"))


STRUCT = sorted(p.stem for p in GOLDEN.glob("struct_*.json"))


@pytest.mark.parametrize("stem", STRUCT)
def test_structure_matches_reference(stem):
    g = load(stem)
    h = hier_from_argv(g["_argv"])
    assert h.levels == len(g["levels"])
    for k, lv in enumerate(g["levels"]):
        info = h.info(k)
        assert (info["nv"], info["ne"], info["nt"]) == (lv["nv"], lv["ne"], lv["nt"])
        assert str(info["hash"]) == lv["hash"], f"level {k} mesh hash"
        assert str(fnv(h.get(k, "edges"))) == lv["fnv_edges"]
        assert str(fnv(h.get(k, "triangles"))) == lv["fnv_triangles"]
        assert str(fnv(h.get(k, "positions"))) == lv["fnv_positions"]
        assert str(fnv(h.get(k, "dual_areas"))) == lv["fnv_dual_areas"], f"level {k} dual areas"
        ops = [("L", "L")] + ([("P", "P"), ("R", "R")] if "P" in lv else [])
        for key, name in ops:
            ref = lv[key]
            assert h.info(k)["nnz"] == lv["L"]["nnz"]
            assert str(fnv(h.get(k, name + "_rp"))) == ref["fnv_row_ptr"], f"{key} row_ptr level {k}"
            assert str(fnv(h.get(k, name + "_ci"))) == ref["fnv_col_idx"], f"{key} col_idx level {k}"
            vals = h.get(k, name + "_v")
            if "values" in ref:
                np.testing.assert_array_equal(vals, np.array(ref["values"]))
            assert str(fnv(vals)) == ref["fnv_values"], f"{key} values level {k}"
        if "edges" in lv:
            np.testing.assert_array_equal(h.get(k, "edges"), np.array(lv["edges"]))
            np.testing.assert_array_equal(h.get(k, "triangles"), np.array(lv["triangles"]))
        if "boundary" in lv:
            np.testing.assert_array_equal(h.get(k, "boundary"), np.array(lv["boundary"]))


CYC = sorted(p.stem for p in GOLDEN.glob("cycles_*.json"))
SMOOTHERS = {"jacobi": 0, "gs": 1, "sgs": 2, "cg": 3}  # orc_run_cycles / ref_harness smoother names


@pytest.mark.parametrize("stem", CYC)
def test_cycles_match_reference_bitwise(stem):
    g = load(stem)
    argv = g["_argv"]
    h = hier_from_argv(argv)
    kind, seed, ncyc = argv[4], int(argv[5]), int(argv[6])
    smoother = SMOOTHERS[argv[7]] if len(argv) > 7 else 0
    b = h.rhs(kind, seed)
    if not h.dirichlet:
        b = h.project(b)
    assert str(fnv(b)) == g["fnv_b"]
    x, hist = h.run_cycles(b, ncycles=ncyc, smoother=smoother)
    np.testing.assert_array_equal(hist, np.array(g["history"]))
    assert str(fnv(x)) == g["fnv_x"]


# The oracle restates the default hierarchy (rediscretised, every level, no
# clamp) with a V(2,2) walk; goldens that set HierarchyOptions, use_levels or
# another walk (argv beyond the smoother) are checked against the device path
# directly (tests/test_gpu_parity.py::test_gmg_solve_vs_reference,
# tests/test_gpu_shim.py).
SOLVE = sorted(p.stem for p in GOLDEN.glob("solve_*.json") if len(load(p.stem)["_argv"]) <= 9)


@pytest.mark.parametrize("stem", SOLVE)
def test_gmg_solve_matches_reference_bitwise(stem):
    g = load(stem)
    argv = g["_argv"]
    h = hier_from_argv(argv)
    kind, seed, tol, maxc = argv[4], int(argv[5]), float(argv[6]), int(argv[7])
    smoother = SMOOTHERS[argv[8]] if len(argv) > 8 else 0
    b = h.rhs(kind, seed)
    x, hist, iters, final = h.solve(b, tol=tol, max_cycles=maxc, smoother=smoother)
    assert iters == g["iterations"]
    np.testing.assert_array_equal(hist, np.array(g["history"]))
    assert final == g["final"]
    assert str(fnv(x)) == g["fnv_x"]


PCG = sorted(p.stem for p in GOLDEN.glob("pcg_*.json"))


def w_walk(levels):
    """standard_plan's W walk (multigrid.cpp:149-194, emit_solve with gamma 2)."""
    import paper_2508_12501_b200 as d
    return d.standard_plan(levels, d.CycleKind.W, 1, 1, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi)).walk_string()


@pytest.mark.parametrize("stem", PCG)
def test_pcg_matches_reference_bitwise(stem):
    """gmg_preconditioned_cg: the oracle reproduces the reference's iterations,
    history, final residual and solution bit for bit."""
    g = load(stem)
    argv = g["_argv"]
    h = hier_from_argv(argv)
    kind, seed, ck, pre, post, cyc, tol, maxit = (argv[4], int(argv[5]), argv[6], int(argv[7]), int(argv[8]),
                                                  int(argv[9]), float(argv[10]), int(argv[11]))
    smoother = SMOOTHERS[argv[12]] if len(argv) > 12 else 0
    b = h.rhs(kind, seed)
    walk = w_walk(h.levels) if ck == "W" else None
    x, hist, iters, final = h.pcg(b, tol, maxit, walk=walk, pre=pre, post=post, smoother=smoother, cycles=cyc)
    assert iters == g["iterations"]
    np.testing.assert_array_equal(hist, np.array(g["history"]))
    assert final == g["final"]
    assert str(fnv(x)) == g["fnv_x"]
