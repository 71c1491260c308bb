"""The C++ drop-in shim (include/decmg_gpu.hpp) driven by compiled C++ callers
on the GPU, against the reference's goldens and the oracle.

* tests/cpp/shim_standalone.cpp (compiled here with g++ against include/ and
  libdecmg_gpu.so): BASELINE config 2 through the shim's own constructor,
  gmg_solve, SolveReport::cumulative_seconds / write_residual_csv, smooth()
  and the level operators' apply() -- reproduces tests/golden/solve_config2.json
  (the reference's own run) and the oracle's sweeps bit for bit.
* oracle/_ref/shim_reference (built by `make -C oracle shim` where
  /root/reference exists; it links the reference's mesh and subdivision code):
  a reference caller that keeps the reference's own EmbeddedComplex2D /
  subdivision_tower / build_hierarchy(base, tower, use_levels, opts) and
  swaps multigrid.hpp + solvers.hpp for the shim.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2508_12501_b200 as d
from paper_2508_12501_b200 import _lib
from oracle_ctypes import OracleHierarchy, fnv

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"


def _build_standalone():
    exe = ROOT / "build" / "shim_standalone"
    exe.parent.mkdir(exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "shim_standalone.cpp"), "-o", str(exe),
                    "-L", str(_lib.LIB_PATH.parent), "-ldecmg_gpu", f"-Wl,-rpath,{_lib.LIB_PATH.parent}"],
                   check=True)
    return exe


def test_cpp_caller_reproduces_reference_config2(tmp_path):
    exe = _build_standalone()
    csv = tmp_path / "res.csv"
    run = subprocess.run([str(exe), str(csv)], capture_output=True, text=True)
    assert run.returncode == 0, run.stderr
    out = json.loads(run.stdout)
    g = json.loads((GOLDEN / "solve_config2.json").read_text())
    assert out["n"] == g["n"] == 40962
    assert out["iterations"] == g["iterations"]
    np.testing.assert_allclose(out["history"], g["history"], rtol=1e-10, atol=0)
    assert out["fnv_x"] == g["fnv_x"], "solution differs from the reference's"
    assert out["converged"] and out["shape_error"] and out["times_ok"]
    lines = csv.read_text().splitlines()
    assert lines[0] == "cycle,rel_residual,cumulative_seconds" and len(lines) == out["iterations"] + 1
    # apply() and smooth() against the oracle, bit for bit
    o = OracleHierarchy("ico", 6)
    b = o.rhs("ylm", 1)
    bc = o.project(b)
    assert int(out["fnv_Lb"]) == fnv(o.spmv(0, "L", bc))
    assert int(out["fnv_gs2"]) == fnv(o.smooth(0, bc, np.zeros_like(bc), 2, smoother=1))
    b1 = o.spmv(0, "R", bc)
    assert int(out["fnv_jac3_l1"]) == fnv(o.smooth(1, b1, np.zeros_like(b1), 3, smoother=0))


@pytest.mark.parametrize("smoother,code", [("GaussSeidel", 1), ("SymmetricGaussSeidel", 2), ("WeightedJacobi", 0)])
def test_python_smooth_matches_oracle(smoother, code):
    """smooth() (multigrid.cpp:95-120) on every level's operator, 1 and 3 sweeps."""
    h = d.MultigridHierarchy.from_base("ico", 5)
    o = OracleHierarchy("ico", 5)
    cfg = d.SmootherConfig(getattr(d.Smoother, smoother))
    for k in range(h.levels()):
        n = o.n(k)
        rng = np.random.default_rng(k)
        b = rng.uniform(-1, 1, n)
        x0 = rng.uniform(-1, 1, n)
        for it in (1, 3):
            np.testing.assert_array_equal(d.smooth(h, k, x0, b, cfg, it), o.smooth(k, b, x0, it, smoother=code))


@pytest.mark.parametrize("graph", ["1", "0"])
def test_cumulative_seconds_filled(monkeypatch, graph):
    """SolveReport::cumulative_seconds (solvers.cpp:269): one entry per cycle,
    nondecreasing, from the device clock (graph loop) or the host (host loop)."""
    monkeypatch.setenv("DECMG_GRAPH", graph)
    h = d.MultigridHierarchy.from_base("ico", 6)
    b = h.make_rhs("uniform", 3)
    jac = d.SmootherConfig(d.Smoother.WeightedJacobi)
    for _ in range(2):
        rep = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=jac), b, 1e-8, 100)
        t = rep.cumulative_seconds
        assert len(t) == rep.iterations and all(b2 >= a for a, b2 in zip(t, t[1:])) and t[0] > 0
    rep = d.gmg_preconditioned_cg(h, d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=jac), b, 1e-9, 50)
    assert len(rep.cumulative_seconds) == rep.iterations + 1


def test_cpp_reference_caller():
    exe = ROOT / "oracle" / "_ref" / "shim_reference"
    if not exe.exists():
        pytest.skip("oracle/_ref/shim_reference not built (needs /root/reference at build time)")
    out = json.loads(subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout)
    for case in out["cases"]:
        g = json.loads((GOLDEN / f"{case['golden']}.json").read_text())
        assert case["n"] == g["n"], case["golden"]
        assert case["iterations"] == g["iterations"], case["golden"]
        np.testing.assert_allclose(case["history"], g["history"], rtol=1e-10, atol=0, err_msg=case["golden"])
        assert case["fnv_x"] == g["fnv_x"], case["golden"]
        assert case["path"] == case["expect_path"], case
