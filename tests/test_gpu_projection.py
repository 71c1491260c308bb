"""project_compatible (proj/src/multigrid.cpp:240-250) on the device: the
exact parallel evaluation of the reference's sequential mean chain
(csrc/seqsum.cuh) must give the bits of the literal loop
`mean += w[i]*b[i]` -- checked against the oracle's literal loop on inputs that
exercise every branch: ordinary random right-hand sides (mostly the O(1)
segment path), one-signed sums (monotone growth across binades), wide dynamic
range (terms larger than the running sum, binade changes), exact ties on the
running sum's grid (dyadic areas on the flat square), signed zeros and sparse
spikes (zero crossings), and sizes across the 2^20-row pass boundary. The
literal chain (DECMG_PROJ_SEQ=1 path) is the fallback inside every test, and
the fallback counter proves the fast path carried most segments."""
import numpy as np
import pytest

import paper_2508_12501_b200 as d
from oracle_ctypes import OracleHierarchy

pytestmark = pytest.mark.gpu


def crafted(kind, n, nrhs, seed):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.uniform(-1, 1, (n, nrhs))
    if kind == "positive":
        return rng.uniform(0, 1, (n, nrhs))
    if kind == "wide":
        return rng.uniform(-1, 1, (n, nrhs)) * np.ldexp(1.0, rng.integers(-40, 40, (n, nrhs)))
    if kind == "ties":  # short dyadic mantissas: sums round on exact halfway points
        return rng.integers(-1023, 1024, (n, nrhs)).astype(np.float64) * np.ldexp(1.0, rng.integers(-60, 0, (n, nrhs)))
    if kind == "zeros_spikes":
        b = np.where(rng.random((n, nrhs)) < 0.5, -0.0, 0.0)
        m = rng.random((n, nrhs)) < 0.01
        b[m] = rng.uniform(-1e3, 1e3, m.sum())
        b[rng.random((n, nrhs)) < 0.2] = rng.uniform(-1e-12, 1e-12)
        return b
    raise ValueError(kind)


def check(h, o, B):
    B = B.reshape(B.shape[0], -1)
    ref = np.stack([o.project(B[:, j].copy()) for j in range(B.shape[1])], axis=1)
    got = h.project_compatible(B)
    np.testing.assert_array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("base,nsub", [("ico", 6), ("square", 7), ("ico", 1), ("square", 2)])
@pytest.mark.parametrize("kind", ["uniform", "positive", "wide", "ties", "zeros_spikes"])
def test_projection_bit_exact(base, nsub, kind):
    nrhs = 5
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=False, max_nrhs=nrhs)
    o = OracleHierarchy(base, nsub)
    B = crafted(kind, h.n(), nrhs, 7)
    check(h, o, B)
    segs = -(-h.n() // 32) * nrhs
    assert 0 <= h.projection_fallbacks() <= segs


@pytest.mark.parametrize("nrhs", [1, 16, 32])
def test_projection_bit_exact_batches(nrhs):
    h = d.MultigridHierarchy.from_base("ico", 8, max_nrhs=nrhs)
    o = OracleHierarchy("ico", 8)
    B = h.make_rhs("uniform", 3, nrhs)
    check(h, o, B)
    # a random walk of 655 k terms crosses a binade or zero in ~5-15 % of its 32-term
    # records (tools/seqsum_proto.c); the rest take the O(1) path
    segs = -(-h.n() // 32) * nrhs
    assert h.projection_fallbacks() < 0.25 * segs


def test_projection_across_passes_and_solve_staging():
    """icosphere x10 (10.5 M rows: 11 passes of 2^20 rows) through
    project_compatible, and gmg_solve's chunked host staging (16 H2D chunks,
    the chain continued chunk by chunk) gives the same projected RHS: the
    solve's first iterate equals run_cycle's from the oracle-projected RHS."""
    nrhs = 2
    h = d.MultigridHierarchy.from_base("ico", 10, max_nrhs=nrhs)
    o = OracleHierarchy("ico", 10)
    B = h.make_rhs("uniform", 1, nrhs)
    check(h, o, B)
    assert h.projection_fallbacks() < 0.04 * (-(-h.n() // 32) * nrhs)
    Bp = np.stack([o.project(B[:, j].copy()) for j in range(nrhs)], axis=1)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    plan.cycles = 1
    res = h.run_cycle(plan, Bp)
    rep = d.gmg_solve(h, plan, B, 1e-30, 1)
    np.testing.assert_array_equal(rep.solution, res.x)


@pytest.mark.parametrize("pre,post", [(2, 1), (1, 0), (2, 2), (0, 1), (3, 2)])
def test_graph_solve_any_sweep_parity(monkeypatch, pre, post):
    """gmg_solve's device loop (a CUDA graph replaying one captured cycle) is
    used only when a cycle keeps level 0's ping-pong parity; V(2,1), V(1,0),
    ... (an odd number of level-0 Jacobi sweeps) fall back to the host loop.
    Either way: the oracle's cycle count and iterate, history within 1e-10."""
    h = d.MultigridHierarchy.from_base("ico", 5)
    o = OracleHierarchy("ico", 5)
    b = h.make_rhs("uniform", 3)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, pre, post,
                           smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    reps = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("DECMG_GRAPH", flag)
        hh = d.MultigridHierarchy.from_base("ico", 5)
        reps[flag] = [d.gmg_solve(hh, plan, b, 1e-8, 60) for _ in range(2)]  # 2nd call: cached graph
    ox, ohist, oit, _ = o.solve(b, tol=1e-8, max_cycles=60, pre=pre, post=post)
    for rep in reps["1"] + reps["0"]:
        assert rep.iterations == oit
        np.testing.assert_array_equal(rep.solution, ox)
        np.testing.assert_allclose(rep.residual_history, ohist, rtol=1e-10, atol=0)
    del h


@pytest.mark.parametrize("base,nsub,dirichlet,nrhs", [("ico", 7, False, 4), ("square", 6, True, 1)])
def test_solve_batches_equal_single_solves(base, nsub, dirichlet, nrhs):
    """decmg_gpu_solve_batches: each batch of the pipelined stream gives the
    bits of its own gmg_solve (solution, history, cycle counts)."""
    h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    kinds = ["uniform", "lr", "uniform"] if not dirichlet else ["uniform", "sinsin", "lr"]
    batches = [h.make_rhs(k, 10 + i, nrhs) if nrhs > 1 else h.make_rhs(k, 10 + i) for i, k in enumerate(kinds)]
    reps = d.gmg_solve_batches(h, plan, batches, 1e-8, 60)
    for b, rep in zip(batches, reps):
        one = d.gmg_solve(h, plan, b, 1e-8, 60)
        np.testing.assert_array_equal(rep.solution, one.solution)
        assert rep.iterations == one.iterations
        assert rep.residual_history == one.residual_history


def test_device_solve_loop_matches_host_loop(monkeypatch):
    """gmg_solve's device-side loop (a CUDA graph: WHILE over one captured
    cycle with the convergence check and an IF around the rest of the cycle)
    gives the host-driven loop's iterates, histories and cycle counts, also
    when calls with different widths, right-hand sides and plans interleave
    (the graph cache is keyed on them)."""
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("DECMG_GRAPH", flag)
        h = d.MultigridHierarchy.from_base("ico", 7, max_nrhs=8)
        v22 = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
        w11 = d.standard_plan(h.levels(), d.CycleKind.W, 1, 1, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
        out = []
        for plan, kind, nrhs, seed in [(v22, "uniform", 8, 1), (v22, "uniform", 3, 2), (w11, "lr", 8, 3),
                                       (v22, "uniform", 8, 4), (v22, "ylm", 1, 5)]:
            b = h.make_rhs(kind, seed, nrhs) if nrhs > 1 else h.make_rhs(kind, seed)
            rep = d.gmg_solve(h, plan, b, 1e-9, 40)
            out.append((rep.solution, rep.iterations, rep.residual_history))
            plan.cycles = 2
            out.append((h.run_cycle(plan, b).x, None, None))  # flips no state the next solve depends on
        res[flag] = out
    for a, b in zip(res["0"], res["1"]):
        np.testing.assert_array_equal(a[0], b[0])
        assert a[1] == b[1] and a[2] == b[2]


def test_solve_batches_edges():
    """Batch streams: no batches, a cycle cap of 0 (the solution is x0 = 0 and
    the residual is reported) and of 1, and a null right-hand side."""
    h = d.MultigridHierarchy.from_base("ico", 5, max_nrhs=2)
    plan = d.standard_plan(h.levels(), d.CycleKind.V, 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
    assert d.gmg_solve_batches(h, plan, [], 1e-8, 10) == []
    b = h.make_rhs("uniform", 2, 2)
    for cap in (0, 1):
        rep = d.gmg_solve_batches(h, plan, [b, b], 1e-8, cap)
        one = d.gmg_solve(h, plan, b, 1e-8, cap)
        for r in rep:
            np.testing.assert_array_equal(r.solution, one.solution)
            assert r.iterations == one.iterations
            assert r.final_relative_residual == one.final_relative_residual
    import ctypes as C
    from paper_2508_12501_b200.multigrid import _plan_struct
    ps, keep = _plan_struct(plan, h.levels())
    ptrs = (C.c_void_p * 1)(None)
    rc = h._lib.decmg_gpu_solve_batches(h.ctx, C.byref(ps), 2, 1, ptrs, 1e-8, 10, ptrs, None, None, None)
    assert rc == 1  # DECMG_INVALID_ARGUMENT


@pytest.mark.parametrize("base,nsub,dirichlet,nrhs,kind", [("ico", 7, False, 16, "V"), ("ico", 6, False, 5, "W"),
                                                           ("square", 7, True, 1, "F"), ("square", 6, True, 3, "V")])
def test_bottom_of_v_kernel_bitwise(monkeypatch, base, nsub, dirichlet, nrhs, kind):
    """The cooperative bottom-of-V kernel (k_vtail, DECMG_VTAIL=1, default)
    gives the per-pass kernels' iterates bit for bit for V, W and F walks,
    Neumann and Dirichlet, 1-16 right-hand sides, from a threshold that puts
    every level but the finest into it."""
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("DECMG_VTAIL", flag)
        monkeypatch.setenv("DECMG_VTAIL_ITEMS", "100000000")
        h = d.MultigridHierarchy.from_base(base, nsub, dirichlet=dirichlet, max_nrhs=nrhs)
        b = h.make_rhs("uniform", 6, nrhs) if nrhs > 1 else h.make_rhs("uniform", 6)
        if not dirichlet:
            b = h.project_compatible(b)
        plan = d.standard_plan(h.levels(), getattr(d.CycleKind, kind), 2, 2, smoother=d.SmootherConfig(d.Smoother.WeightedJacobi))
        plan.cycles = 3
        res = h.run_cycle(plan, b)
        rep = d.gmg_solve(h, plan, b, 1e-9, 30)
        out[flag] = (res.x, rep.solution, rep.iterations)
    np.testing.assert_array_equal(out["1"][0], out["0"][0])
    np.testing.assert_array_equal(out["1"][1], out["0"][1])
    assert out["1"][2] == out["0"][2]
