"""The reference's own known-answer tests for the path, restated
against both implementations: the CPU oracle (runs everywhere) and the CUDA
library (`-m gpu`). Each case names the reference test it mirrors.

structure : grid / equilateral-grid counts (proj/tests/test_mesh.cpp:151-176),
            subdivision tower 81/289/1089 and the count recurrences
            (test_subdivision.cpp:65-87,167-176), binary^4 = 4,225 and
            cubic^4 = 105,625 (acceptance_main.cpp:91-116), row nnz = 1 + degree
            (test_operators.cpp:193-203), the paper's Laplacian sizes 16,641 /
            115,457 nnz and 4,225 / 29,057 nnz
values    : star1 = 1/sqrt(3) and 1/(2 sqrt(3)) on the equilateral pair, unit axis
            weight and zero diagonal weight on the right-triangle grid
            (test_operators.cpp:116-141), star0^-1 = 2/(s^2 sqrt(3)) and dual-area
            conservation (143-157, test_mesh.cpp:137-149), L 1 = 0 (159-172),
            Laplacian of x^2 + y^2 = 4 on interior rows (174-191), star0-similarity
            symmetry (205-236)
transfers : the worked example's dyadic entries (test_maps.cpp:89-136), constants
            preserved by P and R, restriction row sums = 1 (test_multigrid.cpp:133-149,
            test_maps.cpp:291-317)
"""
import numpy as np
import pytest

from oracle_ctypes import OracleHierarchy

SQ3 = np.sqrt(3.0)


class OracleImpl:
    name = "oracle"

    def __init__(self, base, nsub):
        self.o = OracleHierarchy(base, nsub)
        self.levels = self.o.levels

    def counts(self, k):
        i = self.o.info(k)
        return i["nv"], i["ne"], i["nt"], i["nnz"]

    def csr(self, k, op):
        return (self.o.get(k, f"{op}_rp").astype(np.int64), self.o.get(k, f"{op}_ci").astype(np.int64),
                self.o.get(k, f"{op}_v"))

    def get(self, k, what):
        return self.o.get(k, what)

    def apply(self, k, op, x):
        return self.o.spmv(k, op, x)


class GpuImpl:
    name = "gpu"

    def __init__(self, base, nsub):
        import paper_2508_12501_b200 as d

        self.h = d.MultigridHierarchy.from_base(base, nsub)
        self.levels = self.h.levels()

    def counts(self, k):
        i = self.h.level_info(k)
        return i["nv"], i["ne"], i["nt"], i["nnz_L"]

    def csr(self, k, op):
        return (self.h.export(k, f"{op}_row_ptr").astype(np.int64), self.h.export(k, f"{op}_col_idx").astype(np.int64),
                self.h.export(k, f"{op}_values"))

    def get(self, k, what):
        return self.h.export(k, what)

    def apply(self, k, op, x):
        return self.h.apply(k, op, x)


IMPLS = [pytest.param(OracleImpl, id="oracle"), pytest.param(GpuImpl, id="gpu", marks=pytest.mark.gpu)]


def weights(m, k=0):
    """Per L entry (row i, column j != i): the edge weight |*e|/|e| = L_ij A_i (L = star0^-1 (-d0^T star1 d0):
    off-diagonals +w_e / A_i, diagonal -sum w_e / A_i, operators.cpp:102-122)."""
    rp, ci, v = m.csr(k, "L")
    area = m.get(k, "dual_areas")
    rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    return rows, ci, v * area[rows], area


@pytest.mark.parametrize("impl", IMPLS)
def test_grid_counts(impl):
    for spec, want in (("grid:128:128:1.0:1.0", (16641, 49408, 32768)), ("grid:1:1:1.0:1.0", (4, 5, 2)),
                       ("grid:2:1:1.0:1.0", (6, 9, 4)), ("equi:4:8:1.0", (25, 56, 32))):
        assert impl(spec, 0).counts(0)[:3] == want, spec


@pytest.mark.parametrize("impl", IMPLS)
def test_tower_counts_and_recurrences(impl):
    m = impl("equi:4:8:1.0", 3)
    assert [m.counts(k)[0] for k in range(4)] == [1089, 289, 81, 25]
    for k in range(3, 0, -1):  # fine counts from the coarse ones: V' = V + E, E' = 2E + 3T, T' = 4T
        v, e, t, _ = m.counts(k)
        assert m.counts(k - 1)[:3] == (v + e, 2 * e + 3 * t, 4 * t)
    assert impl("equi:4:8:1.0", 4).counts(0)[0] == 4225
    c = impl("equi:4:8:1.0+cubic", 4)
    assert c.counts(0)[0] == 105625 == 25 * 4225
    v, e, t, _ = c.counts(1)  # cubic: V' = V + 2E + T, E' = 3E + 9T, T' = 9T
    assert c.counts(0)[:3] == (v + 2 * e + t, 3 * e + 9 * t, 9 * t)


@pytest.mark.parametrize("impl", IMPLS)
def test_paper_laplacian_sizes(impl):
    """The paper's figure: 16,641 x 16,641 with 115,457 nonzeros over 4,225 x 4,225 with 29,057 (the unit square
    split into two triangles and subdivided 7 / 6 times; nnz = V + 2E)."""
    m = impl("square", 7)
    assert (m.counts(0)[0], m.counts(0)[3]) == (16641, 115457)
    assert (m.counts(1)[0], m.counts(1)[3]) == (4225, 29057)
    for k in (0, 1):
        v, e, _, nnz = m.counts(k)
        assert nnz == v + 2 * e


@pytest.mark.parametrize("impl", IMPLS)
def test_row_nnz_is_one_plus_degree(impl):
    m = impl("grid:2:2:1.0:1.0", 0)
    rp, _, _ = m.csr(0, "L")
    deg = np.bincount(m.get(0, "edges").ravel(), minlength=rp.size - 1)
    np.testing.assert_array_equal(np.diff(rp), 1 + deg)


@pytest.mark.parametrize("impl", IMPLS)
def test_star1_values(impl):
    m = impl("equi:2:4:1.0", 0)  # equilateral triangles: interior edges 1/sqrt(3), boundary edges half of it
    rows, ci, w, _ = weights(m)
    off = rows != ci
    near = lambda a, b: np.abs(a - b) <= 1e-13 * b
    assert np.all(near(w[off], 1 / SQ3) | near(w[off], 1 / (2 * SQ3)))
    assert near(w[off], 1 / SQ3).any() and near(w[off], 1 / (2 * SQ3)).any()
    g = impl("grid:4:4:4.0:4.0", 0)  # unit cells: interior axis edges weigh 1, cell diagonals 0
    rows, ci, w, _ = weights(g)
    lo, hi, dg = 2 * 5 + 2, 3 * 5 + 2, 3 * 5 + 3
    assert abs(w[(rows == lo) & (ci == hi)][0] - 1.0) <= 1e-13
    assert abs(w[(rows == lo) & (ci == dg)][0]) <= 1e-13


@pytest.mark.parametrize("impl", IMPLS)
def test_star0_hexagonal_cell_and_area_conservation(impl):
    for s in (1.0, 2.0):
        m = impl(f"equi:2:4:{s}", 0)
        rp, _, _ = m.csr(0, "L")
        area = m.get(0, "dual_areas")
        interior = np.diff(rp) == 7  # valence 6
        assert interior.any()
        np.testing.assert_allclose(1.0 / area[interior], 2.0 / (s * s * SQ3), rtol=1e-12)
        # dual cells tile the mesh: 2 x 4 cells of area s * (s sqrt(3)/2) each... summed triangle areas
        ntri = m.counts(0)[2]
        np.testing.assert_allclose(area.sum(), ntri * (SQ3 / 4) * s * s, rtol=1e-12)


@pytest.mark.parametrize("impl", IMPLS)
def test_laplacian_constants_and_quadratic(impl):
    for spec in ("grid:5:4:1.0:1.0", "equi:2:6:0.5"):
        m = impl(spec, 0)
        _, _, v = m.csr(0, "L")
        lap = m.apply(0, "L", np.ones(m.counts(0)[0]))
        assert np.max(np.abs(lap)) <= 1e-12 * max(1.0, np.max(np.abs(v)))
    prev = -1.0
    for n in (8, 16, 32):  # the analytic Laplacian of x^2 + y^2 is 4; interior rows reproduce it to rounding
        m = impl(f"grid:{n}:{n}:1.0:1.0", 0)
        pos = m.get(0, "positions").reshape(-1, 3)
        lap = m.apply(0, "L", pos[:, 0] ** 2 + pos[:, 1] ** 2)
        inner = (pos[:, 0] > 1e-9) & (pos[:, 0] < 1 - 1e-9) & (pos[:, 1] > 1e-9) & (pos[:, 1] < 1 - 1e-9)
        err = np.max(np.abs(lap[inner] - 4.0))
        assert err <= 1e-9
        assert prev < 0 or err <= prev / 1.5 or err <= 4e-10
        prev = err


@pytest.mark.parametrize("impl", IMPLS)
def test_star0_similarity_symmetry(impl):
    m = impl("equi:2:4:1.0", 0)
    rp, ci, v = m.csr(0, "L")
    area = m.get(0, "dual_areas")
    n = rp.size - 1
    S = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    S[rows, ci] = np.sqrt(area[rows]) * v / np.sqrt(area[ci])
    assert np.max(np.abs(S - S.T)) <= 1e-10 * np.max(np.abs(S))
    for seed in range(5):  # the symmetric factor -d0^T star1 d0 = star0 L is negative semidefinite
        x = np.random.default_rng(seed).random(n)
        assert x @ (area * m.apply(0, "L", x)) <= 1e-12


@pytest.mark.parametrize("impl", IMPLS)
def test_transfers(impl):
    m = impl("equi:4:8:1.0", 3)
    for k in range(3):
        nf, nc = m.counts(k)[0], m.counts(k + 1)[0]
        np.testing.assert_allclose(m.apply(k, "P", np.ones(nc)), 1.0, rtol=1e-13)
        np.testing.assert_allclose(m.apply(k, "R", np.ones(nf)), 1.0, rtol=1e-13)
        prp, pci, pv = m.csr(k, "P")
        assert set(np.unique(pv)) <= {0.5, 1.0}  # dyadic, exact: copies and edge midpoints
        np.testing.assert_array_equal(pv[prp[:nc]], 1.0)  # coarse vertices keep their ids: identity rows first
        np.testing.assert_array_equal(pci[prp[:nc]], np.arange(nc))
        rrp, rci, rv = m.csr(k, "R")
        sums = np.add.reduceat(rv, rrp[:-1])
        np.testing.assert_allclose(sums, 1.0, rtol=1e-13)
        # R is P^T with rows scaled to sum 1: entry (i, j) = P_ji / sum_j P_ji
        col_sum = np.bincount(pci, weights=pv, minlength=nc)
        rows = np.repeat(np.arange(nc), np.diff(rrp))
        dense_p = dict(zip(zip(np.repeat(np.arange(nf), np.diff(prp)).tolist(), pci.tolist()), pv.tolist()))
        want = np.array([dense_p[(j, i)] for i, j in zip(rows.tolist(), rci.tolist())]) * (1.0 / col_sum[rows])
        np.testing.assert_array_equal(rv, want)


@pytest.mark.gpu
def test_worked_example_hexagon_to_triangle():
    """One triangle subdivided once (test_maps.cpp:89-136): M = P^T has the dyadic entries of the worked example,
    interpolation gives (a+b)/2 on the midpoints, the full-weighting restriction is R^T = P / 2 (row sums 2)."""
    import paper_2508_12501_b200 as d

    pos = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.5, SQ3 / 2, 0.0]])
    h = d.MultigridHierarchy.from_base((pos, np.array([[0, 1, 2]], dtype=np.int32)), 1)
    prp, pci, pv = (h.export(0, "P_row_ptr"), h.export(0, "P_col_idx"), h.export(0, "P_values"))
    P = np.zeros((6, 3))
    P[np.repeat(np.arange(6), np.diff(prp)), pci] = pv
    np.testing.assert_array_equal(P[:3], np.eye(3))
    assert sorted(map(tuple, P[3:].tolist())) == sorted([(0.5, 0.5, 0.0), (0.5, 0.0, 0.5), (0.0, 0.5, 0.5)])
    a, b, c = 3.0, 5.0, -7.0
    u = h.apply(0, "P", np.array([a, b, c]))
    np.testing.assert_array_equal(u[:3], [a, b, c])
    assert sorted(u[3:].tolist()) == sorted([(a + b) / 2, (b + c) / 2, (c + a) / 2])
    rrp, rci, rv = (h.export(0, "R_row_ptr"), h.export(0, "R_col_idx"), h.export(0, "R_values"))
    R = np.zeros((3, 6))
    R[np.repeat(np.arange(3), np.diff(rrp)), rci] = rv
    np.testing.assert_array_equal(R, P.T / 2)
    np.testing.assert_allclose(h.apply(0, "R", np.ones(6)), 1.0, rtol=1e-13)


# ---- solver known answers (proj/tests/test_multigrid.cpp) --------------------------------------
# The coarse solve is the stand-in for Eigen's SparseLU; these are the reference's
# contract tests at that boundary, which pin tolerances, not bits.

def test_oracle_solver_contracts():
    """zero data stays zero (151-164), two-level exactness with CG as an exact smoother (166-181), one-level
    hierarchy = the direct solve (183-193), V-cycle contraction <= 0.5 for seeds 1-5 and bit-identical reruns
    (195-227), exact preconditioner => PCG in <= 2 iterations (255-265), gmg_solve W(3,3) to 1e-10 (308-317),
    pinned solve: residual <= 1e-12 and weighted mean <= 1e-10 (319-330)."""
    o = OracleHierarchy("equi:4:8:1.0", 2)  # make_test_hierarchy(2): 289 / 81 / 25
    n = o.n()
    x, hist = o.run_cycles(np.zeros(n), np.zeros(n), ncycles=3, pre=3, post=3, smoother=1)
    assert np.all(x == 0.0) and np.all(hist == 0.0)
    for seed in range(1, 6):
        b = o.project(o.rhs("lr", seed))
        x, r = o.run_cycles(b, ncycles=10, pre=2, post=2, smoother=0)
        for k in range(len(r) - 1):
            if r[k] > 1e-10:
                assert r[k + 1] <= 0.5 * r[k]
        x2, r2 = o.run_cycles(b, ncycles=10, pre=2, post=2, smoother=0)
        np.testing.assert_array_equal(r, r2)
        np.testing.assert_array_equal(x, x2)
    two = OracleHierarchy("equi:4:8:1.0", 1)  # fine 81, coarse 25
    b = two.project(two.rhs("lr", 3))
    _, r = two.run_cycles(b, ncycles=1, pre=4 * two.n(), post=4 * two.n(), smoother=3, walk="du")
    assert r[-1] <= 1e-10
    one = OracleHierarchy("equi:4:8:1.0", 0)
    b = one.project(one.rhs("lr", 5))
    _, r = one.run_cycles(b, ncycles=1, pre=3, post=3, smoother=1, walk="")
    assert r[-1] <= 1e-12
    _, hist, it, fin = one.pcg(one.rhs("lr", 7), 1e-9, 30, walk="", pre=3, post=3, smoother=1)
    assert it <= 2 and fin <= 1e-9
    b = o.project(o.rhs("lr", 23))
    _, hist, it, fin = o.solve(b, tol=1e-10, max_cycles=50, pre=3, post=3, smoother=1)  # V here; W below on the GPU
    assert it <= 50 and fin <= 1e-10
    pin = OracleHierarchy("equi:2:4:1.0", 0)
    b = pin.rhs("lr", 29)
    xs = pin.coarse_solve(b)
    area = pin.get(0, "dual_areas")
    bp = pin.project(b)
    res = bp - pin.spmv(0, "L", xs)
    assert np.linalg.norm(res) <= 1e-12 * max(np.linalg.norm(bp), 1e-300)
    assert abs(np.dot(area, xs)) <= 1e-10


@pytest.mark.gpu
def test_gpu_solver_contracts():
    """The same contracts on the CUDA library (the cases test_gpu_parity.py::test_reference_unit_semantics does not
    hold already): two-level exactness with CG smoothers, exact-preconditioner PCG, gmg_solve W(3,3) to 1e-10."""
    import paper_2508_12501_b200 as d

    two = d.MultigridHierarchy.from_base("equi:4:8:1.0", 1)
    n = two.n()
    plan = d.CyclePlan(walk=[d.Transition.Down, d.Transition.Up], pre=[4 * n] * 2, post=[4 * n] * 2,
                       smoother=d.SmootherConfig(d.Smoother.Cg))
    plan.cycles = 1
    b = two.project_compatible(two.make_rhs("lr", 3))
    assert two.run_cycle(plan, b, np.zeros(n)).residual_history[-1] <= 1e-10
    one = d.MultigridHierarchy.from_base("equi:4:8:1.0", 0)
    rep = d.gmg_preconditioned_cg(one, d.standard_plan(1, d.CycleKind.V), one.make_rhs("lr", 7), 1e-9, 30)
    assert rep.converged and rep.iterations <= 2 and rep.final_relative_residual <= 1e-9
    h = d.MultigridHierarchy.from_base("equi:4:8:1.0", 2)
    rep = d.gmg_solve(h, d.standard_plan(h.levels(), d.CycleKind.W, 3, 3), h.project_compatible(h.make_rhs("lr", 23)),
                      1e-10, 50)
    assert rep.converged and rep.final_relative_residual <= 1e-10 and rep.iterations <= 50
