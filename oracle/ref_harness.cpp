// TEST INFRASTRUCTURE ONLY (oracle). Harness around the UNMODIFIED reference
// library compiled from /root/reference/proj/src (see oracle/Makefile). It
// produces golden vectors that pin oracle/decmg_oracle.c (tests/golden/) and
// times the reference's CPU solver for bench.py's reference arm.
//
// Everything here calls the reference's own public API:
//   make_triangulated_grid / make_equilateral_grid  proj/src/mesh.cpp:232-291
//   EmbeddedComplex2D::from_triangles               proj/src/mesh.cpp:122-157
//   binary_subdivide / subdivision_tower            proj/src/subdivision.cpp:114-139
//   build_hierarchy / MultigridHierarchy            proj/src/multigrid.cpp:196-341
//   run_cycle / project_compatible                  proj/src/multigrid.cpp:240-323
//   gmg_solve                                       proj/src/solvers.cpp:251-279
//   smooth / SparseOperator::apply                  proj/src/multigrid.cpp:95-120, sparse.cpp:209-218
// The BASELINE extensions are harness code only:
//   x1 Dirichlet mask  -> dirichlet_cycle() below (a copy of the cycle_once walk
//                         with identity boundary rows; the reference has no BCs)
//   x2 icosahedron + projected binary subdivision -> ico_base(), projected_tower()
//   x3 RHS generators -> make_rhs()
#include "decmg/geometric_map.hpp"
#include "decmg/kernels.hpp"
#include "decmg/mesh.hpp"
#include "decmg/multigrid.hpp"
#include "decmg/operators.hpp"
#include "decmg/rng.hpp"
#include "decmg/solvers.hpp"
#include "decmg/subdivision.hpp"

#include <omp.h>

#include "ref_cases.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace decmg {
std::vector<double> standin_coarse_cg(const SparseOperator& A, const std::vector<double>& w,
                                      const std::vector<double>& b, bool project);
}

using namespace decmg;
using refcases::Case;
using refcases::ico_base;
using refcases::make_case;
using refcases::projected_subdivide;
using refcases::tower_of;

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

std::uint64_t fnv(const void* data, std::size_t n, std::uint64_t h = 1469598103934665603ULL) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}
template <class T>
std::uint64_t fnv_vec(const std::vector<T>& v) {
    return fnv(v.data(), v.size() * sizeof(T));
}

// ico_base, projected_subdivide, Case, make_case, tower_of: oracle/ref_cases.hpp

// ---- extension x3: RHS generators --------------------------------
std::vector<double> make_rhs(const std::string& kind, const EmbeddedComplex2D& m,
                             const SparseOperator& L, std::uint64_t seed,
                             const std::vector<char>* boundary) {
    const int n = m.num_vertices();
    std::vector<double> b(n, 0.0);
    if (kind == "uniform") {
        std::mt19937_64 rng(seed);
        for (int i = 0; i < n; ++i) b[i] = 2.0 * uniform01(rng) - 1.0;
    } else if (kind == "lr") {  // proj/src/physics.cpp:50-53
        b = L.apply(uniform01_vector(seed, n));
    } else if (kind == "ylm") {
        std::mt19937_64 rng(seed);
        std::vector<double> g(n);
        for (int i = 0; i < n; i += 2) {
            const double u1 = uniform01(rng);
            const double u2 = uniform01(rng);
            const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
            const double th = 2.0 * M_PI * u2;
            g[i] = rad * std::cos(th);
            if (i + 1 < n) g[i + 1] = rad * std::sin(th);
        }
        const double c = 0.25 * std::sqrt(105.0 / M_PI);
        for (int i = 0; i < n; ++i) {
            const Vec3& p = m.positions[i];
            b[i] = c * ((p.x * p.x - p.y * p.y) * p.z) + 1e-3 * g[i];
        }
    } else if (kind == "sinsin") {
        for (int i = 0; i < n; ++i) {
            const Vec3& p = m.positions[i];
            const double f = ((2.0 * M_PI * M_PI) * std::sin(M_PI * p.x)) * std::sin(M_PI * p.y);
            b[i] = -f;
        }
    } else {
        throw std::invalid_argument("unknown rhs " + kind);
    }
    if (boundary) {
        for (int i = 0; i < n; ++i)
            if ((*boundary)[i]) b[i] = 0.0;
    }
    return b;
}

// ---- extension x1: Dirichlet mask --------------------------------------------
std::vector<char> boundary_of(const EmbeddedComplex2D& m) {
    std::vector<char> bd(m.num_vertices(), 0);
    const auto& et = m.triangles_of_edge();
    for (int e = 0; e < m.num_edges(); ++e) {
        if (et[e].size() == 1) {
            bd[m.edge_src(e)] = 1;
            bd[m.edge_tgt(e)] = 1;
        }
    }
    return bd;
}

// Identity rows at boundary vertices; the off-diagonals stay as structural
// zeros so the sparsity is unchanged.
SparseOperator dirichlet_rows(const SparseOperator& L, const std::vector<char>& bd) {
    std::vector<int> ri, ci;
    std::vector<double> v;
    for (int j = 0; j < L.cols(); ++j) {
        for (int k = L.col_ptr()[j]; k < L.col_ptr()[j + 1]; ++k) {
            const int i = L.row_idx()[k];
            ri.push_back(i);
            ci.push_back(j);
            v.push_back(bd[i] ? (i == j ? 1.0 : 0.0) : L.values()[k]);
        }
    }
    return SparseOperator::from_triplets(L.rows(), L.cols(), ri, ci, v, "laplacian0(dirichlet)");
}

struct DirichletLevels {
    std::vector<SparseOperator> A;
    std::vector<std::vector<char>> bd;
    std::vector<std::vector<double>> w;
};

DirichletLevels dirichlet_levels(const MultigridHierarchy& h) {
    DirichletLevels d;
    for (int k = 0; k < h.levels(); ++k) {
        const auto bd = boundary_of(*h.level(k).mesh);
        d.A.push_back(dirichlet_rows(h.level(k).ops.laplacian, bd));
        d.bd.push_back(bd);
        d.w.push_back(h.level(k).ops.dual_areas);
    }
    return d;
}

// proj/src/multigrid.cpp:252-285 walk with the x1 extension: coarse RHS zeroed
// on boundary vertices after restriction; unpinned coarse CG.
void dirichlet_cycle(const MultigridHierarchy& h, const DirichletLevels& d, const CyclePlan& plan,
                     std::vector<std::vector<double>>& xs, std::vector<std::vector<double>>& bs) {
    const int nw = static_cast<int>(plan.walk.size());
    const int L = h.levels();
    int level = 0;
    std::vector<double> r;
    for (int w = 0; w < nw; ++w) {
        if (plan.walk[w] == Transition::Down) {
            smooth(d.A[level], xs[level], bs[level], plan.smoother, plan.pre[level], d.w[level]);
            r.resize(xs[level].size());
            d.A[level].apply(xs[level].data(), r.data());
            for (std::size_t i = 0; i < r.size(); ++i) r[i] = bs[level][i] - r[i];
            ++level;
            bs[level] = h.level(level - 1).restriction.apply(r);
            for (std::size_t i = 0; i < bs[level].size(); ++i)
                if (d.bd[level][i]) bs[level][i] = 0.0;
            kernels::fill(0.0, xs[level].data(), xs[level].size());
            if (level == L - 1) {
                xs[level] = standin_coarse_cg(d.A[level], d.w[level], bs[level], false);
            } else if (w + 1 < nw && plan.walk[w + 1] == Transition::Up) {
                smooth(d.A[level], xs[level], bs[level], plan.smoother, plan.pre[level],
                       d.w[level]);
            }
        } else {
            const std::vector<double> corr = h.level(level - 1).prolongation.apply(xs[level]);
            --level;
            for (std::size_t i = 0; i < corr.size(); ++i) xs[level][i] += corr[i];
            smooth(d.A[level], xs[level], bs[level], plan.smoother, plan.post[level], d.w[level]);
        }
    }
}

// run_cycle (proj/src/multigrid.cpp:287-323) over the Dirichlet levels.
MultigridHierarchy::CycleResult dirichlet_run(const MultigridHierarchy& h,
                                              const DirichletLevels& d, const CyclePlan& plan,
                                              const std::vector<double>& b,
                                              const std::vector<double>& x0) {
    const int L = h.levels();
    std::vector<std::vector<double>> xs(L), bs(L);
    for (int k = 0; k < L; ++k) {
        xs[k].assign(d.A[k].rows(), 0.0);
        bs[k].assign(d.A[k].rows(), 0.0);
    }
    xs[0] = x0;
    bs[0] = b;
    MultigridHierarchy::CycleResult res;
    const double bn = kernels::norm2(b.data(), b.size());
    const double denom = bn > 0.0 ? bn : 1.0;
    std::vector<double> r(b.size());
    for (int c = 0; c < plan.cycles; ++c) {
        if (L == 1) {
            xs[0] = standin_coarse_cg(d.A[0], d.w[0], bs[0], false);
        } else {
            dirichlet_cycle(h, d, plan, xs, bs);
        }
        d.A[0].apply(xs[0].data(), r.data());
        for (std::size_t i = 0; i < r.size(); ++i) r[i] = b[i] - r[i];
        res.residual_history.push_back(kernels::norm2(r.data(), r.size()) / denom);
    }
    res.x = std::move(xs[0]);
    return res;
}

// ---- output helpers -----------------------------------------------------------
void print_dvec(const char* key, const std::vector<double>& v, bool comma = true) {
    std::printf("\"%s\": [", key);
    for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
    std::printf("]%s\n", comma ? "," : "");
}
template <class T>
void print_ivec(const char* key, const std::vector<T>& v, bool comma = true) {
    std::printf("\"%s\": [", key);
    for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%lld", i ? ", " : "", (long long)v[i]);
    std::printf("]%s\n", comma ? "," : "");
}

void emit_operator(const char* name, const SparseOperator& A, bool full) {
    std::printf("\"%s\": {\"rows\": %d, \"cols\": %d, \"nnz\": %lld, ", name, A.rows(), A.cols(),
                (long long)A.nnz());
    std::printf("\"fnv_row_ptr\": \"%llu\", \"fnv_col_idx\": \"%llu\", \"fnv_values\": \"%llu\"",
                (unsigned long long)fnv_vec(A.row_ptr()), (unsigned long long)fnv_vec(A.col_idx()),
                (unsigned long long)fnv_vec(A.csr_values()));
    if (full) {
        std::printf(",\n");
        print_ivec("row_ptr", A.row_ptr());
        print_ivec("col_idx", A.col_idx());
        print_dvec("values", A.csr_values(), false);
    }
    std::printf("}");
}

int cmd_structure(const Case& c, int k, bool dirichlet, bool full) {
    const auto tower = tower_of(c, k);
    MultigridHierarchy h = build_hierarchy(c.base, tower);
    std::printf("{\"levels\": [\n");
    for (int l = 0; l < h.levels(); ++l) {
        const auto& lv = h.level(l);
        const auto& m = *lv.mesh;
        std::printf("{\"nv\": %d, \"ne\": %d, \"nt\": %d, \"hash\": \"%llu\",\n", m.num_vertices(),
                    m.num_edges(), m.num_triangles(), (unsigned long long)m.hash());
        std::vector<int> edges, tris;
        for (const auto& e : m.edges) edges.insert(edges.end(), e.begin(), e.end());
        for (const auto& t : m.triangles) tris.insert(tris.end(), t.begin(), t.end());
        std::printf("\"fnv_edges\": \"%llu\", \"fnv_triangles\": \"%llu\", \"fnv_positions\": \"%llu\", "
                    "\"fnv_dual_areas\": \"%llu\",\n",
                    (unsigned long long)fnv_vec(edges), (unsigned long long)fnv_vec(tris),
                    (unsigned long long)fnv(m.positions.data(), m.positions.size() * sizeof(Vec3)),
                    (unsigned long long)fnv_vec(lv.ops.dual_areas));
        if (full) {
            print_ivec("edges", edges);
            print_ivec("triangles", tris);
            std::vector<double> pos;
            for (const auto& p : m.positions) {
                pos.push_back(p.x);
                pos.push_back(p.y);
                pos.push_back(p.z);
            }
            print_dvec("positions", pos);
            print_dvec("dual_areas", lv.ops.dual_areas);
        }
        if (dirichlet) {
            const auto bd = boundary_of(m);
            emit_operator("L", dirichlet_rows(lv.ops.laplacian, bd), full);
            std::vector<int> bdi(bd.begin(), bd.end());
            std::printf(",\n");
            print_ivec("boundary", bdi, false);
        } else {
            emit_operator("L", lv.ops.laplacian, full);
        }
        if (lv.has_transfer) {
            std::printf(",\n");
            emit_operator("P", lv.prolongation, full);
            std::printf(",\n");
            emit_operator("R", lv.restriction, full);
        }
        std::printf("}%s\n", l + 1 < h.levels() ? "," : "");
    }
    std::printf("]}\n");
    return 0;
}

SmootherConfig jacobi() { return SmootherConfig{Smoother::WeightedJacobi, 2.0 / 3.0}; }

// "jacobi" | "gs" | "sgs" -> the reference's SmootherConfig (multigrid.hpp:55-60)
SmootherConfig smoother_of(const std::string& name) {
    if (name == "gs") return SmootherConfig{Smoother::GaussSeidel, 2.0 / 3.0};
    if (name == "sgs") return SmootherConfig{Smoother::SymmetricGaussSeidel, 2.0 / 3.0};
    if (name == "cg") return SmootherConfig{Smoother::Cg, 2.0 / 3.0};
    return jacobi();
}

int cmd_cycles(const Case& c, int k, bool dirichlet, const std::string& rhs, std::uint64_t seed,
               int ncycles, const std::string& smoother) {
    const auto tower = tower_of(c, k);
    MultigridHierarchy h = build_hierarchy(c.base, tower);
    CyclePlan plan = standard_plan(h.levels(), CycleKind::V, 2, 2, smoother_of(smoother));
    plan.cycles = ncycles;
    const auto& m = *h.level(0).mesh;
    MultigridHierarchy::CycleResult out;
    std::vector<double> b;
    if (dirichlet) {
        const DirichletLevels d = dirichlet_levels(h);
        b = make_rhs(rhs, m, d.A[0], seed, &d.bd[0]);
        out = dirichlet_run(h, d, plan, b, std::vector<double>(b.size(), 0.0));
    } else {
        b = h.project_compatible(make_rhs(rhs, m, h.fine_operator(), seed, nullptr));
        out = h.run_cycle(plan, b, std::vector<double>(b.size(), 0.0));
    }
    std::printf("{\"n\": %d, \"fnv_b\": \"%llu\", \"fnv_x\": \"%llu\",\n", (int)b.size(),
                (unsigned long long)fnv_vec(b), (unsigned long long)fnv_vec(out.x));
    print_dvec("history", out.residual_history, false);
    std::printf("}\n");
    return 0;
}

// solve ... [smoother] [use_levels] [rediscretize|galerkin] [V|W|F] [pre] [post]:
// build_hierarchy(base, tower, use_levels, HierarchyOptions{galerkin})
// (multigrid.cpp:196-238, 325-341) and standard_plan(levels, kind, pre, post)
struct SolveOpts {
    int use_levels = 0;
    bool galerkin = false;
    bool clamp = false;  // HodgeOptions::clamp_dual_areas
    std::string kind = "V";
    int pre = 2, post = 2;
};

int cmd_solve(const Case& c, int k, bool dirichlet, const std::string& rhs, std::uint64_t seed,
              double tol, int maxc, const std::string& smoother, const SolveOpts& so = {}) {
    const auto tower = tower_of(c, k);
    HierarchyOptions hopts;
    hopts.galerkin = so.galerkin;
    hopts.hodge.clamp_dual_areas = so.clamp;
    MultigridHierarchy h = build_hierarchy(c.base, tower, so.use_levels, hopts);
    const CycleKind kind = so.kind == "W" ? CycleKind::W : (so.kind == "F" ? CycleKind::F : CycleKind::V);
    CyclePlan plan = standard_plan(h.levels(), kind, so.pre, so.post, smoother_of(smoother));
    const auto& m = *h.level(0).mesh;
    std::vector<double> hist, x;
    int iters = 0;
    double final_res = 0.0;
    std::vector<double> b;
    if (dirichlet) {
        // gmg_solve (proj/src/solvers.cpp:251-279) without the Neumann projection
        const DirichletLevels d = dirichlet_levels(h);
        b = make_rhs(rhs, m, d.A[0], seed, &d.bd[0]);
        CyclePlan one = plan;
        one.cycles = 1;
        x.assign(b.size(), 0.0);
        double res = 0.0;
        while (iters < maxc) {
            auto out = dirichlet_run(h, d, one, b, x);
            x = std::move(out.x);
            res = out.residual_history.back();
            hist.push_back(res);
            ++iters;
            if (res <= tol) break;
        }
        final_res = res;
    } else {
        b = make_rhs(rhs, m, h.fine_operator(), seed, nullptr);
        const SolveReport rep = gmg_solve(h, plan, b, tol, maxc);
        hist = rep.residual_history;
        x = rep.solution;
        iters = rep.iterations;
        final_res = rep.final_relative_residual;
    }
    std::printf("{\"n\": %d, \"iterations\": %d, \"final\": %.17g, \"fnv_x\": \"%llu\",\n",
                (int)b.size(), iters, final_res, (unsigned long long)fnv_vec(x));
    print_dvec("history", hist, false);
    std::printf("}\n");
    return 0;
}

// CPU baseline: the reference protocol (proj/tools/decmg_main.cpp:133-147):
// gmg_preconditioned_cg (proj/src/solvers.cpp:118-130) with an inner plan
// standard_plan(levels, V|W, pre, post, smoother), inner.cycles = icyc
// (Neumann; the reference projects b itself).
int cmd_pcg(const Case& c, int k, const std::string& rhs, std::uint64_t seed, const std::string& kind, int pre,
            int post, int icyc, double tol, int maxit, const std::string& smoother) {
    const auto tower = tower_of(c, k);
    MultigridHierarchy h = build_hierarchy(c.base, tower);
    CyclePlan inner = standard_plan(h.levels(), kind == "W" ? CycleKind::W : CycleKind::V, pre, post,
                                    smoother_of(smoother));
    inner.cycles = icyc;
    const auto& m = *h.level(0).mesh;
    const std::vector<double> b = make_rhs(rhs, m, h.fine_operator(), seed, nullptr);
    const SolveReport rep = gmg_preconditioned_cg(h, inner, b, tol, maxit);
    std::printf("{\"n\": %d, \"iterations\": %d, \"converged\": %s, \"final\": %.17g, \"fnv_x\": \"%llu\",\n",
                (int)b.size(), rep.iterations, rep.converged ? "true" : "false", rep.final_relative_residual,
                (unsigned long long)fnv_vec(rep.solution));
    print_dvec("history", rep.residual_history, false);
    std::printf("}\n");
    return 0;
}

// I/O parity: write_obj / write_matrix_market of level `lvl` (mesh_io.cpp:71-82,
// sparse.cpp:247-259) and read_obj (mesh_io.cpp:19-69) + its mesh hash.
int cmd_write(const Case& c, int k, int lvl, const std::string& what, const std::string& out) {
    const auto tower = tower_of(c, k);
    MultigridHierarchy h = build_hierarchy(c.base, tower);
    const auto& L = h.level(lvl);
    if (what == "obj") write_obj(*L.mesh, out);
    else if (what == "L") L.ops.laplacian.write_matrix_market(out);
    else if (what == "P") L.prolongation.write_matrix_market(out);
    else if (what == "R") L.restriction.write_matrix_market(out);
    else throw std::invalid_argument("write: obj|L|P|R");
    return 0;
}

int cmd_readobj(const std::string& path) {
    try {
        const auto m = read_obj(path);
        std::printf("{\"nv\": %d, \"ne\": %d, \"nt\": %d, \"hash\": \"%llu\"}\n", m->num_vertices(),
                    m->num_edges(), m->num_triangles(), (unsigned long long)m->hash());
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
    }
    return 0;
}

// per-cycle cost = (t(2n) - t(n)) / n with run_cycle from x0 = 0, plus a full
// gmg_solve. nrhs independent right-hand sides are solved one after another
// (the reference has no batched solve).
int cmd_time(const Case& c, int k, bool dirichlet, int nrhs, int ncyc, double tol, int maxc,
             const std::string& smoother) {
    auto t0 = Clock::now();
    const auto tower = tower_of(c, k);
    MultigridHierarchy h = build_hierarchy(c.base, tower);
    const double setup_s = since(t0);
    CyclePlan plan = standard_plan(h.levels(), CycleKind::V, 2, 2, smoother_of(smoother));
    const auto& m = *h.level(0).mesh;
    const int n = m.num_vertices();
    double t_cycles_small = 0, t_cycles_big = 0, t_solve = 0;
    int solve_iters = 0;
    for (int r = 0; r < nrhs; ++r) {
        std::vector<double> b;
        if (dirichlet) {
            throw std::invalid_argument("time: dirichlet not supported");
        }
        b = h.project_compatible(make_rhs("uniform", m, h.fine_operator(), 1000 + r, nullptr));
        std::vector<double> x0(n, 0.0);
        CyclePlan p = plan;
        p.cycles = ncyc;
        t0 = Clock::now();
        h.run_cycle(p, b, x0);
        t_cycles_small += since(t0);
        p.cycles = 2 * ncyc;
        t0 = Clock::now();
        h.run_cycle(p, b, x0);
        t_cycles_big += since(t0);
        if (maxc > 0) {
            t0 = Clock::now();
            const SolveReport rep = gmg_solve(h, plan, b, tol, maxc);
            t_solve += since(t0);
            solve_iters += rep.iterations;
        }
    }
    const double per_cycle = (t_cycles_big - t_cycles_small) / (ncyc * nrhs);
    std::printf("{\"n\": %d, \"levels\": %d, \"nrhs\": %d, \"threads\": %d, \"setup_s\": %.6g, "
                "\"seconds_per_cycle\": %.9g, \"unknown_cycles_per_s\": %.9g, "
                "\"solve_s_per_rhs\": %.9g, \"solve_iters_per_rhs\": %.3f}\n",
                n, h.levels(), nrhs, omp_get_max_threads(), setup_s, per_cycle,
                per_cycle > 0 ? n / per_cycle : 0.0, maxc > 0 ? t_solve / nrhs : 0.0,
                maxc > 0 ? double(solve_iters) / nrhs : 0.0);
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    try {
        if (argc == 3 && std::string(argv[1]) == "readobj") return cmd_readobj(argv[2]);
        if (argc < 4) {
            std::fprintf(stderr,
                         "usage: ref_harness structure <case> <k> <bc> [full]\n"
                         "       ref_harness cycles <case> <k> <bc> <rhs> <seed> <ncycles> [jacobi|gs|sgs|cg]\n"
                         "       ref_harness solve <case> <k> <bc> <rhs> <seed> <tol> <maxc> [jacobi|gs|sgs|cg] "
                         "[use_levels] [rediscretize|galerkin|clamp|galerkin+clamp] [V|W|F] [pre] [post]\n"
                         "       ref_harness time <case> <k> <bc> <nrhs> <ncyc> <tol> <maxc> [jacobi|gs|sgs|cg]\n"
                         "       ref_harness write <case> <k> <level> <obj|L|P|R> <out>\n"
                         "       ref_harness readobj <file.obj>\n"
                         "       ref_harness pcg <case> <k> neumann <rhs> <seed> <V|W> <pre> <post> <cycles> <tol> <maxit> [jacobi|gs|sgs|cg]\n");
            return 2;
        }
        const std::string cmd = argv[1];
        const Case c = make_case(argv[2]);
        const int k = std::atoi(argv[3]);
        const bool dirichlet = argc > 4 && std::string(argv[4]) == "dirichlet";
        if (cmd == "structure") return cmd_structure(c, k, dirichlet, argc > 5 && std::string(argv[5]) == "full");
        if (cmd == "write" && argc >= 7) return cmd_write(c, k, std::atoi(argv[4]), argv[5], argv[6]);
        if (cmd == "pcg" && argc >= 13)
            return cmd_pcg(c, k, argv[5], std::strtoull(argv[6], nullptr, 10), argv[7], std::atoi(argv[8]),
                           std::atoi(argv[9]), std::atoi(argv[10]), std::atof(argv[11]), std::atoi(argv[12]),
                           argc > 13 ? argv[13] : "jacobi");
        if (cmd == "cycles")
            return cmd_cycles(c, k, dirichlet, argv[5], std::strtoull(argv[6], nullptr, 10),
                              std::atoi(argv[7]), argc > 8 ? argv[8] : "jacobi");
        if (cmd == "solve") {
            SolveOpts so;
            if (argc > 10) so.use_levels = std::atoi(argv[10]);
            if (argc > 11) {
                const std::string o = argv[11];
                so.galerkin = o.find("galerkin") != std::string::npos;
                so.clamp = o.find("clamp") != std::string::npos;
            }
            if (argc > 12) so.kind = argv[12];
            if (argc > 13) so.pre = std::atoi(argv[13]);
            if (argc > 14) so.post = std::atoi(argv[14]);
            return cmd_solve(c, k, dirichlet, argv[5], std::strtoull(argv[6], nullptr, 10),
                             std::atof(argv[7]), std::atoi(argv[8]), argc > 9 ? argv[9] : "jacobi", so);
        }
        if (cmd == "time")
            return cmd_time(c, k, dirichlet, std::atoi(argv[5]), std::atoi(argv[6]),
                            std::atof(argv[7]), std::atoi(argv[8]), argc > 9 ? argv[9] : "jacobi");
        std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_harness: %s\n", e.what());
        return 1;
    }
}
