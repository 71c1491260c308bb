// A reference caller switched to the GPU: it keeps the reference's own mesh,
// subdivision and map types (decmg/mesh.hpp, subdivision.hpp, geometric_map.hpp)
// and swaps decmg/multigrid.hpp + solvers.hpp for the drop-in shim. Each case
// is one of the reference's golden solves (tests/golden/make_golden.py):
// build_hierarchy(base, tower, use_levels, HierarchyOptions) + gmg_solve with
// the harness's plan and right-hand side. Prints one JSON object with the
// solve of every case and whether the shim built the hierarchy on the device
// or assembled it on the host (Galerkin). Built by `make -C oracle shim`.
#define DECMG_GPU_REFERENCE_TYPES
#include "decmg_gpu.hpp"

#include "decmg/rng.hpp"
#include "ref_cases.hpp"

#include <cstdio>
#include <random>
#include <string>
#include <vector>

namespace {

unsigned long long fnv(const std::vector<double>& v) {
    unsigned long long h = 1469598103934665603ULL;
    const unsigned char* c = reinterpret_cast<const unsigned char*>(v.data());
    for (size_t i = 0; i < v.size() * sizeof(double); ++i) {
        h ^= c[i];
        h *= 1099511628211ULL;
    }
    return h;
}

struct Case {
    const char* golden;
    const char* spec;
    int k;
    unsigned long long seed;
    decmg::Smoother smoother;
    int use_levels;
    bool galerkin, clamp;
    decmg::CycleKind kind;
    const char* expect_path;
};

}  // namespace

int main() {
    using decmg::CycleKind;
    using decmg::Smoother;
    const Case cases[] = {
        {"solve_square_5_gs", "square", 5, 5, Smoother::GaussSeidel, 0, false, false, CycleKind::V, "device"},
        {"solve_levels_used_2", "equi:24:48:1.0", 3, 7, Smoother::GaussSeidel, 2, false, false, CycleKind::W, "device"},
        {"solve_levels_used_3", "equi:24:48:1.0", 3, 7, Smoother::GaussSeidel, 3, false, false, CycleKind::W, "device"},
        {"solve_levels_used_all", "equi:24:48:1.0", 3, 7, Smoother::GaussSeidel, 0, false, false, CycleKind::W,
         "device"},
        {"solve_ico_5_clamp", "ico", 5, 5, Smoother::WeightedJacobi, 0, false, true, CycleKind::V, "device"},
        {"solve_ico_4_galerkin", "ico", 4, 5, Smoother::GaussSeidel, 0, true, false, CycleKind::V, "host"},
    };
    std::printf("{\"cases\": [");
    bool first = true;
    for (const Case& cs : cases) {
        const refcases::Case c = refcases::make_case(cs.spec);
        const auto tower = refcases::tower_of(c, cs.k);
        decmg::HierarchyOptions opts;
        opts.galerkin = cs.galerkin;
        opts.hodge.clamp_dual_areas = cs.clamp;
        decmg::MultigridHierarchy h = decmg::build_hierarchy(c.base, tower, cs.use_levels, opts);
        const decmg::CyclePlan plan =
            decmg::standard_plan(h.levels(), cs.kind, 2, 2, decmg::SmootherConfig{cs.smoother});
        // ref_harness make_rhs("uniform"): 2 u - 1 from mt19937_64(seed)
        const int n = h.fine_rows();
        std::vector<double> b(n);
        std::mt19937_64 rng(cs.seed);
        for (int i = 0; i < n; ++i) b[i] = 2.0 * decmg::uniform01(rng) - 1.0;
        const decmg::SolveReport rep = decmg::gmg_solve(h, plan, b, 1e-8, cs.galerkin ? 100 : 60);
        std::printf("%s\n{\"golden\": \"%s\", \"path\": \"%s\", \"expect_path\": \"%s\", \"levels\": %d, \"n\": %d, "
                    "\"iterations\": %d, \"fnv_x\": \"%llu\", \"history\": [",
                    first ? "" : ",", cs.golden, h.assembled_on_device() ? "device" : "host", cs.expect_path,
                    h.levels(), n, rep.iterations, fnv(rep.solution));
        for (size_t i = 0; i < rep.residual_history.size(); ++i)
            std::printf("%s%.17g", i ? ", " : "", rep.residual_history[i]);
        std::printf("]}");
        first = false;
    }
    std::printf("\n]}\n");
    return 0;
}
