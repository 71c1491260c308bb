// A reference-style C++ caller of the drop-in shim (include/decmg_gpu.hpp)
// without the reference's mesh types: BASELINE config 2 (icosphere x6 pushed
// to the sphere, Y_3^2 + noise RHS, weighted-Jacobi V(2,2), gmg_solve to 1e-8)
// built and solved on the device through the shim, plus smooth() and the level
// operators' apply(). Prints one JSON object for tests/test_gpu_shim.py.
#include "decmg_gpu.hpp"

#include <cstdio>
#include <vector>

static unsigned long long fnv(const void* p, size_t n) {
    unsigned long long h = 1469598103934665603ULL;
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= c[i];
        h *= 1099511628211ULL;
    }
    return h;
}

int main(int argc, char** argv) {
    const char* csv = argc > 1 ? argv[1] : nullptr;
    int nv = 0, nt = 0;
    decmg_base_mesh("ico", nullptr, &nv, nullptr, &nt);
    std::vector<double> pos(3 * nv);
    std::vector<int> tri(3 * nt);
    decmg_base_mesh("ico", pos.data(), &nv, tri.data(), &nt);
    decmg::MultigridHierarchy h(pos, tri, 6, DECMG_PROJECT_SPHERE);
    const int n = h.fine_rows();
    std::vector<double> b(n);
    if (decmg_gpu_make_rhs(h.handle(), "ylm", 1, 1, b.data()) != DECMG_OK) return 3;
    // the reference default smoother is Gauss-Seidel; config 2 asks for weighted Jacobi
    const decmg::SmootherConfig jac{decmg::Smoother::WeightedJacobi};
    const decmg::CyclePlan plan = decmg::standard_plan(h.levels(), decmg::CycleKind::V, 2, 2, jac);
    const decmg::SolveReport rep = decmg::gmg_solve(h, plan, b, 1e-8, 200);
    if (csv) rep.write_residual_csv(csv);
    // SparseOperator::apply and smooth on the fine level (x = projected b, 2 GS sweeps)
    const std::vector<double> bc = h.project_compatible(b);
    const std::vector<double> Lb = h.fine_operator().apply(bc);
    std::vector<double> xs(n, 0.0);
    decmg::smooth(h.fine_operator(), xs, bc, decmg::SmootherConfig{}, 2);
    std::vector<double> xj(h.level(1).ops.laplacian.rows(), 0.0);
    decmg::smooth(h.level(1).ops.laplacian, xj, h.level(0).restriction.apply(bc), jac, 3);
    bool threw = false;
    try {
        decmg::smooth(h.fine_operator(), xs, std::vector<double>(n + 1), decmg::SmootherConfig{}, 1);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    bool mono = rep.cumulative_seconds.size() == rep.residual_history.size();
    for (size_t i = 1; i < rep.cumulative_seconds.size(); ++i)
        mono = mono && rep.cumulative_seconds[i] >= rep.cumulative_seconds[i - 1];
    std::printf("{\"n\": %d, \"levels\": %d, \"iterations\": %d, \"converged\": %s, \"final\": %.17g, "
                "\"fnv_x\": \"%llu\", \"fnv_Lb\": \"%llu\", \"fnv_gs2\": \"%llu\", \"fnv_jac3_l1\": \"%llu\", "
                "\"shape_error\": %s, \"times_ok\": %s, \"history\": [",
                n, h.levels(), rep.iterations, rep.converged ? "true" : "false", rep.final_relative_residual,
                fnv(rep.solution.data(), sizeof(double) * n), fnv(Lb.data(), sizeof(double) * n),
                fnv(xs.data(), sizeof(double) * n), fnv(xj.data(), sizeof(double) * xj.size()),
                threw ? "true" : "false", mono ? "true" : "false");
    for (size_t i = 0; i < rep.residual_history.size(); ++i)
        std::printf("%s%.17g", i ? ", " : "", rep.residual_history[i]);
    std::printf("]}\n");
    return 0;
}
