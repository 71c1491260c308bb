// The reference's downstream consumer of the multigrid path: porous convection
// (integrate_convection, /root/reference/proj/src/physics.cpp:220-272), whose
// right-hand side solves a pressure Poisson problem per Runge-Kutta stage with
// a warm-started gmg_solve (solve_pressure_rhs, physics.cpp:136-166).
//
// This file only uses decmg/physics.hpp. It is compiled twice by
// `make -C oracle convection`:
//   oracle/_ref/convection_ref  against the reference's own headers and objects
//                               (CPU; generates tests/golden/convection_*.json);
//   oracle/_ref/convection_gpu  the SAME reference sources physics.cpp and
//                               rk54.cpp, unmodified, compiled with
//                               include/dropin first on the include path, so
//                               their MultigridHierarchy / gmg_solve /
//                               gmg_preconditioned_cg are the CUDA library's.
// usage: convection_* nx ny levels t_final samples smoother cycle pre post solver [rtol]
#include "decmg/physics.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
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

}  // namespace

int main(int argc, char** argv) {
    if (argc < 11) {
        std::fprintf(stderr, "usage: %s nx ny levels t_final samples gs|sgs|jacobi V|W|F pre post gmg|gmgpcg [rtol]\n",
                     argv[0]);
        return 2;
    }
    decmg::ConvectionConfig cfg;
    cfg.nx = std::atoi(argv[1]);
    cfg.ny = std::atoi(argv[2]);
    cfg.levels = std::atoi(argv[3]);
    cfg.t_final = std::atof(argv[4]);
    cfg.num_samples = std::atoi(argv[5]);
    const std::string sm = argv[6], cy = argv[7], sv = argv[10];
    decmg::SolverSpec& sp = cfg.pressure_solver;
    sp.smoother = sm == "jacobi" ? decmg::Smoother::WeightedJacobi
                  : sm == "sgs"  ? decmg::Smoother::SymmetricGaussSeidel
                                 : decmg::Smoother::GaussSeidel;
    sp.cycle = cy == "V" ? decmg::CycleKind::V : cy == "F" ? decmg::CycleKind::F : decmg::CycleKind::W;
    sp.pre_smooth = std::atoi(argv[8]);
    sp.post_smooth = std::atoi(argv[9]);
    sp.kind = sv == "gmgpcg" ? decmg::SolverKind::GmgPcg : decmg::SolverKind::Gmg;
    if (argc > 11) cfg.rtol = cfg.atol = std::atof(argv[11]);
    try {
        const decmg::ConvectionRun run = decmg::integrate_convection(cfg);
        std::printf("{\"nx\": %d, \"ny\": %d, \"levels\": %d, \"n\": %d, \"t_final\": %.17g, \"accepted\": %ld, "
                    "\"rejected\": %ld, \"rhs_evaluations\": %ld, \"pressure_solves\": %ld, "
                    "\"max_pressure_residual\": %.17g, \"max_relative_divergence\": %.17g, \"wall_seconds\": %.6f, "
                    "\"samples\": [",
                    cfg.nx, cfg.ny, cfg.levels, run.mesh->num_vertices(), cfg.t_final, run.stats.accepted,
                    run.stats.rejected, run.stats.rhs_evaluations, run.pressure_solves, run.max_pressure_residual,
                    run.max_relative_divergence, run.wall_seconds);
        for (size_t i = 0; i < run.samples.size(); ++i) {
            const decmg::ConvectionSample& s = run.samples[i];
            double tmax = 0, pmax = 0;
            for (double v : s.T) tmax = std::abs(v) > tmax ? std::abs(v) : tmax;
            for (double v : s.P) pmax = std::abs(v) > pmax ? std::abs(v) : pmax;
            const size_t mid = s.T.size() / 2 + 3;
            std::printf("%s{\"t\": %.17g, \"fnv_T\": \"%llu\", \"fnv_P\": \"%llu\", \"T_mid\": %.17g, \"P_mid\": %.17g, "
                        "\"T_absmax\": %.17g, \"P_absmax\": %.17g}",
                        i ? ", " : "", s.t, fnv(s.T), fnv(s.P), s.T[mid], s.P[mid], tmax, pmax);
        }
        std::printf("]}\n");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "convection: %s\n", e.what());
        return 1;
    }
    return 0;
}
