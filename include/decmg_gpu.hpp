// Header-only C++ shim over the C ABI (decmg_gpu.h) that re-exposes the
// reference library's multigrid API with the same names, argument meaning and
// exception types, so a reference caller swaps
//     #include "decmg/multigrid.hpp" / "decmg/solvers.hpp"
// for
//     #include "decmg_gpu.hpp"
// and links -ldecmg_gpu. Mirrors (all /root/reference/proj/include/decmg/):
//   Smoother, SmootherConfig, Transition, CyclePlan, CycleKind, standard_plan
//                                                  multigrid.hpp:55-89
//   MultigridHierarchy::{levels, project_compatible, run_cycle}
//                                                  multigrid.hpp:106-136
//   build_hierarchy                                multigrid.hpp:140-143
//   SolveReport, gmg_solve                         solvers.hpp:17-30, 57-59
// std::invalid_argument / std::runtime_error are thrown exactly where the
// reference throws them (status codes DECMG_INVALID_ARGUMENT / DECMG_RUNTIME).
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "decmg_gpu.h"

namespace decmg {

enum class Smoother { GaussSeidel, SymmetricGaussSeidel, WeightedJacobi, Cg };

struct SmootherConfig {
    // device path: weighted Jacobi (default), (symmetric) Gauss-Seidel, Cg
    Smoother method = Smoother::WeightedJacobi;
    double jacobi_omega = 2.0 / 3.0;
};

enum class Transition { Down, Up };

struct CyclePlan {
    std::vector<Transition> walk;
    std::vector<int> pre;
    std::vector<int> post;
    SmootherConfig smoother;
    int cycles = 1;

    int depth() const {
        int level = 0, deepest = 0;
        for (Transition t : walk) {
            level += t == Transition::Down ? 1 : -1;
            deepest = level > deepest ? level : deepest;
        }
        return deepest + 1;
    }
    void validate(int levels) const {
        int level = 0;
        for (Transition t : walk) {
            level += t == Transition::Down ? 1 : -1;
            if (level < 0) throw std::invalid_argument("CyclePlan: walk rises above the finest level");
            if (level > levels - 1) throw std::invalid_argument("CyclePlan: walk descends below the coarsest level");
        }
        if (level != 0) throw std::invalid_argument("CyclePlan: walk does not return to the finest level");
        if (static_cast<int>(pre.size()) < levels || static_cast<int>(post.size()) < levels)
            throw std::invalid_argument("CyclePlan: missing per-level smoothing counts");
        if (cycles < 0) throw std::invalid_argument("CyclePlan: negative cycle count");
    }
};

enum class CycleKind { V, W, F };

namespace detail {
inline void emit_solve(std::vector<Transition>& out, int k, int levels, int gamma) {
    if (k == levels - 1) return;
    for (int g = 0; g < gamma; ++g) {
        out.push_back(Transition::Down);
        emit_solve(out, k + 1, levels, gamma);
        out.push_back(Transition::Up);
    }
}
inline void emit_f(std::vector<Transition>& out, int k, int levels) {
    if (k == levels - 1) return;
    out.push_back(Transition::Down);
    emit_f(out, k + 1, levels);
    out.push_back(Transition::Up);
    out.push_back(Transition::Down);
    emit_solve(out, k + 1, levels, 1);
    out.push_back(Transition::Up);
}
[[noreturn]] inline void raise(int rc, const decmg_gpu_ctx* ctx) {
    const std::string msg = decmg_gpu_last_error(ctx);
    if (rc == DECMG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == DECMG_OOM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}
inline void check(int rc, const decmg_gpu_ctx* ctx) {
    if (rc != DECMG_OK) raise(rc, ctx);
}
struct PlanC {
    std::string walk;
    std::vector<int> pre, post;
    decmg_gpu_plan s{};
    explicit PlanC(const CyclePlan& p) : pre(p.pre), post(p.post) {

        for (Transition t : p.walk) walk.push_back(t == Transition::Down ? 'd' : 'u');
        s.walk = walk.c_str();
        s.pre = pre.data();
        s.post = post.data();
        s.smoother = p.smoother.method == Smoother::GaussSeidel            ? DECMG_SMOOTHER_GS
                     : p.smoother.method == Smoother::SymmetricGaussSeidel ? DECMG_SMOOTHER_SGS
                     : p.smoother.method == Smoother::Cg                   ? DECMG_SMOOTHER_CG
                                                                            : DECMG_SMOOTHER_JACOBI;
        s.jacobi_omega = p.smoother.jacobi_omega;
    }
};
}  // namespace detail

inline CyclePlan standard_plan(int levels, CycleKind kind, int pre = 3, int post = 3,
                               SmootherConfig smoother = {}) {
    if (levels < 1) throw std::invalid_argument("standard_plan: levels >= 1");
    CyclePlan plan;
    plan.pre.assign(levels, pre);
    plan.post.assign(levels, post);
    plan.smoother = smoother;
    if (levels > 1) {
        if (kind == CycleKind::V) {
            detail::emit_solve(plan.walk, 0, levels, 1);
        } else {
            plan.walk.push_back(Transition::Down);
            if (kind == CycleKind::W) detail::emit_solve(plan.walk, 1, levels, 2);
            else detail::emit_f(plan.walk, 1, levels);
            plan.walk.push_back(Transition::Up);
        }
    }
    plan.validate(levels);
    return plan;
}

class MultigridHierarchy {
public:
    struct CycleResult {
        std::vector<double> x;
        std::vector<double> residual_history;
    };

    // GPU construction from a base complex (positions + corner triples, as
    // for EmbeddedComplex2D::from_triangles) and nsub binary subdivisions.
    MultigridHierarchy(const std::vector<double>& positions, const std::vector<int>& corner_triples, int nsub,
                       unsigned flags = 0, int device = 0, int max_nrhs = 1) {
        decmg_gpu_config cfg{device, max_nrhs};
        decmg_gpu_ctx* c = nullptr;
        const int rc = decmg_gpu_create_from_base(positions.data(), static_cast<int>(positions.size() / 3),
                                                  corner_triples.data(), static_cast<int>(corner_triples.size() / 3),
                                                  nsub, flags, &cfg, &c);
        if (rc != DECMG_OK) detail::raise(rc, nullptr);
        ctx_ = std::shared_ptr<decmg_gpu_ctx>(c, Del{});
    }

    int levels() const { return decmg_gpu_levels(ctx_.get()); }
    int fine_rows() const {
        int64_t c[6];
        detail::check(decmg_gpu_level_info(ctx_.get(), 0, c), ctx_.get());
        return static_cast<int>(c[0]);
    }
    decmg_gpu_ctx* handle() const { return ctx_.get(); }

    std::vector<double> project_compatible(std::vector<double> b) const {
        detail::check(decmg_gpu_project_compatible(ctx_.get(), 1, b.data()), ctx_.get());
        return b;
    }

    CycleResult run_cycle(const CyclePlan& plan, const std::vector<double>& b, const std::vector<double>& x0) const {
        plan.validate(levels());
        if (static_cast<int>(b.size()) != fine_rows() || b.size() != x0.size())
            throw std::invalid_argument("run_cycle: rhs size mismatch");
        detail::PlanC pc(plan);
        CycleResult r;
        r.x.resize(b.size());
        r.residual_history.resize(plan.cycles);
        detail::check(decmg_gpu_run_cycles(ctx_.get(), &pc.s, 1, b.data(), x0.data(), plan.cycles, r.x.data(),
                                           r.residual_history.data()),
                      ctx_.get());
        return r;
    }

private:
    struct Del {
        void operator()(decmg_gpu_ctx* c) const { decmg_gpu_destroy(c); }
    };
    std::shared_ptr<decmg_gpu_ctx> ctx_{nullptr, Del{}};
};

struct SolveReport {
    std::vector<double> solution;
    std::vector<double> residual_history;
    std::vector<double> cumulative_seconds;
    int iterations = 0;
    bool converged = false;
    bool stagnated = false;
    double final_relative_residual = 0.0;
    double wall_seconds = 0.0;
};

inline SolveReport gmg_solve(const MultigridHierarchy& h, const CyclePlan& plan, const std::vector<double>& b,
                             double tol, int max_cycles, const std::vector<double>* x0 = nullptr) {
    const auto t0 = std::chrono::steady_clock::now();
    plan.validate(h.levels());
    if (static_cast<int>(b.size()) != h.fine_rows()) throw std::invalid_argument("run_cycle: rhs size mismatch");
    detail::PlanC pc(plan);
    SolveReport rep;
    rep.solution.resize(b.size());
    std::vector<double> hist(max_cycles > 0 ? max_cycles : 1);
    int done = 0;
    double fin = 0.0;
    detail::check(decmg_gpu_solve(h.handle(), &pc.s, 1, b.data(), x0 ? x0->data() : nullptr, tol, max_cycles,
                                  rep.solution.data(), hist.data(), &done, &fin),
                  h.handle());
    rep.residual_history.assign(hist.begin(), hist.begin() + done);
    rep.iterations = done;
    rep.converged = fin <= tol;
    rep.final_relative_residual = fin;
    rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rep;
}

// A stream of independent single-RHS gmg_solve calls (extension x6,
// decmg_gpu_solve_batches): the next right-hand side's upload and projection
// and the previous solution's download overlap the current solve's cycles.
// Each report equals gmg_solve(h, plan, bs[k], tol, max_cycles) bit for bit.
// (Host vectors are pageable here; pinned buffers through the C ABI overlap fully.)
inline std::vector<SolveReport> gmg_solve_batches(const MultigridHierarchy& h, const CyclePlan& plan,
                                                  const std::vector<std::vector<double>>& bs, double tol,
                                                  int max_cycles) {
    const auto t0 = std::chrono::steady_clock::now();
    plan.validate(h.levels());
    const int nb = static_cast<int>(bs.size());
    for (const auto& b : bs)
        if (static_cast<int>(b.size()) != h.fine_rows()) throw std::invalid_argument("run_cycle: rhs size mismatch");
    detail::PlanC pc(plan);
    std::vector<SolveReport> reps(bs.size());
    std::vector<const double*> bp(bs.size());
    std::vector<double*> xp(bs.size());
    for (int k = 0; k < nb; ++k) {
        reps[k].solution.resize(bs[k].size());
        bp[k] = bs[k].data();
        xp[k] = reps[k].solution.data();
    }
    const int mc = max_cycles > 0 ? max_cycles : 1;
    std::vector<double> hist(static_cast<size_t>(nb) * mc), fin(nb);
    std::vector<int> done(nb);
    detail::check(decmg_gpu_solve_batches(h.handle(), &pc.s, 1, nb, bp.data(), tol, max_cycles, xp.data(),
                                          hist.data(), done.data(), fin.data()),
                  h.handle());
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int k = 0; k < nb; ++k) {
        reps[k].residual_history.assign(hist.begin() + static_cast<size_t>(k) * mc,
                                        hist.begin() + static_cast<size_t>(k) * mc + done[k]);
        reps[k].iterations = done[k];
        reps[k].converged = fin[k] <= tol;
        reps[k].final_relative_residual = fin[k];
        reps[k].wall_seconds = wall;
    }
    return reps;
}

// gmg_preconditioned_cg (proj/src/solvers.cpp:118-130); inner_plan.cycles
// cycles of the inner plan precondition each CG step. Single RHS, like the
// reference; the C ABI (decmg_gpu_pcg) also takes [n][nrhs] batches.
inline SolveReport gmg_preconditioned_cg(const MultigridHierarchy& h, const CyclePlan& inner_plan,
                                         const std::vector<double>& b, double tol, int maxiter) {
    const auto t0 = std::chrono::steady_clock::now();
    inner_plan.validate(h.levels());
    if (static_cast<int>(b.size()) != h.fine_rows()) throw std::invalid_argument("run_cycle: rhs size mismatch");
    detail::PlanC pc(inner_plan);
    SolveReport rep;
    rep.solution.resize(b.size());
    std::vector<double> hist(static_cast<size_t>(maxiter > 0 ? maxiter : 0) + 1);
    int its = 0, conv = 0;
    double fin = 0.0;
    detail::check(decmg_gpu_pcg(h.handle(), &pc.s, inner_plan.cycles, 1, b.data(), tol, maxiter,
                                rep.solution.data(), hist.data(), &its, &conv, &fin),
                  h.handle());
    rep.residual_history.assign(hist.begin(), hist.begin() + its + 1);
    rep.iterations = its;
    rep.converged = conv != 0;
    rep.final_relative_residual = fin;
    rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rep;
}

}  // namespace decmg
