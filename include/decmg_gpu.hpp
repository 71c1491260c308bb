// Header-only C++ shim over the C ABI (decmg_gpu.h) that re-exposes the
// reference library's multigrid API with the same names, argument meaning,
// defaults and exception types, so a reference caller swaps
//     #include "decmg/multigrid.hpp" / "decmg/solvers.hpp"
// for
//     #define DECMG_GPU_REFERENCE_TYPES   // keeps the reference's mesh/map types
//     #include "decmg_gpu.hpp"
// and links -ldecmg_gpu (plus the reference's mesh/geometry objects it already
// builds its towers with). Mirrors (all /root/reference/proj/include/decmg/):
//   Smoother, SmootherConfig, Transition, CyclePlan, CycleKind, standard_plan,
//   smooth                                         multigrid.hpp:55-89
//   HierarchyOptions, MultigridLevel               multigrid.hpp:91-104
//   MultigridHierarchy(meshes, maps, opts), levels, level, fine_operator,
//   project_compatible, run_cycle                  multigrid.hpp:106-136
//   build_hierarchy(base, tower, use_levels, opts) multigrid.hpp:140-143
//   SolveReport (+ to_json, write_residual_csv), gmg_solve,
//   gmg_preconditioned_cg                          solvers.hpp:17-30, 44-59
//   SparseOperator::apply of the level operators   sparse.hpp:63-64
// std::invalid_argument / std::runtime_error are thrown exactly where the
// reference throws them (status codes DECMG_INVALID_ARGUMENT / DECMG_RUNTIME),
// with the reference's messages.
//
// Without DECMG_GPU_REFERENCE_TYPES the shim stands alone: a hierarchy is
// built on the device from a base complex (positions + corner triples) and a
// subdivision count.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "decmg_gpu.h"

#if defined(__has_include)
#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define DECMG_GPU_HAVE_JSON 1
#endif
#endif

#ifdef DECMG_GPU_REFERENCE_TYPES
#include "decmg/geometric_map.hpp"
#include "decmg/mesh.hpp"
#include "decmg/operators.hpp"
#include "decmg/sparse.hpp"
#include "decmg/subdivision.hpp"
#endif

namespace decmg {

enum class Smoother { GaussSeidel, SymmetricGaussSeidel, WeightedJacobi, Cg };

struct SmootherConfig {
    // the reference default (multigrid.hpp:58); the device runs the exact
    // lexicographic sweep as a level schedule (bit-identical)
    Smoother method = Smoother::GaussSeidel;
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
inline int smoother_code(Smoother m) {
    return m == Smoother::GaussSeidel            ? DECMG_SMOOTHER_GS
           : m == Smoother::SymmetricGaussSeidel ? DECMG_SMOOTHER_SGS
           : m == Smoother::Cg                   ? DECMG_SMOOTHER_CG
                                                 : DECMG_SMOOTHER_JACOBI;
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
        s.smoother = smoother_code(p.smoother.method);
        s.jacobi_omega = p.smoother.jacobi_omega;
    }
};
inline std::vector<double> last_times(decmg_gpu_ctx* c) {
    const int n = decmg_gpu_last_times(c, nullptr, 0);
    std::vector<double> t(n > 0 ? n : 0);
    if (n > 0) decmg_gpu_last_times(c, t.data(), n);
    return t;
}
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

// A level operator resident on the device (L_k, P_k or R_k of a hierarchy):
// the SparseOperator surface the solver path uses -- shape, nnz, CSR arrays
// (copied back on request) and apply (sparse.hpp:63-64, sparse.cpp:209-218,
// bit-identical row sums).
class DeviceOperator {
public:
    DeviceOperator() = default;
    DeviceOperator(std::shared_ptr<decmg_gpu_ctx> ctx, int level, char op) : ctx_(std::move(ctx)), level_(level), op_(op) {
        int64_t c[6];
        detail::check(decmg_gpu_level_info(ctx_.get(), level, c), ctx_.get());
        int64_t cn[6] = {0, 0, 0, 0, 0, 0};
        if (op != 'L') detail::check(decmg_gpu_level_info(ctx_.get(), level + 1, cn), ctx_.get());
        rows_ = static_cast<int>(op == 'R' ? cn[0] : c[0]);
        cols_ = static_cast<int>(op == 'P' ? cn[0] : c[0]);
        nnz_ = op == 'L' ? c[3] : (op == 'P' ? c[4] : c[5]);
    }
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    std::int64_t nnz() const { return nnz_; }
    int level() const { return level_; }
    char kind() const { return op_; }
    decmg_gpu_ctx* handle() const { return ctx_.get(); }

    void apply(const double* x, double* y) const {
        detail::check(decmg_gpu_apply(ctx_.get(), level_, op_, x, y), ctx_.get());
    }
    std::vector<double> apply(const std::vector<double>& x) const {
        if (static_cast<int>(x.size()) != cols_) throw std::invalid_argument("apply: size mismatch");
        std::vector<double> y(rows_);
        apply(x.data(), y.data());
        return y;
    }
    std::vector<int> row_ptr() const { return fetch<int>("_row_ptr"); }
    std::vector<int> col_idx() const { return fetch<int>("_col_idx"); }
    std::vector<double> csr_values() const { return fetch<double>("_values"); }

private:
    template <class T>
    std::vector<T> fetch(const char* suffix) const {
        const std::string name = std::string(1, op_) + suffix;
        const int64_t n = decmg_gpu_export(ctx_.get(), level_, name.c_str(), nullptr);
        if (n < 0) throw std::runtime_error("export failed: " + name);
        std::vector<T> v(static_cast<size_t>(n));
        decmg_gpu_export(ctx_.get(), level_, name.c_str(), v.data());
        return v;
    }
    std::shared_ptr<decmg_gpu_ctx> ctx_;
    int level_ = 0;
    char op_ = 'L';
    int rows_ = 0, cols_ = 0;
    std::int64_t nnz_ = 0;
};

// smooth (multigrid.hpp:66-68, multigrid.cpp:95-120) with A a level
// Laplacian of a device hierarchy: iters sweeps in place. weights: empty
// (plain dots for the CG smoother) or the level's dual areas (what cycle_once
// passes).
inline void smooth(const DeviceOperator& A, std::vector<double>& x, const std::vector<double>& b,
                   const SmootherConfig& cfg, int iters, const std::vector<double>& weights = {}) {
    if (A.rows() != A.cols() || static_cast<int>(x.size()) != A.rows() || x.size() != b.size())
        throw std::invalid_argument("smooth: shape mismatch");
    if (A.kind() != 'L') throw std::invalid_argument("smooth: the device smoother runs on a level Laplacian");
    int weighted = 0;
    if (!weights.empty()) {
        std::vector<double> w(static_cast<size_t>(A.rows()));
        decmg_gpu_export(A.handle(), A.level(), "dual_areas", w.data());
        if (weights != w)
            throw std::invalid_argument("smooth: device weights must be empty or the level's dual areas");
        weighted = 1;
    }
    detail::check(decmg_gpu_smooth(A.handle(), A.level(), detail::smoother_code(cfg.method), cfg.jacobi_omega,
                                   iters, 1, x.data(), b.data(), weighted),
                  A.handle());
}

#ifdef DECMG_GPU_REFERENCE_TYPES
struct HierarchyOptions {
    /// Assemble coarse operators by Galerkin projection R A P instead of
    /// rediscretizing on each mesh (comparison experiments only).
    bool galerkin = false;
    HodgeOptions hodge;
};
#endif

// The operators of one level (MultigridLevel, multigrid.hpp:91-97), on the device.
struct DeviceLevelOps {
    DeviceOperator laplacian;
    std::vector<double> dual_areas;
};
struct MultigridLevel {
#ifdef DECMG_GPU_REFERENCE_TYPES
    std::shared_ptr<const EmbeddedComplex2D> mesh;  // set by the reference-type constructor
#endif
    DeviceLevelOps ops;
    DeviceOperator prolongation;  // absent on the coarsest level
    DeviceOperator restriction;
    bool has_transfer = false;
};

class MultigridHierarchy {
public:
    struct CycleResult {
        std::vector<double> x;
        std::vector<double> residual_history;
    };

    // GPU construction from a base complex (positions + corner triples, as
    // for EmbeddedComplex2D::from_triangles) and nsub subdivisions.
    MultigridHierarchy(const std::vector<double>& positions, const std::vector<int>& corner_triples, int nsub,
                       unsigned flags = 0, int device = 0, int max_nrhs = 1) {
        adopt(create_base(positions, corner_triples, nsub, flags, device, max_nrhs));
    }

#ifdef DECMG_GPU_REFERENCE_TYPES
    /// meshes are ordered finest first; maps[k] sends mesh k to mesh k+1
    /// (MultigridHierarchy ctor, multigrid.cpp:196-238). A tower that is the
    /// binary or cubic subdivision of its coarsest mesh (plain or pushed to
    /// the unit sphere) is built on the device -- every mesh hash is checked
    /// against the given meshes; anything else (other towers, Galerkin coarse
    /// operators, clamped dual areas) is assembled on the host by the
    /// reference's own builders and uploaded. The cycles run on the device
    /// either way.
    MultigridHierarchy(std::vector<std::shared_ptr<const EmbeddedComplex2D>> meshes,
                       const std::vector<GeometricMap>& maps, const HierarchyOptions& opts = {}, int device = 0,
                       int max_nrhs = 1) {
        if (meshes.empty()) throw std::invalid_argument("hierarchy: no meshes");
        if (maps.size() + 1 != meshes.size()) throw std::invalid_argument("hierarchy: need one map per mesh pair");
        const int L = static_cast<int>(meshes.size());
        for (int k = 0; k + 1 < L; ++k) {
            const GeometricMap& f = maps[k];
            if (f.domain()->hash() != meshes[k]->hash() || f.codomain()->hash() != meshes[k + 1]->hash())
                throw std::invalid_argument("hierarchy: map " + std::to_string(k) + " does not connect its meshes");
        }
        meshes_ = meshes;
        decmg_gpu_ctx* c = nullptr;
        if (!opts.galerkin)
            c = try_device_tower(meshes, opts.hodge.clamp_dual_areas ? DECMG_CLAMP_DUAL_AREAS : 0u, device, max_nrhs);
        on_device_ = c != nullptr;
        if (!c) c = assemble_on_host(meshes, maps, opts, device, max_nrhs);
        adopt(c);
    }
#endif

    int levels() const { return decmg_gpu_levels(ctx_.get()); }
    /// true: meshes and operators were built on the device (subdivision tower
    /// recognised); false: assembled on the host by the reference and uploaded
    bool assembled_on_device() const { return on_device_; }
    int fine_rows() const {
        int64_t c[6];
        detail::check(decmg_gpu_level_info(ctx_.get(), 0, c), ctx_.get());
        return static_cast<int>(c[0]);
    }
    decmg_gpu_ctx* handle() const { return ctx_.get(); }
    const MultigridLevel& level(int k) const {
        if (k < 0 || k >= levels()) throw std::out_of_range("hierarchy: level out of range");
        return levels_[k];
    }
    const DeviceOperator& fine_operator() const { return levels_.front().ops.laplacian; }

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
    static decmg_gpu_ctx* create_base(const std::vector<double>& positions, const std::vector<int>& corner_triples,
                                      int nsub, unsigned flags, int device, int max_nrhs) {
        decmg_gpu_config cfg{device, max_nrhs};
        decmg_gpu_ctx* c = nullptr;
        const int rc = decmg_gpu_create_from_base(positions.data(), static_cast<int>(positions.size() / 3),
                                                  corner_triples.data(), static_cast<int>(corner_triples.size() / 3),
                                                  nsub, flags, &cfg, &c);
        if (rc != DECMG_OK) detail::raise(rc, nullptr);
        return c;
    }
    void adopt(decmg_gpu_ctx* c) {
        ctx_ = std::shared_ptr<decmg_gpu_ctx>(c, Del{});
        const int L = levels();
        levels_.resize(L);
        for (int k = 0; k < L; ++k) {
            MultigridLevel& lv = levels_[k];
            lv.ops.laplacian = DeviceOperator(ctx_, k, 'L');
            const int64_t n = decmg_gpu_export(ctx_.get(), k, "dual_areas", nullptr);
            lv.ops.dual_areas.resize(n > 0 ? static_cast<size_t>(n) : 0);
            if (n > 0) decmg_gpu_export(ctx_.get(), k, "dual_areas", lv.ops.dual_areas.data());
            if (k + 1 < L) {
                lv.prolongation = DeviceOperator(ctx_, k, 'P');
                lv.restriction = DeviceOperator(ctx_, k, 'R');
                lv.has_transfer = true;
            }
#ifdef DECMG_GPU_REFERENCE_TYPES
            if (k < static_cast<int>(meshes_.size())) lv.mesh = meshes_[k];
#endif
        }
    }
#ifdef DECMG_GPU_REFERENCE_TYPES
    static void flatten(const EmbeddedComplex2D& m, std::vector<double>* pos, std::vector<int>* tri) {
        pos->clear();
        tri->clear();
        for (const Vec3& p : m.positions) {
            pos->push_back(p.x);
            pos->push_back(p.y);
            pos->push_back(p.z);
        }
        if (!m.has_corners()) return;
        for (int t = 0; t < m.num_triangles(); ++t)
            for (int v : m.corners(t)) tri->push_back(v);
    }
    static bool hashes_match(decmg_gpu_ctx* c, const std::vector<std::shared_ptr<const EmbeddedComplex2D>>& meshes,
                             int first_mesh) {
        const int L = decmg_gpu_levels(c);
        if (L != static_cast<int>(meshes.size()) - first_mesh) return false;
        for (int k = 0; k < L; ++k) {
            uint64_t h = 0;
            if (decmg_gpu_mesh_hash(c, k, &h) != DECMG_OK || h != meshes[first_mesh + k]->hash()) return false;
        }
        return true;
    }
    // The device tower of the coarsest mesh, if it reproduces every given mesh.
    static decmg_gpu_ctx* try_device_tower(const std::vector<std::shared_ptr<const EmbeddedComplex2D>>& meshes,
                                           unsigned hodge, int device, int max_nrhs) {
        const int L = static_cast<int>(meshes.size());
        std::vector<double> pos;
        std::vector<int> tri;
        flatten(*meshes.back(), &pos, &tri);
        if (tri.empty()) return nullptr;
        decmg_gpu_config cfg{device, max_nrhs};
        const int V = meshes.back()->num_vertices(), E = meshes.back()->num_edges(), T = meshes.back()->num_triangles();
        unsigned scheme = 0;
        if (L >= 2) {
            const int nf = meshes[L - 2]->num_vertices();
            if (nf == V + 2 * E + T) scheme = DECMG_CUBIC;
            else if (nf != V + E) return nullptr;
        }
        // plain or sphere-projected: decided on one subdivision, then checked on every level
        for (unsigned proj : {0u, static_cast<unsigned>(DECMG_PROJECT_SPHERE)}) {
            decmg_gpu_ctx* c = nullptr;
            if (L >= 2) {
                if (decmg_gpu_create_from_base(pos.data(), V, tri.data(), T, 1, scheme | proj | hodge, &cfg, &c) !=
                    DECMG_OK)
                    return nullptr;
                const bool ok = hashes_match(c, meshes, L - 2);
                decmg_gpu_destroy(c);
                c = nullptr;
                if (!ok) continue;
            }
            if (decmg_gpu_create_from_base(pos.data(), V, tri.data(), T, L - 1, scheme | proj | hodge, &cfg, &c) !=
                DECMG_OK)
                return nullptr;
            if (hashes_match(c, meshes, 0)) return c;
            decmg_gpu_destroy(c);
            return nullptr;
        }
        return nullptr;
    }
    // The reference's own assembly (multigrid.cpp:215-235) on the host, uploaded.
    static decmg_gpu_ctx* assemble_on_host(const std::vector<std::shared_ptr<const EmbeddedComplex2D>>& meshes,
                                           const std::vector<GeometricMap>& maps, const HierarchyOptions& opts,
                                           int device, int max_nrhs) {
        const int L = static_cast<int>(meshes.size());
        std::vector<SparseOperator> A(L), P(L), R(L);
        std::vector<std::vector<double>> w(L);
        for (int k = 0; k + 1 < L; ++k) {
            P[k] = matrix_of(maps[k]).transposed("prolongation");
            R[k] = restriction_matrix(maps[k]);
        }
        for (int k = 0; k < L; ++k) {
            const DualGeometry dual = build_dual(*meshes[k]);
            if (!opts.galerkin || k == 0) {
                LaplacianOperators ops = laplacian_0(*meshes[k], dual, opts.hodge);
                A[k] = std::move(ops.laplacian);
                w[k] = std::move(ops.dual_areas);
            } else {
                A[k] = R[k - 1].multiply(A[k - 1]).multiply(P[k - 1]);
                A[k].set_tag("laplacian0(galerkin)");
                w[k] = dual.dual_cell_area;
            }
        }
        std::vector<decmg_gpu_level_desc> d(L);
        for (int k = 0; k < L; ++k) {
            decmg_gpu_level_desc& x = d[k];
            x = decmg_gpu_level_desc{};
            x.nv = A[k].rows();
            x.L_row_ptr = A[k].row_ptr().data();
            x.L_col_idx = A[k].col_idx().data();
            x.L_values = A[k].csr_values().data();
            x.L_nnz = A[k].nnz();
            x.dual_areas = w[k].data();
            if (k + 1 < L) {
                x.P_row_ptr = P[k].row_ptr().data();
                x.P_col_idx = P[k].col_idx().data();
                x.P_values = P[k].csr_values().data();
                x.P_nnz = P[k].nnz();
                x.R_row_ptr = R[k].row_ptr().data();
                x.R_col_idx = R[k].col_idx().data();
                x.R_values = R[k].csr_values().data();
                x.R_nnz = R[k].nnz();
            }
        }
        decmg_gpu_config cfg{device, max_nrhs};
        decmg_gpu_ctx* c = nullptr;
        const int rc = decmg_gpu_create_from_levels(d.data(), L, 0, &cfg, &c);
        if (rc != DECMG_OK) detail::raise(rc, nullptr);
        return c;
    }
    std::vector<std::shared_ptr<const EmbeddedComplex2D>> meshes_;
#endif
    std::shared_ptr<decmg_gpu_ctx> ctx_{nullptr, Del{}};
    std::vector<MultigridLevel> levels_;
    bool on_device_ = true;
};

#ifdef DECMG_GPU_REFERENCE_TYPES
/// Convenience: hierarchy over a subdivision tower plus its base complex.
/// `use_levels` keeps only the finest `use_levels` meshes (0 = all), so the
/// coarse solve runs on a finer mesh (build_hierarchy, multigrid.cpp:325-341).
inline MultigridHierarchy build_hierarchy(const std::shared_ptr<const EmbeddedComplex2D>& base,
                                          const std::vector<SubdivisionResult>& tower, int use_levels = 0,
                                          const HierarchyOptions& opts = {}, int device = 0, int max_nrhs = 1) {
    std::vector<std::shared_ptr<const EmbeddedComplex2D>> meshes;
    std::vector<GeometricMap> maps;
    for (const auto& s : tower) {
        meshes.push_back(s.fine);
        maps.push_back(s.map);
    }
    meshes.push_back(base);
    if (use_levels > 0 && use_levels < static_cast<int>(meshes.size())) {
        meshes.resize(use_levels);
        maps.resize(use_levels - 1);
    }
    return MultigridHierarchy(std::move(meshes), maps, opts, device, max_nrhs);
}
#endif

struct SolveReport {
    std::vector<double> solution;
    std::vector<double> residual_history;    // per cycle / iteration
    std::vector<double> cumulative_seconds;  // same length as the history
    int iterations = 0;
    bool converged = false;
    bool stagnated = false;
    double final_relative_residual = 0.0;
    double wall_seconds = 0.0;
#ifdef DECMG_GPU_HAVE_JSON
    nlohmann::json config_echo;

    nlohmann::json to_json(bool include_solution = false) const {  // solvers.cpp:31-43
        nlohmann::json j;
        j["iterations"] = iterations;
        j["converged"] = converged;
        j["stagnated"] = stagnated;
        j["final_relative_residual"] = final_relative_residual;
        j["wall_seconds"] = wall_seconds;
        j["residual_history"] = residual_history;
        j["cumulative_seconds"] = cumulative_seconds;
        j["config"] = config_echo;
        if (include_solution) j["solution"] = solution;
        return j;
    }
#endif
    void write_residual_csv(const std::string& path) const {  // solvers.cpp:45-54
        std::FILE* f = std::fopen(path.c_str(), "w");
        if (!f) throw std::runtime_error("cannot open " + path + " for writing");
        std::fprintf(f, "cycle,rel_residual,cumulative_seconds\n");
        for (std::size_t i = 0; i < residual_history.size(); ++i) {
            const double t = i < cumulative_seconds.size() ? cumulative_seconds[i] : 0.0;
            std::fprintf(f, "%zu,%.17g,%.17g\n", i + 1, residual_history[i], t);
        }
        std::fclose(f);
    }
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
    rep.cumulative_seconds = detail::last_times(h.handle());
    rep.cumulative_seconds.resize(rep.residual_history.size());
    rep.iterations = done;
    rep.converged = done > 0 ? rep.residual_history.back() <= tol : fin <= tol;
    rep.final_relative_residual = fin;
    rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
#ifdef DECMG_GPU_HAVE_JSON
    rep.config_echo["solver"] = "gmg";
#endif
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
        reps[k].converged = done[k] > 0 ? reps[k].residual_history.back() <= tol : fin[k] <= tol;
        reps[k].final_relative_residual = fin[k];
        reps[k].wall_seconds = wall;
#ifdef DECMG_GPU_HAVE_JSON
        reps[k].config_echo["solver"] = "gmg";
#endif
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
    rep.cumulative_seconds = detail::last_times(h.handle());
    rep.cumulative_seconds.resize(rep.residual_history.size());
    rep.iterations = its;
    rep.converged = conv != 0;
    rep.final_relative_residual = fin;
    rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
#ifdef DECMG_GPU_HAVE_JSON
    rep.config_echo["solver"] = "gmg_pcg";
#endif
    return rep;
}

}  // namespace decmg
