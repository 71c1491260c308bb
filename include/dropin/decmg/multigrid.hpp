// Drop-in replacement for the reference header decmg/multigrid.hpp
// (/root/reference/proj/include/decmg/multigrid.hpp). Put this directory BEFORE
// the reference's include directory on the compiler's search path,
//     g++ -I<repo>/include/dropin -I<repo>/include -I<reference>/proj/include ...
// and every reference translation unit that includes "decmg/multigrid.hpp" or
// "decmg/solvers.hpp" (physics.cpp, the CLI, the tests) compiles UNCHANGED
// against the CUDA library: MultigridHierarchy, build_hierarchy, run_cycle,
// project_compatible, standard_plan, smooth, gmg_solve and
// gmg_preconditioned_cg then run on the GPU through libdecmg_gpu.so
// (include/decmg_gpu.hpp holds the definitions). The link line drops the
// reference's multigrid.o / solvers.o / direct.o and adds -ldecmg_gpu.
//
// The sparse-LU classes the reference declares in the same header
// (multigrid.hpp:16-54) are not part of the GPU path; they are declared here
// with the reference's interface so that callers holding one (ConvectionSetup,
// physics.hpp:95) still compile. Whoever needs them links an implementation
// (the reference's direct.cpp); the GPU hierarchy has its own coarse solve.
#pragma once

#ifndef DECMG_GPU_REFERENCE_TYPES
#define DECMG_GPU_REFERENCE_TYPES
#endif
#include "decmg_gpu.hpp"

#include <memory>
#include <optional>
#include <vector>

namespace decmg {

class PinnedDirectSolver {  // multigrid.hpp:20-37
public:
    PinnedDirectSolver();
    PinnedDirectSolver(const SparseOperator& A, std::vector<double> weights);
    ~PinnedDirectSolver();
    PinnedDirectSolver(PinnedDirectSolver&&) noexcept;
    PinnedDirectSolver& operator=(PinnedDirectSolver&&) noexcept;

    std::vector<double> solve(const std::vector<double>& b) const;
    bool ready() const { return impl_ != nullptr; }

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
    std::vector<double> weights_;
    double weight_total_ = 0.0;
};

class DirectSolver {  // multigrid.hpp:40-54
public:
    DirectSolver();
    explicit DirectSolver(const SparseOperator& A);
    ~DirectSolver();
    DirectSolver(DirectSolver&&) noexcept;
    DirectSolver& operator=(DirectSolver&&) noexcept;

    std::vector<double> solve(const std::vector<double>& b) const;
    bool ready() const { return impl_ != nullptr; }

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace decmg
