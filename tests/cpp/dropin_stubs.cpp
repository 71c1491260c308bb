// Link-time stand-ins for the reference solvers that are NOT on the GPU path,
// for reference callers compiled against include/dropin (see
// include/dropin/decmg/solvers.hpp): the sparse-LU classes (direct.cpp, needs
// Eigen) and the hierarchy-free Krylov solvers (solvers.cpp weighted_cg,
// gmres). A caller that selects one of them gets a std::logic_error instead
// of a silent CPU route; the Gmg and GmgPcg solver kinds never reach these.
#include "decmg/solvers.hpp"

#include <stdexcept>

namespace decmg {

struct PinnedDirectSolver::Impl {};
PinnedDirectSolver::PinnedDirectSolver() = default;
PinnedDirectSolver::PinnedDirectSolver(const SparseOperator&, std::vector<double>) {
    throw std::logic_error("PinnedDirectSolver: not part of the GPU drop-in (link the reference's direct.cpp)");
}
PinnedDirectSolver::~PinnedDirectSolver() = default;
PinnedDirectSolver::PinnedDirectSolver(PinnedDirectSolver&&) noexcept = default;
PinnedDirectSolver& PinnedDirectSolver::operator=(PinnedDirectSolver&&) noexcept = default;
std::vector<double> PinnedDirectSolver::solve(const std::vector<double>&) const {
    throw std::logic_error("PinnedDirectSolver: not part of the GPU drop-in");
}

struct DirectSolver::Impl {};
DirectSolver::DirectSolver() = default;
DirectSolver::DirectSolver(const SparseOperator&) {
    throw std::logic_error("DirectSolver: not part of the GPU drop-in (link the reference's direct.cpp)");
}
DirectSolver::~DirectSolver() = default;
DirectSolver::DirectSolver(DirectSolver&&) noexcept = default;
DirectSolver& DirectSolver::operator=(DirectSolver&&) noexcept = default;
std::vector<double> DirectSolver::solve(const std::vector<double>&) const {
    throw std::logic_error("DirectSolver: not part of the GPU drop-in");
}

SolveReport weighted_cg(const SparseOperator&, const std::vector<double>&, const std::vector<double>&, double, int,
                        const std::function<std::vector<double>(const std::vector<double>&)>*,
                        const std::vector<double>*) {
    throw std::logic_error("weighted_cg: not part of the GPU drop-in (link the reference's solvers.cpp)");
}

SolveReport gmres(const SparseOperator&, const std::vector<double>&,
                  const std::function<std::vector<double>(const std::vector<double>&)>*, int, double, int,
                  const std::vector<double>*) {
    throw std::logic_error("gmres: not part of the GPU drop-in (link the reference's solvers.cpp)");
}

}  // namespace decmg
