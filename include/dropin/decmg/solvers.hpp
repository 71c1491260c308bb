// Drop-in replacement for the reference header decmg/solvers.hpp
// (/root/reference/proj/include/decmg/solvers.hpp); see multigrid.hpp in this
// directory. SolveReport, gmg_solve (solvers.hpp:57-59) and
// gmg_preconditioned_cg (solvers.hpp:44-46) are the GPU shim's. The Krylov
// solvers that do not use the multigrid hierarchy (weighted_cg, gmres;
// solvers.hpp:32-55) are outside the GPU path: they are declared with the
// reference's signatures and resolved at link time by whatever the caller
// links (the reference's own definitions, or a stub that throws).
#pragma once

#include "decmg/multigrid.hpp"
#include "decmg/sparse.hpp"

#include <functional>
#include <string>
#include <vector>

namespace decmg {

SolveReport weighted_cg(const SparseOperator& A, const std::vector<double>& weights,
                        const std::vector<double>& b, double tol, int maxiter,
                        const std::function<std::vector<double>(const std::vector<double>&)>*
                            preconditioner = nullptr,
                        const std::vector<double>* x0 = nullptr);

SolveReport gmres(const SparseOperator& A, const std::vector<double>& b,
                  const std::function<std::vector<double>(const std::vector<double>&)>*
                      preconditioner,
                  int restart, double tol, int maxiter,
                  const std::vector<double>* x0 = nullptr);

}  // namespace decmg
