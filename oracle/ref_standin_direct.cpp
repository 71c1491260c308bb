// TEST INFRASTRUCTURE ONLY (oracle). Builder-written stand-in for the
// reference's proj/src/direct.cpp, which needs Eigen3 (absent in this image).
//
// It implements the interface declared at
//   /root/reference/proj/include/decmg/multigrid.hpp:20-53
// (PinnedDirectSolver / DirectSolver) with the contract the reference's own
// tests pin (proj/tests/test_multigrid.cpp:319-330: residual <= 1e-12,
// weighted mean <= 1e-10), but with the coarse-level algorithm this
// framework uses everywhere: projected weighted CG run to convergence
// (DESIGN.md "coarse solve"). The same arithmetic, in the same order, is in
// oracle/decmg_oracle.c (dec_coarse_cg) and in the CUDA coarse kernel, so
// the reference V-cycle linked with this file, the C oracle and the GPU all
// produce bit-identical coarse corrections.
//
// Semantics follow PinnedDirectSolver::solve (proj/src/direct.cpp:59-76):
// project the RHS to star0-weighted mean zero, solve, and return a
// weighted-mean-zero solution. Pinning vertex 0 is unnecessary for CG on the
// consistent singular system (the solution is unique up to the constant the
// final projection removes).

#include "decmg/multigrid.hpp"

#include <stdexcept>

namespace decmg {

namespace {

struct CsrCopy {
    int n = 0;
    std::vector<int> rp, ci;
    std::vector<double> v;
};

CsrCopy copy_csr(const SparseOperator& A) {
    if (A.rows() != A.cols()) throw std::invalid_argument("direct solver: square matrix required");
    CsrCopy c;
    c.n = A.rows();
    c.rp = A.row_ptr();
    c.ci = A.col_idx();
    c.v = A.csr_values();
    return c;
}

// Projected weighted CG; arithmetic order documented in DESIGN.md and mirrored
// by dec_coarse_cg (oracle/decmg_oracle.c) and coarse_cg_kernel (CUDA).
// The stand-in's sums: index order from 0.0 for n <= 32 terms, else a
// fixed-shape tree (chunks of 256, zero-padded, folded pairwise, then the
// chunk sums the same way) -- the device's grid CG order.
double standin_sum(std::vector<double>& q, std::size_t n) {
    if (n <= 32) {
        double s = 0.0;
        for (std::size_t i = 0; i < n; ++i) s += q[i];
        return s;
    }
    while (n > 1) {
        const std::size_t nc = (n + 255) / 256;
        for (std::size_t c = 0; c < nc; ++c) {
            double t[256];
            for (std::size_t j = 0; j < 256; ++j) t[j] = c * 256 + j < n ? q[c * 256 + j] : 0.0;
            for (int h = 128; h >= 1; h >>= 1)
                for (int j = 0; j < h; ++j) t[j] = t[j] + t[j + h];
            q[c] = t[0];
        }
        n = nc;
    }
    return q[0];
}

std::vector<double> coarse_cg(const CsrCopy& A, const std::vector<double>& w, double wtotal,
                              const std::vector<double>& b, bool project) {
    const int n = A.n;
    std::vector<double> rhs(b), q(n);
    if (project) {
        for (int i = 0; i < n; ++i) q[i] = w[i] * b[i];
        const double m = standin_sum(q, n) / wtotal;
        for (int i = 0; i < n; ++i) rhs[i] = b[i] - m;
    }
    std::vector<double> x(n, 0.0), r(rhs), p(rhs), Ap(n);
    for (int i = 0; i < n; ++i) q[i] = (w[i] * r[i]) * r[i];
    double rr = standin_sum(q, n);
    const double rr0 = rr;
    const int maxit = 4 * n + 20;
    for (int it = 0; it < maxit; ++it) {
        if (!(rr > 1e-30 * rr0)) break;
        for (int i = 0; i < n; ++i) {
            double s = 0.0;
            for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) s += A.v[k] * p[A.ci[k]];
            Ap[i] = s;
        }
        for (int i = 0; i < n; ++i) q[i] = (w[i] * p[i]) * Ap[i];
        const double curv = standin_sum(q, n);
        if (curv == 0.0) break;
        const double alpha = rr / curv;
        for (int i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] = r[i] - alpha * Ap[i];
        for (int i = 0; i < n; ++i) q[i] = (w[i] * r[i]) * r[i];
        const double rn = standin_sum(q, n);
        const double beta = rn / rr;
        for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        rr = rn;
    }
    if (project) {
        for (int i = 0; i < n; ++i) q[i] = w[i] * x[i];
        const double ym = standin_sum(q, n) / wtotal;
        for (int i = 0; i < n; ++i) x[i] = x[i] - ym;
    }
    return x;
}

} // namespace

// Harness entry (oracle/ref_harness.cpp): the same CG for the Dirichlet
// extension's unpinned coarse solve (weights = dual areas, no projection).
std::vector<double> standin_coarse_cg(const SparseOperator& A, const std::vector<double>& w,
                                      const std::vector<double>& b, bool project) {
    double wt = 0.0;
    for (double x : w) wt += x;
    return coarse_cg(copy_csr(A), w, wt, b, project);
}

struct PinnedDirectSolver::Impl {
    CsrCopy A;
};

PinnedDirectSolver::PinnedDirectSolver(const SparseOperator& A, std::vector<double> weights)
    : impl_(new Impl), weights_(std::move(weights)) {
    if (static_cast<int>(weights_.size()) != A.rows()) {
        throw std::invalid_argument("PinnedDirectSolver: weight length mismatch");
    }
    weight_total_ = 0.0;
    for (double w : weights_) weight_total_ += w;
    impl_->A = copy_csr(A);
}

PinnedDirectSolver::PinnedDirectSolver() = default;
PinnedDirectSolver::~PinnedDirectSolver() = default;
PinnedDirectSolver::PinnedDirectSolver(PinnedDirectSolver&&) noexcept = default;
PinnedDirectSolver& PinnedDirectSolver::operator=(PinnedDirectSolver&&) noexcept = default;

std::vector<double> PinnedDirectSolver::solve(const std::vector<double>& b) const {
    return coarse_cg(impl_->A, weights_, weight_total_, b, true);
}

struct DirectSolver::Impl {
    CsrCopy A;
    std::vector<double> ones;
};

DirectSolver::DirectSolver(const SparseOperator& A) : impl_(new Impl) {
    impl_->A = copy_csr(A);
    impl_->ones.assign(A.rows(), 1.0);
}

DirectSolver::DirectSolver() = default;
DirectSolver::~DirectSolver() = default;
DirectSolver::DirectSolver(DirectSolver&&) noexcept = default;
DirectSolver& DirectSolver::operator=(DirectSolver&&) noexcept = default;

std::vector<double> DirectSolver::solve(const std::vector<double>& b) const {
    return coarse_cg(impl_->A, impl_->ones, static_cast<double>(b.size()), b, false);
}

} // namespace decmg
