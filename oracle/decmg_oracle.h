/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle (checker) for the DEC geometric
 * multigrid V-cycle. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference leg may load it; the product (libdecmg_gpu.so)
 * never links or calls it.
 *
 * A plain-C restatement of the reference algorithm (arxiv/paper_2508_12501,
 * C++ `decmg` under /root/reference/proj), single-threaded, compiled with
 * -ffp-contract=off so every floating-point expression rounds exactly like
 * the reference built with the same flags. Each function in decmg_oracle.c
 * cites the reference file:line it restates. It is pinned against golden
 * vectors produced by the reference itself (oracle/_ref/ref_harness ->
 * tests/golden/, generator tests/golden/make_golden.py).
 */
#ifndef DECMG_ORACLE_H
#define DECMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_hier orc_hier;

/* base: "square" (make_triangulated_grid(1,1,1,1)), "ico" (canonical
 * icosahedron, projected subdivision), "grid:nx:ny:lx:ly", "equi:rows:cols:side".
 * nsub binary subdivisions; dirichlet != 0 applies the x1 extension. */
orc_hier* orc_build(const char* base, int nsub, int dirichlet);
void orc_free(orc_hier* h);
const char* orc_last_error(void);

int orc_levels(const orc_hier* h);
/* counts[0..3] = nv, ne, nt, nnz(L); hash = EmbeddedComplex2D::hash() */
void orc_level_info(const orc_hier* h, int k, int64_t* counts, uint64_t* hash);
/* name: "positions" f64[nv*3], "edges" i32[ne*2], "triangles" i32[nt*3],
 * "dual_areas" f64[nv], "boundary" i32[nv], "L_rp" i32[nv+1], "L_ci" i32[nnz],
 * "L_v" f64[nnz], "P_rp" "P_ci" "P_v", "R_rp" "R_ci" "R_v" (k < levels-1),
 * "nnzP" / "nnzR" via orc_level_nnz. Returns element count or -1. */
int64_t orc_get(const orc_hier* h, int k, const char* name, void* out);
int64_t orc_level_nnz(const orc_hier* h, int k, const char* op);

/* mt19937_64-based synthetic right-hand sides (x3 extension):
 * kind "uniform" (2u-1), "ylm" (Y_3^2 + 1e-3 N(0,1)), "sinsin", "lr" (L*u). */
int orc_rhs(const orc_hier* h, const char* kind, uint64_t seed, double* out);
void orc_project(const orc_hier* h, double* b);                /* project_compatible */
void orc_spmv(const orc_hier* h, int k, const char* op, const double* x, double* y);
double orc_norm2(const double* a, int64_t n);                  /* kernels::norm2 */
uint64_t orc_fnv(const void* data, int64_t nbytes);

/* smoother: 0 = weighted Jacobi (omega), 1 = Gauss-Seidel (forward),
 * 2 = symmetric Gauss-Seidel (forward + reverse per iteration).
 * walk: string of 'd'/'u' (NULL = V-cycle); pre/post sweeps uniform. */
int orc_run_cycles(const orc_hier* h, const char* walk, int pre, int post, int smoother,
                   double omega, const double* b, const double* x0, int ncycles,
                   double* x_out, double* hist_out);
int orc_solve(const orc_hier* h, int pre, int post, int smoother, double omega,
              const double* b, double tol, int max_cycles, double* x_out, double* hist_out,
              int* iters_out, double* final_out);
void orc_coarse_solve(const orc_hier* h, const double* b, double* x);
/* smooth (multigrid.cpp:95-120) on level k's Laplacian, x in place; smoother as above, 3 = cg_fixed
 * with the level's dual areas as weights. Returns nonzero on a zero diagonal. */
int orc_smooth(const orc_hier* h, int k, int smoother, double omega, int iters, const double* b, double* x);
/* gmg_preconditioned_cg (proj/src/solvers.cpp:118-130): hist_out needs
 * maxiter + 1 entries; returns -2 on a CG breakdown (message in last_error). */
int orc_pcg(const orc_hier* h, const char* walk, int pre, int post, int smoother, double omega, int ncycles,
            const double* b, double tol, int maxiter, double* x_out, double* hist_out, int* iters_out,
            double* final_out);

#ifdef __cplusplus
}
#endif
#endif
