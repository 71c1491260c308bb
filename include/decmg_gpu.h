/*
 * decmg_gpu -- B200-native (sm_100a) geometric multigrid for the DEC 0-form
 * Poisson problem on nested binary-subdivided triangle meshes.
 *
 * C ABI (plain pointers and sizes, no exceptions, no torch types). This is the
 * drop-in boundary for the reference C++ library `decmg`
 * (/root/reference/proj); every entry point names the reference interface it
 * replaces. A header-only C++ shim with the reference's own class/function
 * names and exception types is in include/decmg_gpu.hpp; INTEGRATION.md shows
 * how a reference user binds it.
 *
 * Conventions
 *  - Status codes: DECMG_OK (0) or one of the error classes below; the message
 *    is available from decmg_gpu_last_error(ctx) (or decmg_gpu_last_error(NULL)
 *    when creation failed).
 *  - Vectors are row-major [n][nrhs] fp64 (the nrhs right-hand sides of one
 *    vertex are adjacent). nrhs = 1 is the reference's single-vector case.
 *  - Host-pointer entry points copy in/out synchronously and retain no pointer.
 *    `_dev` entry points take device pointers and only enqueue work on the
 *    context's stream (decmg_gpu_stream).
 *  - Level 0 is the finest level (reference order, proj/src/multigrid.cpp:196).
 *  - One in-flight call per context; several contexts may run concurrently.
 */
#ifndef DECMG_GPU_H
#define DECMG_GPU_H

#include <stdint.h>

#if defined(__GNUC__)
#define DECMG_API __attribute__((visibility("default")))
#else
#define DECMG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct decmg_gpu_ctx decmg_gpu_ctx;

enum {
    DECMG_OK = 0,
    DECMG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    DECMG_RUNTIME = 2,          /* std::runtime_error in the reference     */
    DECMG_CUDA = 3,
    DECMG_NCCL = 4,
    DECMG_OOM = 5
};

/* creation flags */
#define DECMG_PROJECT_SPHERE 1u /* push new midpoints to the unit sphere (x2)   */
#define DECMG_DIRICHLET 2u      /* identity rows on boundary vertices (x1)      */
#define DECMG_CUBIC 4u          /* SubdivisionScheme::Cubic (1 -> 9, subdivision.cpp:116-120) instead of Binary */
#define DECMG_CLAMP_DUAL_AREAS 8u /* HodgeOptions::clamp_dual_areas (operators.hpp:31-35, operators.cpp:80-114) */

typedef struct {
    int device;   /* CUDA device ordinal                                    */
    int max_nrhs; /* largest batch run_cycles/solve will see (1..32)        */
} decmg_gpu_config;

/* Hierarchy construction on the device: replaces
 *   subdivision_tower (proj/src/subdivision.cpp:127-139) +
 *   build_hierarchy / MultigridHierarchy ctor (proj/src/multigrid.cpp:196-238,325-341)
 * including from_triangles (mesh.cpp:122-157), build_dual (dual.cpp:7-63),
 * laplacian_0 (operators.cpp:102-122), matrix_of/transposed (multigrid.cpp:215)
 * and restriction_matrix (geometric_map.cpp:205-223).
 * `positions` [nv][3], `corner_triples` [nt][3] describe the base complex
 * (as passed to EmbeddedComplex2D::from_triangles); nsub binary subdivisions. */
DECMG_API int decmg_gpu_create_from_base(const double* positions, int nv, const int* corner_triples, int nt,
                               int nsub, unsigned flags, const decmg_gpu_config* cfg,
                               decmg_gpu_ctx** out);

/* The same with build_hierarchy's use_levels (multigrid.cpp:325-341): keep
 * only the finest use_levels meshes of the tower (0 = all), so the coarse
 * solve runs on a finer mesh. */
DECMG_API int decmg_gpu_create_from_base_ex(const double* positions, int nv, const int* corner_triples, int nt,
                                           int nsub, int use_levels, unsigned flags, const decmg_gpu_config* cfg,
                                           decmg_gpu_ctx** out);

/* Upload an already assembled hierarchy (reference layout: CSR of L per level,
 * P = prolongation n_k x n_{k+1}, R = restriction n_{k+1} x n_k, dual areas).
 * Replaces MultigridHierarchy(meshes, maps) for callers that assemble on the
 * host. boundary may be NULL (Neumann). */
typedef struct {
    int nv;
    const int* L_row_ptr;
    const int* L_col_idx;
    const double* L_values;
    int64_t L_nnz;
    const double* dual_areas;
    const int* boundary;
    const int* P_row_ptr; /* NULL on the coarsest level */
    const int* P_col_idx;
    const double* P_values;
    int64_t P_nnz;
    const int* R_row_ptr;
    const int* R_col_idx;
    const double* R_values;
    int64_t R_nnz;
} decmg_gpu_level_desc;
DECMG_API int decmg_gpu_create_from_levels(const decmg_gpu_level_desc* levels, int nlevels, unsigned flags,
                                 const decmg_gpu_config* cfg, decmg_gpu_ctx** out);

DECMG_API void decmg_gpu_destroy(decmg_gpu_ctx* ctx);
DECMG_API const char* decmg_gpu_last_error(const decmg_gpu_ctx* ctx);

/* CyclePlan (proj/include/decmg/multigrid.hpp:70-89); a NULL plan pointer is
 * standard_plan(levels, CycleKind::V) with the reference defaults (V(3,3),
 * Gauss-Seidel, multigrid.hpp:58,88-89). walk: 'd'/'u' string
 * (NULL = the V walk of standard_plan, multigrid.cpp:171-194); pre/post:
 * per-level sweep counts (NULL = pre_all/post_all on every level).
 * smoother (SmootherConfig, multigrid.hpp:55-60; smooth, multigrid.cpp:95-120):
 * weighted Jacobi, Gauss-Seidel (forward lexicographic, bit-identical to the
 * sequential sweep via a level schedule), symmetric Gauss-Seidel (forward +
 * reverse per iteration) or the fixed-iteration CG smoother (cg_fixed,
 * multigrid.cpp:63-91; deterministic tree dots, so within rounding of the
 * reference's sequential ones). The partitioned solve (decmg_gpu_dist_*) runs
 * Jacobi only. */
enum { DECMG_SMOOTHER_JACOBI = 0, DECMG_SMOOTHER_GS = 1, DECMG_SMOOTHER_SGS = 2, DECMG_SMOOTHER_CG = 3 };
typedef struct {
    const char* walk;
    const int* pre;
    const int* post;
    int pre_all;
    int post_all;
    int smoother;
    double jacobi_omega;
} decmg_gpu_plan;

/* MultigridHierarchy::run_cycle (proj/src/multigrid.cpp:287-323): ncycles
 * cycles from x0 (NULL = zeros); x_out [n0][nrhs]; hist_out [ncycles][nrhs]
 * = fine relative residual after each cycle. */
DECMG_API int decmg_gpu_run_cycles(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs, const double* b,
                         const double* x0, int ncycles, double* x_out, double* hist_out);

/* gmg_solve (proj/src/solvers.cpp:251-279): projects b (Neumann), repeats
 * one-cycle runs until every RHS has relative residual <= tol or max_cycles.
 * hist_out [max_cycles][nrhs] (rows past *cycles_done untouched);
 * final_out [nrhs] = recomputed final relative residual. */
DECMG_API int decmg_gpu_solve(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs, const double* b,
                    const double* x0, double tol, int max_cycles, double* x_out, double* hist_out,
                    int* cycles_done, double* final_out);

/* A stream of nbatch independent gmg_solve calls (extension x6: no reference
 * counterpart; a caller would otherwise loop over decmg_gpu_solve). Batch k =
 * host arrays b[k] -> x_out[k] ([n][nrhs] each, pinned memory for overlap),
 * every batch bit-identical to its own decmg_gpu_solve; batch k+1's upload and
 * projection and batch k-1's download run on copy/auxiliary streams while
 * batch k cycles. hist_out [nbatch][max_cycles][nrhs], cycles_done and
 * final_out [nbatch][nrhs] (each may be NULL). x0 = 0. */
DECMG_API int decmg_gpu_solve_batches(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs, int nbatch,
                                      const double* const* b, double tol, int max_cycles, double* const* x_out,
                                      double* hist_out, int* cycles_done, double* final_out);

/* gmg_preconditioned_cg (proj/src/solvers.cpp:118-130): weighted CG
 * (solvers.cpp:56-116, dual-area weights) preconditioned by inner_cycles
 * cycles of the inner plan from zero; projects b (Neumann hierarchies only).
 * hist_out [maxiter+1][nrhs] (entry 0 = initial residual; rows past
 * iters_out[l] of lane l untouched); iters_out, converged_out, final_out
 * [nrhs] (final = recomputed relative residual of the solution). Weighted
 * dots are deterministic trees, not the reference's sequential sums: iterates
 * agree to rounding, histories within 1e-10. A CG
 * breakdown returns DECMG_RUNTIME with the reference's message. */
DECMG_API int decmg_gpu_pcg(decmg_gpu_ctx* ctx, const decmg_gpu_plan* inner, int inner_cycles, int nrhs,
                            const double* b, double tol, int maxiter, double* x_out, double* hist_out,
                            int* iters_out, int* converged_out, double* final_out);

/* Device-pointer variants (inputs already resident in HBM). hist/final are
 * device arrays too. */
DECMG_API int decmg_gpu_run_cycles_dev(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs,
                             const double* d_b, const double* d_x0, int ncycles, double* d_x,
                             double* d_hist);
DECMG_API void* decmg_gpu_stream(decmg_gpu_ctx* ctx); /* cudaStream_t of the context */

/* MultigridHierarchy::project_compatible (proj/src/multigrid.cpp:240-250), in place. */
DECMG_API int decmg_gpu_project_compatible(decmg_gpu_ctx* ctx, int nrhs, double* b);

/* smooth (proj/include/decmg/multigrid.hpp:66-68, src/multigrid.cpp:95-120)
 * with A = level k's Laplacian: iters sweeps of `smoother` (DECMG_SMOOTHER_*,
 * omega for Jacobi) on x in place ([n_k][nrhs], reference numbering).
 * weighted != 0: the CG smoother's inner product uses the level's dual areas
 * (what cycle_once passes), else plain dots (smooth's default weights = {}).
 * Errors as the reference: zero diagonal -> DECMG_RUNTIME. */
DECMG_API int decmg_gpu_smooth(decmg_gpu_ctx* ctx, int level, int smoother, double omega, int iters, int nrhs,
                               double* x, const double* b, int weighted);

/* SolveReport::cumulative_seconds (proj/include/decmg/solvers.hpp:20) of the
 * last decmg_gpu_solve / decmg_gpu_pcg on ctx: seconds since the call began
 * at which each cycle's (iteration's) residual was known; for a batch, the
 * cycles of the longest lane. Returns the count (query with out = NULL). */
DECMG_API int decmg_gpu_last_times(const decmg_gpu_ctx* ctx, double* out, int max);

/* SparseOperator::apply (proj/src/sparse.cpp:209-218) of level k's operator
 * op = 'L' (n_k x n_k), 'P' (n_k x n_{k+1}), 'R' (n_{k+1} x n_k). */
DECMG_API int decmg_gpu_apply(decmg_gpu_ctx* ctx, int level, char op, const double* x, double* y);

/* Structure export for parity. counts = {nv, ne, nt, nnz(L), nnz(P), nnz(R)}.
 * name: positions, edges, triangles, corners, dual_areas, boundary, diag,
 * L_row_ptr, L_col_idx, L_values, P_*, R_*, order (the Morton row order of the
 * level's ELL operators: row q is vertex order[q]). Returns the element count (query
 * with out = NULL) or -1. hash = EmbeddedComplex2D::hash (mesh.cpp:112-119). */
DECMG_API int decmg_gpu_levels(const decmg_gpu_ctx* ctx);
DECMG_API int decmg_gpu_level_info(decmg_gpu_ctx* ctx, int level, int64_t counts[6]);
DECMG_API int64_t decmg_gpu_export(decmg_gpu_ctx* ctx, int level, const char* name, void* out);
DECMG_API int decmg_gpu_mesh_hash(decmg_gpu_ctx* ctx, int level, uint64_t* hash);

/* Per-kernel device timing (CUDA events around every launch when enabled).
 * Kernel classes: 0 level-0 sweep, 1 level-0 residual, 2 level-0 restrict,
 * 3 level-0 prolong, 4 coarser-level work, 5 coarse solve, 6 norms and
 * projections, 7 zero-start sweeps. cls = -1 resets the accumulators.
 * bytes = algorithmic bytes of the launches. */
DECMG_API int decmg_gpu_set_timing(decmg_gpu_ctx* ctx, int enable);
DECMG_API int decmg_gpu_get_timing(decmg_gpu_ctx* ctx, int cls, int64_t* launches, double* total_ms,
                         double* bytes);
DECMG_API int64_t decmg_gpu_launch_count(decmg_gpu_ctx* ctx); /* kernels launched since creation */
/* Diagnostic of the exact parallel projection chain (project_compatible): how many
 * (256-row segment, RHS) pairs ran the literal sequential add chain since creation (the rest were
 * applied in O(1) on their binade's integer grid). -1 on error. */
DECMG_API int64_t decmg_gpu_projection_fallbacks(decmg_gpu_ctx* ctx);

/* Input generators (extension x3): base meshes and synthetic RHS.
 * base_mesh spec: "square", "ico", "grid:nx:ny:lx:ly", "equi:rows:cols:side".
 * Query sizes with positions = corners = NULL. */
DECMG_API int decmg_base_mesh(const char* spec, double* positions, int* nv, int* corners, int* nt);

/* Mesh and operator files (proj/src/mesh_io.cpp:19-82, sparse.cpp:247-259).
 * read_obj: "v x y z" / "f i j k" (1-based) records; query sizes with
 * positions = corners = NULL; errors carry the reference's messages
 * (decmg_io_last_error). write_obj / write_matrix_market write level k's
 * complex or its L, P, R ('L', 'P', 'R'; tags laplacian0 / prolongation /
 * restriction) byte-for-byte as the reference's writers do. */
DECMG_API const char* decmg_io_last_error(void);
DECMG_API int decmg_read_obj(const char* path, double* positions, int* nv, int* corners, int* nt);
DECMG_API int decmg_gpu_write_obj(decmg_gpu_ctx* ctx, int level, const char* path);
DECMG_API int decmg_gpu_write_matrix_market(decmg_gpu_ctx* ctx, int level, char op, const char* path);
/* kind: "uniform" (2u-1), "ylm" (Y_3^2 + 1e-3 N(0,1)), "sinsin", "lr" (L*u);
 * RHS j uses seed + j. Writes [n0][nrhs]. Dirichlet contexts zero boundary rows. */
DECMG_API int decmg_gpu_make_rhs(decmg_gpu_ctx* ctx, const char* kind, uint64_t seed, int nrhs, double* b);


/* ---- Vertex-partitioned multi-GPU V-cycle ----
 * The reference has no distribution; this is the north star's
 * "vertex set partitioned across 1/2/4/8 GPUs". Every rank builds the full
 * hierarchy; level-0 vertices are split into contiguous ranges of the Morton
 * row order (coarse vertices follow their fine copies); levels with >=
 * agglomerate_below vertices per rank are partitioned with 1-ring halos,
 * coarser levels run replicated on every rank. Iterates are bit-identical to
 * the single-GPU solve for any rank count; residual histories agree within
 * rounding (per-rank partial sums added in rank order).
 * Transports:
 *   DECMG_DIST_EMULATE  all world_size ranks inside this process on
 *                       cfg->device (device copies; rank is ignored)
 *   DECMG_DIST_NCCL     one process per GPU; nccl_id = the 128-byte
 *                       ncclUniqueId from decmg_gpu_nccl_unique_id on rank 0
 *   DECMG_DIST_SHM      one process per rank, host-staged halos through the
 *                       file shm_path (same path on every rank, e.g. under
 *                       /dev/shm; created if absent, must start empty) with a
 *                       host barrier; ranks may share one GPU. */
typedef struct decmg_gpu_dist decmg_gpu_dist;
enum { DECMG_DIST_EMULATE = 0, DECMG_DIST_NCCL = 1, DECMG_DIST_SHM = 2 };
typedef struct {
    int kind;
    const void* nccl_id;
    const char* shm_path;
} decmg_gpu_dist_transport;
DECMG_API int decmg_gpu_nccl_unique_id(void* out, int bytes);
DECMG_API int decmg_gpu_dist_create_ex(const double* positions, int nv, const int* corner_triples, int nt, int nsub,
                                       unsigned flags, const decmg_gpu_config* cfg, int world_size, int rank,
                                       const decmg_gpu_dist_transport* transport, int agglomerate_below,
                                       decmg_gpu_dist** out);
/* nccl_id == NULL: emulation; otherwise NCCL (decmg_gpu_dist_create_ex). */
DECMG_API int decmg_gpu_dist_create(const double* positions, int nv, const int* corner_triples, int nt, int nsub,
                                    unsigned flags, const decmg_gpu_config* cfg, int world_size, int rank,
                                    const void* nccl_id, int agglomerate_below, decmg_gpu_dist** out);
DECMG_API void decmg_gpu_dist_destroy(decmg_gpu_dist* d);
DECMG_API const char* decmg_gpu_dist_last_error(const decmg_gpu_dist* d);
DECMG_API int decmg_gpu_dist_info(const decmg_gpu_dist* d, int* agglomeration_level, int* levels, int64_t* owned0,
                                  int64_t* halo0);
/* The full (replicated) hierarchy of this rank: every single-context entry
 * point (make_rhs, export, apply, timing, ...) works on it; owned by d. */
DECMG_API decmg_gpu_ctx* decmg_gpu_dist_context(decmg_gpu_dist* d);
/* CUDA-event time of the last decmg_gpu_dist_run's cycle loop on this rank
 * (cycles + per-cycle residual norms; excludes input staging, projection and
 * the solution gather), and the kernel launches of this rank so far. */
DECMG_API double decmg_gpu_dist_last_cycle_ms(const decmg_gpu_dist* d);
DECMG_API int64_t decmg_gpu_dist_launch_count(const decmg_gpu_dist* d);
/* run_cycle (solve == 0, ncycles = max_cycles) or gmg_solve (solve != 0) with
 * full-length host vectors replicated on every rank; x_out receives the full
 * solution on every rank. Weighted Jacobi only. */
DECMG_API int decmg_gpu_dist_run(decmg_gpu_dist* d, const decmg_gpu_plan* plan, int nrhs, const double* b,
                                 const double* x0, int max_cycles, int solve, double tol, double* x_out,
                                 double* hist_out, int* cycles_done, double* final_out);

#ifdef __cplusplus
}
#endif
#endif
