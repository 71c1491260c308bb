// decmg_gpu internals shared by setup.cu, cycle.cu and capi.cu.
//
// All translation units are compiled with --fmad=false (see Makefile): the
// reference is compiled with -ffp-contract=off, and every floating-point
// expression below is written in the reference's evaluation order, so the
// device produces the reference's bits.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/decmg_gpu.h"

namespace decmg_gpu {

// Row ids of the padded ELL operators (Le_row / Re_row) carry the slot of
// the row's diagonal entry in bits kRowBits..30; -1 marks a padding row.
constexpr int kRowBits = 28;

// Error propagation without exceptions across the ABI.
struct Status {
    int code = DECMG_OK;
    std::string msg;
    bool ok() const { return code == DECMG_OK; }
    static Status Ok() { return {}; }
    static Status Err(int c, std::string m) { return {c, std::move(m)}; }
};

inline Status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return Status::Ok();
    const int code = e == cudaErrorMemoryAllocation ? DECMG_OOM : DECMG_CUDA;
    return Status::Err(code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define DG_TRY(expr)                         \
    do {                                     \
        ::decmg_gpu::Status _s = (expr);     \
        if (!_s.ok()) return _s;             \
    } while (0)
#define DG_CUDA(call) DG_TRY(::decmg_gpu::cuda_status((call), #call))

// One level of the hierarchy, device resident. Finest level is index 0.
struct Level {
    int nv = 0, ne = 0, nt = 0;
    // complex (EmbeddedComplex2D, proj/include/decmg/mesh.hpp:32-86)
    double* pos = nullptr;   // [nv][3]
    int* edges = nullptr;    // [ne][2] src < tgt, lexicographic
    int* tris = nullptr;     // [nt][3] (e0,e1,e2), e_i opposite corner i
    int* corners = nullptr;  // [nt][3] (v0,v1,v2)
    int* eptr = nullptr;     // [nv+1] edges with src == v
    int* ve_ptr = nullptr;   // [nv+1] vertex -> incident edges (ascending)
    int* ve = nullptr;       // [2 ne]
    // operators
    double* area = nullptr;  // dual cell areas (star0 diagonal)
    int* bd = nullptr;       // boundary flag (extension x1)
    double* diag = nullptr;  // L_ii
    int* L_rp = nullptr;
    int* L_ci = nullptr;
    double* L_v = nullptr;
    int64_t nnzL = 0;
    // transfers to the next coarser level (absent on the coarsest)
    int* P_rp = nullptr;
    int* P_ci = nullptr;
    double* P_v = nullptr;
    int64_t nnzP = 0;
    int* R_rp = nullptr;
    int* R_ci = nullptr;
    double* R_v = nullptr;
    int64_t nnzR = 0;
    // Internal numbering: the V-cycle stores every
    // vector of a level in the Morton order of its vertex positions -- row q
    // of x, b, r is vertex ord[q] -- so row passes stream their own rows and
    // the x gathers stay local. The *o operators are the reference operators
    // renumbered on both sides (row q = reference row ord[q], columns mapped
    // through inv of the column level) with every row's entries kept in the
    // reference order, so each row sum is bit-identical. ord == nullptr:
    // identity (the coarsest level, hierarchies without positions). The API
    // keeps the reference numbering; level-0 vectors are permuted at the
    // boundary (driver.cuh to_internal / from_internal).
    int* ord = nullptr;      // [nv] internal row -> vertex
    int* inv = nullptr;      // [nv] vertex -> internal row
    double* diag_i = nullptr;  // L_ii by internal row (== diag without ord)
    double* area_i = nullptr;  // dual areas by internal row (== area without ord)
    int* bd_i = nullptr;       // boundary flag by internal row (== bd without ord)
    int* Lo_rp = nullptr;
    int* Lo_ci = nullptr;
    double* Lo_v = nullptr;
    int* Po_rp = nullptr;    // fine rows of P (internal), coarse columns (internal)
    int* Po_ci = nullptr;
    double* Po_v = nullptr;
    int* Ro_rp = nullptr;    // coarse rows of R (internal), fine columns (internal)
    int* Ro_ci = nullptr;
    double* Ro_v = nullptr;
    // Padded ELL copies of Lo (width 7/8), Po (width 2), Ro (width 7/8) used
    // when every row fits (nullptr otherwise): row q at [q*W, q*W + W),
    // padding entries (real column, value 0.0) after the real ones.
    int* Le_ci = nullptr;
    double* Le_v = nullptr;
    int* Pe_ci = nullptr;
    double* Pe_v = nullptr;
    int* Re_ci = nullptr;
    double* Re_v = nullptr;
    int Le_w = 0;            // ELL widths (7 or 8; 0 = no ELL copy)
    int Re_w = 0;
    int* Le_row = nullptr;   // row q | diag slot << kRowBits per ELL row of Le/Pe (-1 = padding)
    // Exact lexicographic Gauss-Seidel as a level schedule (setup.cu
    // build_gs_schedule): phase p of the forward (f) / reverse (r) sweep is
    // the internal rows gs?_rows[gs?_ptr[p] .. gs?_ptr[p+1]), ascending.
    int* gsf_rows = nullptr;
    int* gsr_rows = nullptr;
    std::vector<int> gsf_ptr, gsr_ptr;
    int* Re_row = nullptr;   // coarse row q per ELL row of Re (-1 = padding)
    // Plans of the two-sweep pass k_sweep_pair (driver.cuh prepare_pairs), one per tile shape
    // (rows per tile, set by the number of right-hand sides); grid == 0: the level keeps separate sweeps
    struct PairPlan {
        int rows = 0, ctas = 0, grid = 0, group = 0, ahead = 0, rounds = 0, ndefer = 0;  // ctas: CTAs per SM asked for
        int* ord2 = nullptr;      // Le_row with the deferred rows set to -1
        int* defer = nullptr;     // deferred ELL rows, ascending
        unsigned* count = nullptr;  // [rounds] round counters
    };
    std::vector<PairPlan> pair_plans;
    int zero_diag_row = -1;  // first row with L_ii == 0 (-1: none)
    double wtot = 0.0;       // sum of dual areas, sequential (coarse solve)
    // work vectors [nv][max_nrhs]
    double* x[2] = {nullptr, nullptr};
    int cur = 0;
    double* b = nullptr;     // level 0: the RHS in the internal numbering (driver.cuh to_internal)
    bool x_zero = false;     // x[cur] known to be exactly +0.0 (fresh descent)
};

struct Timing {
    bool enabled = false;
    struct Rec {
        int cls;
        double bytes;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    int64_t launches[8] = {};
    double ms[8] = {};
    double bytes[8] = {};
};

}  // namespace decmg_gpu

struct decmg_gpu_ctx {
    int device = 0;
    int max_nrhs = 1;
    unsigned flags = 0;
    bool dirichlet = false;
    cudaStream_t stream = nullptr;
    std::vector<decmg_gpu::Level> lv;
    double* r = nullptr;        // residual scratch [n0][max_nrhs]
    double* red = nullptr;      // reduction partials
    size_t red_cap = 0;         // doubles
    double* dsmall = nullptr;   // per-RHS device scalars (256 doubles)
    double* hsmall = nullptr;   // pinned host mirror
    double* hsmall_dev = nullptr;  // its device alias (mapped pinned memory)
    double* coarse_scratch = nullptr;
    double* cg_grid_buf = nullptr;  // coarse grid CG (n > 32): per-lane scalars + tree partials, on first use
    double* bproj = nullptr;    // projected RHS for solve [n0][max_nrhs]
    double* xsol = nullptr;     // solve snapshot [n0][max_nrhs]
    double* hist_dev = nullptr; // [hist_cap][max_nrhs]
    unsigned long long* tstamp_dev = nullptr;  // [hist_cap + 1] %globaltimer at the solve start / each check
    std::vector<double> last_times;  // SolveReport::cumulative_seconds of the last solve / pcg
    int hist_cap = 0;
    double* io_b = nullptr;     // staging for host-pointer calls [n0][max_nrhs]
    double* io_x0 = nullptr;
    double* io_x = nullptr;
    double* pcg_buf = nullptr;  // GMG-PCG vectors (pcg.cu), 5 x [n0][max_nrhs], allocated on first use
    double* pcg_s = nullptr;    // GMG-PCG per-lane scalars [8][32]
    double* cgs_buf = nullptr;  // CG smoother vectors r, p, Ap: 3 x [n0][max_nrhs], on first use
    double* cgs_s = nullptr;    // CG smoother per-lane scalars [6][32] + done flags
    double* seq_buf = nullptr;  // exact parallel projection chain scratch (seqsum.cuh), on first use
    int* seq_fallbacks = nullptr;  // device counter of segments that ran the literal chain
    int proj_seq = 0;           // literal single-lane projection chain instead (env DECMG_PROJ_SEQ=1)
    cudaStream_t io_stream = nullptr;        // chunked host copies (stage_rhs)
    // solve_batches (cycle.cu): second input/output buffers, staging and copy-out streams
    double* bproj2 = nullptr;
    double* io_x2 = nullptr;
    cudaStream_t aux_stream = nullptr;
    cudaStream_t d2h_stream = nullptr;
    cudaEvent_t ev_stage[2] = {nullptr, nullptr};
    cudaEvent_t ev_d2h[2] = {nullptr, nullptr};
    cudaEvent_t ev_start = nullptr;
    // device-side gmg_solve loops (cycle.cu solve_graph): instantiated graphs by key
    struct GraphEntry {
        std::string key;
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        int64_t kernels = 0;  // launches recorded into one replay (launch_count advances by this per replay)
    };
    std::vector<GraphEntry> graphs;
    int64_t last_graph_kernels = 0;  // kernels per iteration of the solve graph launched last
    int graph = 1;              // env DECMG_GRAPH=0: host-driven cycle loop
    // preferred shared-memory carve-out (%) of the row kernels and the projection kernels (env
    // DECMG_CARVEOUT, -1 = driver default): one common split lets a batch stream's projection blocks share
    // SMs with the persistent V-cycle kernels instead of holding them until they drain (DESIGN.md §5 x6)
    int carveout = 30;
    int vtail = 1;              // bottom of the V in one cooperative kernel (env DECMG_VTAIL=0: per-pass kernels)
    int64_t vtail_items = 32768;   // ... from the first level with at most this many thread items, rows x threads per row (env DECMG_VTAIL_ITEMS)
    int vtail_cta_items = 2048;    // ... levels with at most this many thread items on CTA 0 alone (env DECMG_VTAIL_CTA)
    int vtail_ctas_per_sm = 1;     // ... resident CTAs per SM, at most (env DECMG_VTAIL_CTAS)
    unsigned long long* vtail_trace = nullptr;  // per-pass %globaltimer stamps (env DECMG_VTAIL_TRACE=1)
    cudaStream_t cap_stream = nullptr;
    double* gstate_raw = nullptr;  // SolveState (rowkernels.cuh) of the device loop
    int* hcnt = nullptr;           // history slot counter of run_cycle's replayed bodies (cycle.cu run_graph)
    std::vector<cudaEvent_t> io_events;
    int64_t launch_count = 0;
    int rpt = 4;                // right-hand sides per thread in the vector mapping (env DECMG_RPT)
    double wtot0 = 0.0;         // sum of level-0 dual areas in the reference order
    int num_sms = 148;
    int pf = 56;                // row-kernel prefetch distance in rows, 0 = off (env DECMG_PF)
    int tile_group = -1;        // row-kernel tiles per round-robin group (-1: auto, 0: contiguous range per CTA; env DECMG_TGROUP)
    int pair = 1;               // two Jacobi sweeps per pass where a level has enough rounds (env DECMG_PAIR=0: one sweep per launch)
    int pair_group = 0;         // tiles per group of the two-sweep pass (0: auto, a ~45 MB round; env DECMG_PAIR_GROUP)
    int pair_ahead = 0;         // rounds ahead sweep 2 may gather from (env DECMG_PAIR_AHEAD)
    int pair_ctas = 3;          // resident CTAs per SM of the two-sweep pass (env DECMG_PAIR_CTAS)
    int pair_ctas_overlap = 0;  // ... inside a batch stream (0: separate sweeps there; env DECMG_PAIR_CTAS_OVERLAP)
    bool batch_overlap = false; // inside solve_batches with concurrent staging: no cooperative two-sweep passes
    int pair_min_rounds = 8;    // levels with fewer rounds keep separate sweeps (env DECMG_PAIR_MIN_ROUNDS)
    int pfl = 2;                // prefetch into L1 (1) or L2 (2) (env DECMG_PFL)
    int kmode = 2;              // row kernels: 2 auto (default), 0 pipelined, 1 high-occupancy (env DECMG_KERNEL)
    decmg_gpu::Timing timing;
    std::string err;
    std::vector<void*> allocations;
};

namespace decmg_gpu {

// Device allocation owned by the context (freed in destroy).
template <class T>
Status dalloc(decmg_gpu_ctx* c, T** p, size_t n) {
    void* q = nullptr;
    DG_CUDA(cudaMalloc(&q, (n ? n : 1) * sizeof(T)));
    c->allocations.push_back(q);
    *p = static_cast<T*>(q);
    return Status::Ok();
}

// Kernel launch bookkeeping: counts every launch and, with timing enabled,
// brackets it with CUDA events on the context stream.
void timing_begin(decmg_gpu_ctx* c, int cls, double bytes, cudaEvent_t* a, cudaEvent_t* b);
void timing_end(decmg_gpu_ctx* c, cudaEvent_t b);

template <class F>
Status launch(decmg_gpu_ctx* c, int cls, double bytes, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (c->timing.enabled) timing_begin(c, cls, bytes, &a, &b);
    f();
    ++c->launch_count;
    if (c->timing.enabled) timing_end(c, b);
    return cuda_status(cudaGetLastError(), "kernel launch");
}

// One-time setup per (device, kernel): cudaFuncSetAttribute applies to the
// device current at the call, so a process with contexts on several devices
// must repeat it for each. first_on_device(c, fn) is true on the first call
// for (c->device, fn); block_occupancy caches the resident blocks per SM of
// (device, fn) at the given block shape.
inline bool first_on_device(const decmg_gpu_ctx* c, const void* fn) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> seen;
    std::lock_guard<std::mutex> g(mu);
    return seen.emplace(c->device, fn).second;
}
inline int block_occupancy(const decmg_gpu_ctx* c, const void* fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
    std::lock_guard<std::mutex> g(mu);
    const auto key = std::make_tuple(c->device, fn, threads, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess) nb = 0;
    cache[key] = nb;
    return nb;
}

inline unsigned grid_for(int64_t threads, int block) {
    return static_cast<unsigned>((threads + block - 1) / block);
}

// setup.cu
Status build_from_base(decmg_gpu_ctx* c, const double* pos, int nv, const int* corners, int nt,
                       int nsub, unsigned flags, int use_levels = 0);
Status build_from_levels(decmg_gpu_ctx* c, const decmg_gpu_level_desc* levels, int nlevels,
                         unsigned flags);
Status alloc_work(decmg_gpu_ctx* c);
Status exclusive_scan(decmg_gpu_ctx* c, const int* in, int* out, int n);  // out[n] = total
Status level_bbox(decmg_gpu_ctx* c, const Level& m, double lo[3], double sc[3]);
Status morton_keys(decmg_gpu_ctx* c, const Level& m, const double lo[3], const double sc[3],
                   unsigned long long* d_keys, int* d_id);

// cycle.cu
struct Plan {
    std::string walk;
    std::vector<int> pre, post;
    int smoother = DECMG_SMOOTHER_JACOBI;
    double omega = 2.0 / 3.0;
};
Status make_plan(const decmg_gpu_ctx* c, const decmg_gpu_plan* p, Plan* out);
Status run_cycles(decmg_gpu_ctx* c, const Plan& plan, int nrhs, const double* d_b,
                  const double* d_x0, int ncycles, double* d_x, double* d_hist);
Status solve(decmg_gpu_ctx* c, const Plan& plan, int nrhs, const double* d_b, const double* d_x0,
             double tol, int max_cycles, double* d_x, double* h_hist, int* cycles_done,
             double* h_final, bool staged = false, const double* bsrc = nullptr);
Status stage_rhs(decmg_gpu_ctx* c, int nrhs, const double* h_b, bool project, double* dst = nullptr);
Status solve_batches(decmg_gpu_ctx* c, const Plan& plan, int nrhs, int nbatch, const double* const* h_b, double tol,
                     int max_cycles, double* const* h_x, double* h_hist, int* cycles_done, double* h_final);
// pcg.cu: gmg_preconditioned_cg (proj/src/solvers.cpp:118-130)
Status pcg(decmg_gpu_ctx* c, const Plan& inner, int inner_cycles, int nrhs, const double* d_b, double tol,
           int maxiter, double* d_x, double* h_hist, int* iters, int* converged, double* h_final, bool staged = false);
Status project_compatible(decmg_gpu_ctx* c, int nrhs, double* d_b);
Status apply_op(decmg_gpu_ctx* c, int level, char op, const double* d_x, double* d_y);
// smooth (multigrid.cpp:95-120) on level k's operator; vectors in the reference numbering
Status smooth_level(decmg_gpu_ctx* c, int k, const Plan& plan, int iters, int nrhs, const double* d_x,
                    const double* d_b, double* d_out, bool weighted);
Status build_gs_schedule(decmg_gpu_ctx* c, Level& m);

}  // namespace decmg_gpu
