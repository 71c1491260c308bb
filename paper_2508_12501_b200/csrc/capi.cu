// extern "C" boundary of libdecmg_gpu.so (declared in include/decmg_gpu.h).
#include "common.cuh"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

using namespace decmg_gpu;

namespace {

thread_local std::string g_create_error;

int fail(decmg_gpu_ctx* c, const Status& s) {
    if (c) c->err = s.msg;
    else g_create_error = s.msg;
    return s.code;
}

#define API_TRY(ctx, expr)                    \
    do {                                      \
        ::decmg_gpu::Status _s = (expr);      \
        if (!_s.ok()) return fail(ctx, _s);   \
    } while (0)

Status init_ctx(decmg_gpu_ctx* c, const decmg_gpu_config* cfg) {
    c->device = cfg ? cfg->device : 0;
    c->max_nrhs = cfg ? cfg->max_nrhs : 1;
    if (c->max_nrhs < 1 || c->max_nrhs > 32)
        return Status::Err(DECMG_INVALID_ARGUMENT, "max_nrhs must be in [1, 32]");
    int ndev = 0;
    DG_CUDA(cudaGetDeviceCount(&ndev));
    if (c->device < 0 || c->device >= ndev) return Status::Err(DECMG_INVALID_ARGUMENT, "no such CUDA device");
    DG_CUDA(cudaSetDevice(c->device));
    // the context stream runs the V-cycle at the highest priority: staging work
    // of a batch stream (solve_batches, lowest priority) fills in around it
    int prio_lo = 0, prio_hi = 0;
    DG_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    DG_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi));
    DG_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    if (const char* e = std::getenv("DECMG_PF")) c->pf = std::atoi(e);
    if (const char* e = std::getenv("DECMG_PROJ_SEQ")) c->proj_seq = std::atoi(e) != 0;
    if (const char* e = std::getenv("DECMG_GRAPH")) c->graph = std::atoi(e) != 0;
    if (const char* e = std::getenv("DECMG_CARVEOUT")) c->carveout = std::atoi(e);
    if (const char* e = std::getenv("DECMG_VTAIL")) c->vtail = std::atoi(e) != 0;
    if (const char* e = std::getenv("DECMG_VTAIL_ITEMS")) c->vtail_items = std::atoll(e);
    if (const char* e = std::getenv("DECMG_VTAIL_CTA")) c->vtail_cta_items = std::atoi(e);
    if (const char* e = std::getenv("DECMG_VTAIL_CTAS")) c->vtail_ctas_per_sm = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("DECMG_VTAIL_TRACE"))
        if (std::atoi(e)) DG_TRY(dalloc(c, &c->vtail_trace, 256));
    if (const char* e = std::getenv("DECMG_PFL")) c->pfl = std::atoi(e);
    if (const char* e = std::getenv("DECMG_PAIR")) c->pair = std::atoi(e);
    if (const char* e = std::getenv("DECMG_PAIR_GROUP")) c->pair_group = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("DECMG_PAIR_CTAS")) c->pair_ctas = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("DECMG_PAIR_CTAS_OVERLAP")) c->pair_ctas_overlap = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("DECMG_PAIR_AHEAD")) c->pair_ahead = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("DECMG_PAIR_MIN_ROUNDS")) c->pair_min_rounds = std::max(2, std::atoi(e));
    if (const char* e = std::getenv("DECMG_TGROUP")) c->tile_group = std::max(-1, std::atoi(e));
    if (const char* e = std::getenv("DECMG_KERNEL")) {
        const std::string m(e);
        c->kmode = m == "pipe" ? 0 : (m == "ell" ? 1 : 2);
    }
    if (const char* e = std::getenv("DECMG_RPT")) {
        const int v = std::atoi(e);
        if (v == 1 || v == 2 || v == 4) c->rpt = v;
    }
    return Status::Ok();
}

void destroy_ctx(decmg_gpu_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto& r : c->timing.recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : c->timing.pool) cudaEventDestroy(e);
    for (void* p : c->allocations) cudaFree(p);
    if (c->hsmall) cudaFreeHost(c->hsmall);
    if (c->hist_dev) cudaFree(c->hist_dev);
    for (cudaEvent_t e : c->io_events) cudaEventDestroy(e);
    for (cudaStream_t s : {c->io_stream, c->aux_stream, c->d2h_stream})
        if (s) cudaStreamSynchronize(s);
    for (cudaEvent_t e : {c->ev_stage[0], c->ev_stage[1], c->ev_d2h[0], c->ev_d2h[1], c->ev_start})
        if (e) cudaEventDestroy(e);
    for (auto& e : c->graphs) {
        cudaGraphExecDestroy(e.exec);
        cudaGraphDestroy(e.graph);
    }
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    if (c->io_stream) cudaStreamDestroy(c->io_stream);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// RAII device buffer for host-pointer entry points
struct DevBuf {
    double* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    Status alloc(size_t n) {
        DG_CUDA(cudaMalloc(&p, (n ? n : 1) * sizeof(double)));
        return Status::Ok();
    }
};

uint64_t fnv1a(const void* data, size_t n, uint64_t h) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}

}  // namespace

namespace decmg_gpu {

cudaEvent_t pool_event(decmg_gpu_ctx* c) {
    if (!c->timing.pool.empty()) {
        cudaEvent_t e = c->timing.pool.back();
        c->timing.pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void timing_begin(decmg_gpu_ctx* c, int cls, double bytes, cudaEvent_t* a, cudaEvent_t* b) {
    *a = pool_event(c);
    *b = pool_event(c);
    cudaEventRecord(*a, c->stream);
    c->timing.recs.push_back({cls, bytes, *a, *b});
}

void timing_end(decmg_gpu_ctx* c, cudaEvent_t b) { cudaEventRecord(b, c->stream); }

}  // namespace decmg_gpu

extern "C" {

const char* decmg_gpu_last_error(const decmg_gpu_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int decmg_gpu_create_from_base(const double* positions, int nv, const int* corner_triples, int nt,
                               int nsub, unsigned flags, const decmg_gpu_config* cfg,
                               decmg_gpu_ctx** out) {
    return decmg_gpu_create_from_base_ex(positions, nv, corner_triples, nt, nsub, 0, flags, cfg, out);
}

int decmg_gpu_create_from_base_ex(const double* positions, int nv, const int* corner_triples, int nt, int nsub,
                                  int use_levels, unsigned flags, const decmg_gpu_config* cfg, decmg_gpu_ctx** out) {
    if (!out || !positions || !corner_triples)
        return fail(nullptr, Status::Err(DECMG_INVALID_ARGUMENT, "create_from_base: null argument"));
    *out = nullptr;
    auto* c = new decmg_gpu_ctx();
    c->flags = flags;
    Status s = init_ctx(c, cfg);
    if (s.ok()) s = build_from_base(c, positions, nv, corner_triples, nt, nsub, flags, use_levels);
    if (!s.ok()) {
        destroy_ctx(c);
        return fail(nullptr, s);
    }
    *out = c;
    return DECMG_OK;
}

int decmg_gpu_create_from_levels(const decmg_gpu_level_desc* levels, int nlevels, unsigned flags,
                                 const decmg_gpu_config* cfg, decmg_gpu_ctx** out) {
    if (!out) return fail(nullptr, Status::Err(DECMG_INVALID_ARGUMENT, "create_from_levels: null argument"));
    *out = nullptr;
    auto* c = new decmg_gpu_ctx();
    c->flags = flags;
    Status s = init_ctx(c, cfg);
    if (s.ok()) s = build_from_levels(c, levels, nlevels, flags);
    if (!s.ok()) {
        destroy_ctx(c);
        return fail(nullptr, s);
    }
    *out = c;
    return DECMG_OK;
}

void decmg_gpu_destroy(decmg_gpu_ctx* ctx) { destroy_ctx(ctx); }

int decmg_gpu_levels(const decmg_gpu_ctx* ctx) { return ctx ? static_cast<int>(ctx->lv.size()) : 0; }

void* decmg_gpu_stream(decmg_gpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int decmg_gpu_run_cycles(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs, const double* b,
                         const double* x0, int ncycles, double* x_out, double* hist_out) {
    if (!ctx) return DECMG_INVALID_ARGUMENT;
    if (!b) return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "run_cycle: rhs is null"));
    cudaSetDevice(ctx->device);
    Plan p;
    API_TRY(ctx, make_plan(ctx, plan, &p));
    if (nrhs < 1 || nrhs > ctx->max_nrhs)
        return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs]"));
    const size_t n = static_cast<size_t>(ctx->lv[0].nv) * nrhs;
    if (ncycles > ctx->hist_cap) {
        if (ctx->hist_dev) cudaFree(ctx->hist_dev);
        ctx->hist_dev = nullptr;
        ctx->hist_cap = 0;
        API_TRY(ctx, cuda_status(cudaMalloc(&ctx->hist_dev, sizeof(double) * ncycles * 32), "hist"));
        ctx->hist_cap = ncycles;
    }
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(ctx->io_b, b, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D b"));
    if (x0)
        API_TRY(ctx, cuda_status(cudaMemcpyAsync(ctx->io_x0, x0, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D x0"));
    API_TRY(ctx, run_cycles(ctx, p, nrhs, ctx->io_b, x0 ? ctx->io_x0 : nullptr, ncycles, ctx->io_x, ctx->hist_dev));
    if (x_out)
        API_TRY(ctx, cuda_status(cudaMemcpyAsync(x_out, ctx->io_x, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H x"));
    if (hist_out && ncycles > 0)
        API_TRY(ctx, cuda_status(cudaMemcpyAsync(hist_out, ctx->hist_dev, sizeof(double) * ncycles * nrhs,
                                                 cudaMemcpyDeviceToHost, ctx->stream), "D2H hist"));
    API_TRY(ctx, cuda_status(cudaStreamSynchronize(ctx->stream), "run_cycles"));
    return DECMG_OK;
}

int decmg_gpu_run_cycles_dev(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs, const double* d_b,
                             const double* d_x0, int ncycles, double* d_x, double* d_hist) {
    if (!ctx) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    Plan p;
    API_TRY(ctx, make_plan(ctx, plan, &p));
    API_TRY(ctx, run_cycles(ctx, p, nrhs, d_b, d_x0, ncycles, d_x, d_hist));
    return DECMG_OK;
}

int decmg_gpu_solve(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs, const double* b,
                    const double* x0, double tol, int max_cycles, double* x_out, double* hist_out,
                    int* cycles_done, double* final_out) {
    if (!ctx) return DECMG_INVALID_ARGUMENT;
    if (!b) return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "gmg_solve: rhs is null"));
    cudaSetDevice(ctx->device);
    Plan p;
    API_TRY(ctx, make_plan(ctx, plan, &p));
    if (nrhs < 1 || nrhs > ctx->max_nrhs)
        return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs]"));
    const size_t n = static_cast<size_t>(ctx->lv[0].nv) * nrhs;
    // H2D of b overlapped with the projection chain (stage_rhs), into ctx->bproj
    API_TRY(ctx, stage_rhs(ctx, nrhs, b, !ctx->dirichlet));
    if (x0)
        API_TRY(ctx, cuda_status(cudaMemcpyAsync(ctx->io_x0, x0, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D x0"));
    API_TRY(ctx, solve(ctx, p, nrhs, nullptr, x0 ? ctx->io_x0 : nullptr, tol, max_cycles, ctx->io_x, hist_out,
                       cycles_done, final_out, true));
    if (x_out)
        API_TRY(ctx, cuda_status(cudaMemcpyAsync(x_out, ctx->io_x, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H x"));
    API_TRY(ctx, cuda_status(cudaStreamSynchronize(ctx->stream), "gmg_solve"));
    return DECMG_OK;
}

int decmg_gpu_solve_batches(decmg_gpu_ctx* ctx, const decmg_gpu_plan* plan, int nrhs, int nbatch,
                            const double* const* b, double tol, int max_cycles, double* const* x_out,
                            double* hist_out, int* cycles_done, double* final_out) {
    if (!ctx) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    Plan p;
    API_TRY(ctx, make_plan(ctx, plan, &p));
    if (nrhs < 1 || nrhs > ctx->max_nrhs)
        return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs]"));
    API_TRY(ctx, solve_batches(ctx, p, nrhs, nbatch, b, tol, max_cycles, x_out, hist_out, cycles_done, final_out));
    return DECMG_OK;
}

int decmg_gpu_pcg(decmg_gpu_ctx* ctx, const decmg_gpu_plan* inner, int inner_cycles, int nrhs, const double* b,
                  double tol, int maxiter, double* x_out, double* hist_out, int* iters_out, int* converged_out,
                  double* final_out) {
    if (!ctx) return DECMG_INVALID_ARGUMENT;
    if (!b || !iters_out || !converged_out)
        return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "gmg_pcg: null argument"));
    cudaSetDevice(ctx->device);
    Plan p;
    API_TRY(ctx, make_plan(ctx, inner, &p));
    if (nrhs < 1 || nrhs > ctx->max_nrhs)
        return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs]"));
    const size_t n = static_cast<size_t>(ctx->lv[0].nv) * nrhs;
    if (ctx->dirichlet)
        return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT,
                                     "gmg_pcg: Neumann hierarchies only (the reference projects b)"));
    (void)n;
    // H2D of b overlapped with the projection chain (stage_rhs), into ctx->bproj
    API_TRY(ctx, stage_rhs(ctx, nrhs, b, true));
    API_TRY(ctx, pcg(ctx, p, inner_cycles, nrhs, nullptr, tol, maxiter, ctx->io_x, hist_out, iters_out,
                     converged_out, final_out, true));
    if (x_out)
        API_TRY(ctx, cuda_status(cudaMemcpyAsync(x_out, ctx->io_x, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H x"));
    API_TRY(ctx, cuda_status(cudaStreamSynchronize(ctx->stream), "gmg_pcg"));
    return DECMG_OK;
}

int decmg_gpu_project_compatible(decmg_gpu_ctx* ctx, int nrhs, double* b) {
    if (!ctx || !b) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    const size_t n = static_cast<size_t>(ctx->lv[0].nv) * nrhs;
    DevBuf db;
    API_TRY(ctx, db.alloc(n));
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(db.p, b, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D"));
    API_TRY(ctx, project_compatible(ctx, nrhs, db.p));
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(b, db.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H"));
    API_TRY(ctx, cuda_status(cudaStreamSynchronize(ctx->stream), "project"));
    return DECMG_OK;
}

int decmg_gpu_smooth(decmg_gpu_ctx* ctx, int level, int smoother, double omega, int iters, int nrhs, double* x,
                     const double* b, int weighted) {
    if (!ctx || !x || !b) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    const int L = static_cast<int>(ctx->lv.size());
    if (level < 0 || level >= L) return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "smooth: level out of range"));
    decmg_gpu_plan ps{};
    ps.smoother = smoother;
    ps.jacobi_omega = omega;
    ps.pre_all = ps.post_all = 0;
    Plan p;
    API_TRY(ctx, make_plan(ctx, &ps, &p));
    if (nrhs < 1 || nrhs > ctx->max_nrhs)
        return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs] (max 32)"));
    const size_t n = static_cast<size_t>(ctx->lv[level].nv) * nrhs;
    DevBuf dx, db;
    API_TRY(ctx, dx.alloc(n));
    API_TRY(ctx, db.alloc(n));
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(dx.p, x, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D"));
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(db.p, b, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D"));
    API_TRY(ctx, smooth_level(ctx, level, p, iters, nrhs, dx.p, db.p, dx.p, weighted != 0));
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(x, dx.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H"));
    API_TRY(ctx, cuda_status(cudaStreamSynchronize(ctx->stream), "smooth"));
    return DECMG_OK;
}

int decmg_gpu_last_times(const decmg_gpu_ctx* ctx, double* out, int max) {
    if (!ctx) return -1;
    const int n = static_cast<int>(ctx->last_times.size());
    if (out)
        for (int i = 0; i < n && i < max; ++i) out[i] = ctx->last_times[i];
    return n;
}

int decmg_gpu_apply(decmg_gpu_ctx* ctx, int level, char op, const double* x, double* y) {
    if (!ctx || !x || !y) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    const int L = static_cast<int>(ctx->lv.size());
    if (level < 0 || level >= L) return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "apply: level out of range"));
    const int nf = ctx->lv[level].nv;
    const int nc = level + 1 < L ? ctx->lv[level + 1].nv : 0;
    const size_t nin = op == 'P' ? nc : (op == 'R' ? nf : nf);
    const size_t nout = op == 'R' ? nc : nf;
    DevBuf dx, dy;
    API_TRY(ctx, dx.alloc(nin));
    API_TRY(ctx, dy.alloc(nout));
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(dx.p, x, nin * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D"));
    API_TRY(ctx, apply_op(ctx, level, op, dx.p, dy.p));
    API_TRY(ctx, cuda_status(cudaMemcpyAsync(y, dy.p, nout * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H"));
    API_TRY(ctx, cuda_status(cudaStreamSynchronize(ctx->stream), "apply"));
    return DECMG_OK;
}

int decmg_gpu_level_info(decmg_gpu_ctx* ctx, int level, int64_t counts[6]) {
    if (!ctx || level < 0 || level >= static_cast<int>(ctx->lv.size())) return DECMG_INVALID_ARGUMENT;
    const Level& m = ctx->lv[level];
    counts[0] = m.nv;
    counts[1] = m.ne;
    counts[2] = m.nt;
    counts[3] = m.nnzL;
    counts[4] = m.nnzP;
    counts[5] = m.nnzR;
    return DECMG_OK;
}

int64_t decmg_gpu_export(decmg_gpu_ctx* ctx, int level, const char* name, void* out) {
    if (!ctx || !name || level < 0 || level >= static_cast<int>(ctx->lv.size())) return -1;
    cudaSetDevice(ctx->device);
    const Level& m = ctx->lv[level];
    const int nvc = level + 1 < static_cast<int>(ctx->lv.size()) ? ctx->lv[level + 1].nv : 0;
    const void* src = nullptr;
    int64_t count = -1;
    size_t elem = 0;
    const std::string s(name);
    auto pick = [&](const void* p, int64_t n, size_t e) {
        src = p;
        count = p ? n : -1;
        elem = e;
    };
    if (s == "positions") pick(m.pos, 3 * static_cast<int64_t>(m.nv), 8);
    else if (s == "edges") pick(m.edges, 2 * static_cast<int64_t>(m.ne), 4);
    else if (s == "triangles") pick(m.tris, 3 * static_cast<int64_t>(m.nt), 4);
    else if (s == "corners") pick(m.corners, 3 * static_cast<int64_t>(m.nt), 4);
    else if (s == "dual_areas") pick(m.area, m.nv, 8);
    else if (s == "boundary") pick(m.bd, m.nv, 4);
    else if (s == "diag") pick(m.diag, m.nv, 8);
    else if (s == "order") pick(m.ord, m.nv, 4);
    else if (s == "vtail_trace") pick(ctx->vtail_trace, 256, 8);
    else if (s == "L_row_ptr") pick(m.L_rp, m.nv + 1, 4);
    else if (s == "L_col_idx") pick(m.L_ci, m.nnzL, 4);
    else if (s == "L_values") pick(m.L_v, m.nnzL, 8);
    else if (s == "P_row_ptr") pick(m.P_rp, m.nv + 1, 4);
    else if (s == "P_col_idx") pick(m.P_ci, m.nnzP, 4);
    else if (s == "P_values") pick(m.P_v, m.nnzP, 8);
    else if (s == "R_row_ptr") pick(m.R_rp, nvc + 1, 4);
    else if (s == "R_col_idx") pick(m.R_ci, m.nnzR, 4);
    else if (s == "R_values") pick(m.R_v, m.nnzR, 8);
    if (count < 0) return -1;
    if (out && count > 0) {
        if (cudaMemcpyAsync(out, src, count * elem, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess) return -1;
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -1;
    }
    return count;
}

// EmbeddedComplex2D::hash (proj/src/mesh.cpp:112-119): FNV-1a over the counts,
// positions, edges and edge triples, computed on the host from the device arrays.
int decmg_gpu_mesh_hash(decmg_gpu_ctx* ctx, int level, uint64_t* hash) {
    if (!ctx || !hash || level < 0 || level >= static_cast<int>(ctx->lv.size())) return DECMG_INVALID_ARGUMENT;
    const Level& m = ctx->lv[level];
    if (!m.pos) return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "mesh_hash: hierarchy has no mesh data"));
    std::vector<double> pos(3 * static_cast<size_t>(m.nv));
    std::vector<int> edges(2 * static_cast<size_t>(m.ne)), tris(3 * static_cast<size_t>(m.nt));
    if (decmg_gpu_export(ctx, level, "positions", pos.data()) < 0 ||
        decmg_gpu_export(ctx, level, "edges", edges.data()) < 0 ||
        decmg_gpu_export(ctx, level, "triangles", tris.data()) < 0)
        return fail(ctx, Status::Err(DECMG_CUDA, "mesh_hash: export failed"));
    uint64_t h = 1469598103934665603ULL;
    const int counts[3] = {m.nv, m.ne, m.nt};
    h = fnv1a(counts, sizeof counts, h);
    if (!pos.empty()) h = fnv1a(pos.data(), pos.size() * sizeof(double), h);
    if (!edges.empty()) h = fnv1a(edges.data(), edges.size() * sizeof(int), h);
    if (!tris.empty()) h = fnv1a(tris.data(), tris.size() * sizeof(int), h);
    *hash = h;
    return DECMG_OK;
}

int decmg_gpu_set_timing(decmg_gpu_ctx* ctx, int enable) {
    if (!ctx) return DECMG_INVALID_ARGUMENT;
    ctx->timing.enabled = enable != 0;
    return DECMG_OK;
}

int decmg_gpu_get_timing(decmg_gpu_ctx* ctx, int cls, int64_t* launches, double* total_ms, double* bytes) {
    if (!ctx || cls < -1 || cls >= 8) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    auto& T = ctx->timing;
    if (!T.recs.empty()) {
        cudaStreamSynchronize(ctx->stream);
        for (auto& r : T.recs) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            T.launches[r.cls] += 1;
            T.ms[r.cls] += ms;
            T.bytes[r.cls] += r.bytes;
            T.pool.push_back(r.a);
            T.pool.push_back(r.b);
        }
        T.recs.clear();
    }
    if (cls == -1) {  // reset all accumulators
        for (int i = 0; i < 8; ++i) {
            T.launches[i] = 0;
            T.ms[i] = 0;
            T.bytes[i] = 0;
        }
        return DECMG_OK;
    }
    if (launches) *launches = T.launches[cls];
    if (total_ms) *total_ms = T.ms[cls];
    if (bytes) *bytes = T.bytes[cls];
    return DECMG_OK;
}

int64_t decmg_gpu_launch_count(decmg_gpu_ctx* ctx) { return ctx ? ctx->launch_count : -1; }

int64_t decmg_gpu_projection_fallbacks(decmg_gpu_ctx* ctx) {
    if (!ctx) return -1;
    if (!ctx->seq_fallbacks) return 0;
    cudaSetDevice(ctx->device);
    int v = 0;
    if (cudaMemcpyAsync(&v, ctx->seq_fallbacks, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return -1;
    return v;
}

// ---------------------------------------------------------------- inputs ----
// make_triangulated_grid (proj/src/mesh.cpp:232-257), make_equilateral_grid
// (259-291) and the canonical icosahedron of extension x2.
int decmg_base_mesh(const char* spec, double* pos, int* nv_out, int* tri, int* nt_out) {
    if (!spec || !nv_out || !nt_out) return DECMG_INVALID_ARGUMENT;
    std::vector<double> P;
    std::vector<int> T;
    const std::string s(spec);
    auto grid = [&](int nx, int ny, double lx, double ly) {
        const double dx = lx / nx, dy = ly / ny;
        for (int j = 0; j <= ny; ++j)
            for (int i = 0; i <= nx; ++i) {
                P.push_back(i * dx);
                P.push_back(j * dy);
                P.push_back(0.0);
            }
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const int bl = j * (nx + 1) + i, br = bl + 1, tr = (j + 1) * (nx + 1) + i + 1, tl = tr - 1;
                T.insert(T.end(), {bl, br, tr, bl, tr, tl});
            }
    };
    if (s == "square") {
        grid(1, 1, 1.0, 1.0);
    } else if (s.rfind("grid:", 0) == 0) {
        int nx, ny;
        double lx, ly;
        if (std::sscanf(spec, "grid:%d:%d:%lf:%lf", &nx, &ny, &lx, &ly) != 4 || nx < 1 || ny < 1 || lx <= 0 || ly <= 0)
            return DECMG_INVALID_ARGUMENT;
        grid(nx, ny, lx, ly);
    } else if (s.rfind("equi:", 0) == 0) {
        int rows, cols;
        double side;
        if (std::sscanf(spec, "equi:%d:%d:%lf", &rows, &cols, &side) != 3 || rows < 1 || cols < 1 || side <= 0 ||
            (cols % 2 != 0 && rows > 1))
            return DECMG_INVALID_ARGUMENT;
        const int nup = (cols + 1) / 2, ndown = cols / 2, rv = nup + 1;
        const double hy = side * std::sqrt(3.0) / 2.0;
        for (int j = 0; j <= rows; ++j) {
            const int count = (j == rows && ndown < nup) ? ndown + 1 : rv;
            for (int i = 0; i < count; ++i) {
                P.push_back(i * side + j * side / 2.0);
                P.push_back(j * hy);
                P.push_back(0.0);
            }
        }
        for (int j = 0; j < rows; ++j) {
            for (int i = 0; i < nup; ++i) T.insert(T.end(), {j * rv + i, j * rv + i + 1, (j + 1) * rv + i});
            for (int i = 0; i < ndown; ++i) T.insert(T.end(), {j * rv + i + 1, (j + 1) * rv + i + 1, (j + 1) * rv + i});
        }
    } else if (s == "ico") {
        const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
        const double raw[12][3] = {{-1, phi, 0}, {1, phi, 0},  {-1, -phi, 0}, {1, -phi, 0},
                                   {0, -1, phi}, {0, 1, phi},  {0, -1, -phi}, {0, 1, -phi},
                                   {phi, 0, -1}, {phi, 0, 1},  {-phi, 0, -1}, {-phi, 0, 1}};
        for (const auto& r : raw) {
            const double nrm = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
            const double sc = 1.0 / nrm;
            P.push_back(r[0] * sc);
            P.push_back(r[1] * sc);
            P.push_back(r[2] * sc);
        }
        const int F[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                              {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                              {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                              {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
        for (const auto& f : F) T.insert(T.end(), {f[0], f[1], f[2]});
    } else {
        return DECMG_INVALID_ARGUMENT;
    }
    *nv_out = static_cast<int>(P.size() / 3);
    *nt_out = static_cast<int>(T.size() / 3);
    if (pos) std::memcpy(pos, P.data(), P.size() * sizeof(double));
    if (tri) std::memcpy(tri, T.data(), T.size() * sizeof(int));
    return DECMG_OK;
}

// Synthetic right-hand sides (extension x3). uniform01 = (mt19937_64() >> 11)
// * 2^-53 (proj/include/decmg/rng.hpp:11-13); RHS j is seeded with seed + j.
int decmg_gpu_make_rhs(decmg_gpu_ctx* ctx, const char* kind, uint64_t seed, int nrhs, double* b) {
    if (!ctx || !kind || !b || nrhs < 1) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    const Level& m = ctx->lv[0];
    const int n = m.nv;
    const std::string k(kind);
    std::vector<double> pos, col(n);
    std::vector<int> bd(n, 0);
    if (k == "ylm" || k == "sinsin") {
        if (!m.pos) return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "make_rhs: hierarchy has no positions"));
        pos.resize(3 * static_cast<size_t>(n));
        if (decmg_gpu_export(ctx, 0, "positions", pos.data()) < 0) return fail(ctx, Status::Err(DECMG_CUDA, "export"));
    }
    if (ctx->dirichlet && decmg_gpu_export(ctx, 0, "boundary", bd.data()) < 0)
        return fail(ctx, Status::Err(DECMG_CUDA, "export"));
    for (int j = 0; j < nrhs; ++j) {
        std::mt19937_64 rng(seed + j);
        auto u01 = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
        if (k == "uniform") {
            for (int i = 0; i < n; ++i) col[i] = 2.0 * u01() - 1.0;
        } else if (k == "lr") {
            std::vector<double> u(n);
            for (int i = 0; i < n; ++i) u[i] = u01();
            const int rc = decmg_gpu_apply(ctx, 0, 'L', u.data(), col.data());
            if (rc) return rc;
        } else if (k == "ylm") {
            std::vector<double> g(static_cast<size_t>(n) + 1);
            for (int i = 0; i < n; i += 2) {
                const double u1 = u01();
                const double u2 = u01();
                const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
                const double th = 2.0 * M_PI * u2;
                g[i] = rad * std::cos(th);
                g[i + 1] = rad * std::sin(th);
            }
            const double c = 0.25 * std::sqrt(105.0 / M_PI);
            for (int i = 0; i < n; ++i) {
                const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
                col[i] = c * ((x * x - y * y) * z) + 1e-3 * g[i];
            }
        } else if (k == "sinsin") {
            for (int i = 0; i < n; ++i) {
                const double x = pos[3 * i], y = pos[3 * i + 1];
                const double f = ((2.0 * M_PI * M_PI) * std::sin(M_PI * x)) * std::sin(M_PI * y);
                col[i] = -f;
            }
        } else {
            return fail(ctx, Status::Err(DECMG_INVALID_ARGUMENT, "make_rhs: unknown kind " + k));
        }
        for (int i = 0; i < n; ++i) b[static_cast<int64_t>(i) * nrhs + j] = (ctx->dirichlet && bd[i]) ? 0.0 : col[i];
    }
    return DECMG_OK;
}

}  // extern "C"
