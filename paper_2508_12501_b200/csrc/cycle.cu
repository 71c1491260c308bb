// The V-cycle hot path: smoother, residual, restriction, prolongation +
// correction, coarse solve, norms, and the cycle driver.
//
// Reference path (all in /root/reference/proj):
//   jacobi_sweep            src/multigrid.cpp:36-56
//   SparseOperator::apply   src/sparse.cpp:209-218
//   cycle_once / run_cycle  src/multigrid.cpp:252-323
//   project_compatible      src/multigrid.cpp:240-250
//   gmg_solve               src/solvers.cpp:251-279
//   PinnedDirectSolver      src/direct.cpp:39-76 (stand-in: projected weighted CG)
//
// Layout: every vector is [n][nrhs] fp64, so the nrhs values of one vertex
// are adjacent and a gather of x[col] for a batch is one contiguous segment
// (128 B for nrhs = 16). Thread mapping: BP (nrhs rounded up to a power of
// two) consecutive threads own one row, lane = RHS index.
//
// Arithmetic: per-row sums start at 0.0 and add v_k * x[c_k] in CSR order,
// with explicit _rn intrinsics (no FMA), exactly as the reference's CSR loop,
// so sweeps, residuals and transfers are bit-identical to the reference.
// Norms and projections use a fixed-shape tree reduction: deterministic run
// to run, within a few ulps of the reference's blocked sums.
#include "driver.cuh"
#include "seqsum.cuh"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <functional>

namespace decmg_gpu {
namespace {

}  // namespace

Status make_plan(const decmg_gpu_ctx* c, const decmg_gpu_plan* p, Plan* out) {
    const int L = static_cast<int>(c->lv.size());
    Plan q;
    if (p && p->smoother != DECMG_SMOOTHER_JACOBI && p->smoother != DECMG_SMOOTHER_GS &&
        p->smoother != DECMG_SMOOTHER_SGS && p->smoother != DECMG_SMOOTHER_CG)
        return Status::Err(DECMG_INVALID_ARGUMENT, "smoother: unknown smoother");
    // plan == NULL: standard_plan(levels, CycleKind::V) with its defaults
    // (multigrid.hpp:88-89: pre = post = 3, SmootherConfig{} = Gauss-Seidel)
    q.smoother = p ? p->smoother : DECMG_SMOOTHER_GS;
    q.omega = p ? p->jacobi_omega : 2.0 / 3.0;
    if (p && p->walk) {
        q.walk = p->walk;
    } else {
        for (int i = 0; i < L - 1; ++i) q.walk.push_back('d');
        for (int i = 0; i < L - 1; ++i) q.walk.push_back('u');
    }
    for (int k = 0; k < L; ++k) {
        q.pre.push_back(p ? (p->pre ? p->pre[k] : p->pre_all) : 3);
        q.post.push_back(p ? (p->post ? p->post[k] : p->post_all) : 3);
    }
    // CyclePlan::validate (multigrid.cpp:131-143)
    int level = 0;
    for (char t : q.walk) {
        if (t != 'd' && t != 'u') return Status::Err(DECMG_INVALID_ARGUMENT, "CyclePlan: walk must be 'd'/'u'");
        level += t == 'd' ? 1 : -1;
        if (level < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "CyclePlan: walk rises above the finest level");
        if (level > L - 1)
            return Status::Err(DECMG_INVALID_ARGUMENT, "CyclePlan: walk descends below the coarsest level");
    }
    if (level != 0) return Status::Err(DECMG_INVALID_ARGUMENT, "CyclePlan: walk does not return to the finest level");
    *out = std::move(q);
    return Status::Ok();
}

namespace {

// hist[(*cnt) * nrhs + l] = res[l]; ++*cnt (the history slot of a replayed body)
__global__ void k_hist_put(int nrhs, const double* __restrict__ res, double* __restrict__ hist, int* cnt) {
    const int l = threadIdx.x;
    const int c = *cnt;
    if (l < nrhs) hist[static_cast<int64_t>(c) * nrhs + l] = res[l];
    __syncwarp();
    if (l == 0) *cnt = c + 1;
}

// run_cycle's cycles 1 .. ncycles-1 as replays of one captured body: the first
// level-0 sweep with the fused residual norm of the incoming iterate, its
// history store (slot from a device counter), the rest of the cycle. Valid
// when the body keeps level 0's ping-pong parity (checked after the capture,
// as in solve_graph); hist rows 0 .. ncycles-1 end up in d_hist.
Status run_graph(decmg_gpu_ctx* c, Driver& dr, const Plan& plan, int nrhs, double* denom, int ncycles,
                 double* d_hist, bool* graphed) {
    *graphed = false;
    if (!c->hcnt) DG_TRY(dalloc(c, &c->hcnt, 1));
    double* dres = c->dsmall + 256;
    uint64_t omega_bits = 0;
    std::memcpy(&omega_bits, &plan.omega, sizeof omega_bits);
    std::string key = "run|" + plan.walk + "|" + std::to_string(plan.smoother) + "|" + std::to_string(omega_bits) +
                      "|" + std::to_string(nrhs) + "|" + std::to_string(reinterpret_cast<uintptr_t>(dr.b0)) + "|" +
                      std::to_string(reinterpret_cast<uintptr_t>(d_hist)) + "|" + (dr.use_pairs ? "p|" : "s|");
    for (size_t k = 0; k < c->lv.size(); ++k)
        key += std::to_string(plan.pre[k]) + "," + std::to_string(plan.post[k]) + "," +
               std::to_string(c->lv[k].cur) + std::to_string(c->lv[k].x_zero ? 1 : 0) + ";";
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
    for (auto& e : c->graphs)
        if (e.key == key) {
            exec = e.exec;
            kernels = e.kernels;
        }
    if (!exec) {
        std::vector<std::pair<int, bool>> st0;
        for (const Level& L : c->lv) st0.emplace_back(L.cur, L.x_zero);
        const int64_t lc0 = c->launch_count;
        DG_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        dr.fuse_hist = dres;
        dr.fuse_denom = denom;
        dr.fuse_hook = [&](const double*, bool* stop) -> Status {
            *stop = false;
            return launch(c, kNorms, 0.0, [&] { k_hist_put<<<1, 32, 0, c->stream>>>(nrhs, dres, d_hist, c->hcnt); });
        };
        Status hs = dr.one_cycle(plan);
        dr.fuse_hook = nullptr;
        const bool fused = dr.fuse_hist == nullptr;
        dr.fuse_hist = nullptr;
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        kernels = c->launch_count - lc0;  // recorded, not run: counted per replay instead
        c->launch_count = lc0;
        if (hs.ok() && e != cudaSuccess) hs = cuda_status(e, "graph capture (run_cycle body)");
        if (!hs.ok()) {
            if (g) cudaGraphDestroy(g);
            return hs;
        }
        if (!fused || c->lv[0].cur != st0[0].first) {  // no fused norm, or a parity-flipping walk: eager loop
            cudaGraphDestroy(g);
            for (size_t k = 0; k < c->lv.size(); ++k) {
                c->lv[k].cur = st0[k].first;
                c->lv[k].x_zero = st0[k].second;
            }
            return Status::Ok();
        }
        DG_CUDA(cudaGraphInstantiate(&exec, g, 0));
        c->graphs.push_back({key, g, exec, kernels});
    }
    DG_CUDA(cudaMemsetAsync(c->hcnt, 0, sizeof(int), c->stream));
    for (int k = 1; k < ncycles; ++k) {
        DG_CUDA(cudaGraphLaunch(exec, c->stream));
        c->launch_count += kernels;
    }
    DG_TRY(dr.resnorm(d_hist + static_cast<int64_t>(ncycles - 1) * nrhs, denom));
    *graphed = true;
    return Status::Ok();
}

}  // namespace

Status run_cycles(decmg_gpu_ctx* c, const Plan& plan, int nrhs, const double* d_b, const double* d_x0,
                  int ncycles, double* d_x, double* d_hist) {
    DG_TRY(check_nrhs(c, nrhs));
    if (ncycles < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "CyclePlan: negative cycle count");
    Level& L = c->lv[0];
    const double* b_in = d_b;
    if (L.ord || (reinterpret_cast<uintptr_t>(d_b) & 31) != 0) b_in = L.b;  // internal copy (32-byte aligned)
    Driver dr{c, nrhs, bp_of(nrhs), b_in};
    DG_TRY(dr.init());
    if (b_in != d_b) DG_TRY(dr.to_internal(d_b, L.b));
    double* denom = c->dsmall;
    DG_TRY(dr.load_x0(d_x0));
    DG_TRY(dr.make_denom(denom));
    // hist[c] = residual of the iterate after cycle c: computed by the first
    // level-0 sweep of cycle c+1 when possible, else by a separate pass.
    int cyc = 0;
    if (ncycles >= 3 && c->graph && !c->timing.enabled && c->lv.size() > 1) {
        // cycles 1 .. ncycles-1 as replays of one captured body (run_graph)
        DG_TRY(dr.one_cycle(plan));
        cyc = 1;
        bool graphed = false;
        if (dr.can_fuse(plan)) DG_TRY(run_graph(c, dr, plan, nrhs, denom, ncycles, d_hist, &graphed));
        if (graphed) cyc = ncycles;
        else DG_TRY(dr.resnorm(d_hist, denom));  // hist[0] of the eager loop below
    }
    for (; cyc < ncycles; ++cyc) {
        DG_TRY(dr.one_cycle(plan));
        double* hc = d_hist + static_cast<int64_t>(cyc) * nrhs;
        if (cyc + 1 < ncycles && dr.can_fuse(plan)) {
            dr.fuse_hist = hc;
            dr.fuse_denom = denom;
        } else {
            DG_TRY(dr.resnorm(hc, denom));
        }
    }
    DG_TRY(dr.ensure_x(0));
    return dr.from_internal(L.x[L.cur], d_x);
}

namespace {

// The projection's mean chain over rows [r0, r1) (state in c->dsmall + 160),
// mean_out on the last range: the exact parallel chain (seqsum.cuh) in passes
// of at most kSeqPassRows rows.
Status project_chain_par(decmg_gpu_ctx* c, int nrhs, const double* d_b, int r0, int r1, double* mean_out) {
    const Level& L = c->lv[0];
    double* state = c->dsmall + 160;
    const size_t lanes = static_cast<size_t>(c->max_nrhs);
    const size_t per = static_cast<size_t>(kSeqPassRecs) * lanes;  // approx, guess: [lane][record]
    const size_t pstride = static_cast<size_t>((std::min(kSeqPassRows, L.nv) + 3) & ~1);  // even: nodes stay 16-byte aligned
    const size_t nodes_d = lanes * kSeqPassGrps * sizeof(SeqNode) * kGrpNodes / sizeof(double);
    if (!c->seq_buf) {
        DG_TRY(dalloc(c, &c->seq_buf, 2 * per + pstride * lanes + nodes_d));
        DG_TRY(dalloc(c, &c->seq_fallbacks, 1));
        DG_CUDA(cudaMemsetAsync(c->seq_fallbacks, 0, sizeof(int), c->stream));
        const int smax = kTileRows * 33 * static_cast<int>(sizeof(double));
        DG_CUDA(cudaFuncSetAttribute(k_seq_prod, cudaFuncAttributeMaxDynamicSharedMemorySize, smax));
        DG_CUDA(cudaFuncSetAttribute(k_seq_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, kWalkSmem));
        if (c->carveout >= 0) {
            DG_CUDA(cudaFuncSetAttribute(k_seq_walk, cudaFuncAttributePreferredSharedMemoryCarveout, c->carveout));
            DG_CUDA(cudaFuncSetAttribute(k_seq_prod, cudaFuncAttributePreferredSharedMemoryCarveout, c->carveout));
            DG_CUDA(cudaFuncSetAttribute(k_seq_tree, cudaFuncAttributePreferredSharedMemoryCarveout, c->carveout));
            DG_CUDA(cudaFuncSetAttribute(k_seq_guess, cudaFuncAttributePreferredSharedMemoryCarveout, c->carveout));
        }
    }
    double* approx = c->seq_buf;
    double* guess = approx + per;
    double* prodT = guess + per;  // [lane][stride] products of the pass
    SeqNode* nodes = reinterpret_cast<SeqNode*>(prodT + pstride * lanes);
    const size_t smem = static_cast<size_t>(kTileRows) * (nrhs + 1) * sizeof(double);
    for (int a = r0;; a += kSeqPassRows) {
        const int b = std::min(r1, a + kSeqPassRows);
        const int stride = (b - a + 1) & ~1;  // even: 16-byte aligned bulk copies per lane
        const int ntile = (b - a + kTileRows - 1) / kTileRows;
        const int nrec = (b - a + kRecRows - 1) / kRecRows;
        const int ngrp = (b - a + kGrpRows - 1) / kGrpRows;
        double* mo = b >= r1 ? mean_out : nullptr;
        const double rows = b - a, t = rows * nrhs;
        if (ntile > 0) {
            DG_TRY(launch(c, kNorms, 8.0 * rows + 16.0 * t, [&] {
                k_seq_prod<<<ntile, 256, smem, c->stream>>>(a, b, nrhs, stride, L.area, d_b, prodT, approx);
            }));
            DG_TRY(launch(c, kNorms, 16.0 * nrec * nrhs, [&] {
                k_seq_guess<<<nrhs, 1024, 0, c->stream>>>(nrec, approx, state, guess);
            }));
            DG_TRY(launch(c, kNorms, 8.0 * t + 3024.0 * ngrp * nrhs, [&] {
                k_seq_tree<<<dim3(ngrp, (nrhs + 3) / 4), 128, 0, c->stream>>>(a, b, nrhs, stride, prodT, guess,
                                                                             nodes);
            }));
        }
        DG_TRY(launch(c, kNorms, 8.0 * t + 3024.0 * ngrp * nrhs, [&] {
            k_seq_walk<<<nrhs, 32, kWalkSmem, c->stream>>>(a, b, stride, prodT, nodes, state, c->wtot0, mo,
                                                          c->seq_fallbacks);
        }));
        if (b >= r1) break;
    }
    return Status::Ok();
}

// The same chain run literally, one lane per RHS (DECMG_PROJ_SEQ=1).
Status project_chain_seq(decmg_gpu_ctx* c, int nrhs, const double* d_b, int r0, int r1, double* mean_out) {
    const Level& L = c->lv[0];
    double* state = c->dsmall + 160;
    const size_t smem = static_cast<size_t>(kProjStages) * proj_rows(nrhs) * nrhs * sizeof(double);
    if (first_on_device(c, reinterpret_cast<const void*>(k_project_sums)))
        DG_CUDA(cudaFuncSetAttribute(k_project_sums, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kProjStages * kProjTileBytes));
    double* prod = c->r;  // scratch [n0][max_nrhs]: the residual buffer is free outside a cycle
    const int64_t t = static_cast<int64_t>(r1 - r0) * nrhs;
    DG_TRY(launch(c, kNorms, 8.0 * (r1 - r0) + 16.0 * t, [&] {
        if (t > 0) k_project_products<<<grid_for(t, kBlock), kBlock, 0, c->stream>>>(r0, r1, nrhs, L.area, d_b, prod);
    }));
    return launch(c, kNorms, 8.0 * t, [&] {
        k_project_sums<<<1, 64, smem, c->stream>>>(r0, r1, nrhs, prod, c->wtot0, state, mean_out);
    });
}

Status project_chain(decmg_gpu_ctx* c, int nrhs, const double* d_b, int r0, int r1, double* mean_out) {
    return c->proj_seq ? project_chain_seq(c, nrhs, d_b, r0, r1, mean_out)
                       : project_chain_par(c, nrhs, d_b, r0, r1, mean_out);
}

Status project_subtract(decmg_gpu_ctx* c, int nrhs, const double* mean, double* d_b) {
    const Level& L = c->lv[0];
    const int bp = bp_of(nrhs);
    const unsigned g = grid_for(static_cast<int64_t>(L.nv) * bp, kBlock);
    return launch(c, kNorms, 16.0 * L.nv * nrhs, [&] {
        DISPATCH_B1(bp, k_project<BP><<<g, kBlock, 0, c->stream>>>(L.nv, nrhs, mean, d_b));
    });
}

}  // namespace

Status project_compatible(decmg_gpu_ctx* c, int nrhs, double* d_b) {
    DG_TRY(check_nrhs(c, nrhs));
    // TMA bulk copies need 16-byte aligned sources (cudaMalloc'd buffers are)
    if ((reinterpret_cast<uintptr_t>(d_b) & 15) != 0)
        return Status::Err(DECMG_INVALID_ARGUMENT, "project_compatible: rhs must be 16-byte aligned");
    double* mean = c->dsmall + 128;
    DG_CUDA(cudaMemsetAsync(c->dsmall + 160, 0, sizeof(double) * 32, c->stream));
    DG_TRY(project_chain(c, nrhs, d_b, 0, c->lv[0].nv, mean));
    return project_subtract(c, nrhs, mean, d_b);
}

// Host right-hand side -> c->bproj, projected (Neumann): the H2D copy runs in
// chunks on a second stream and the sequential mean chain follows chunk by
// chunk on the context stream, so the copy hides under the chain.
Status stage_rhs(decmg_gpu_ctx* c, int nrhs, const double* h_b, bool project, double* dst) {
    DG_TRY(check_nrhs(c, nrhs));
    const int n = c->lv[0].nv;
    if (!dst) dst = c->bproj;
    if (!project) {
        DG_CUDA(cudaMemcpyAsync(dst, h_b, sizeof(double) * n * nrhs, cudaMemcpyHostToDevice, c->stream));
        return Status::Ok();
    }
    if (!c->io_stream) DG_CUDA(cudaStreamCreateWithFlags(&c->io_stream, cudaStreamNonBlocking));
    constexpr int kChunks = 16;
    while (static_cast<int>(c->io_events.size()) < kChunks + 1) {
        cudaEvent_t e;
        DG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->io_events.push_back(e);
    }
    // the copy stream starts after everything already queued on the context stream
    DG_CUDA(cudaEventRecord(c->io_events[kChunks], c->stream));
    DG_CUDA(cudaStreamWaitEvent(c->io_stream, c->io_events[kChunks], 0));
    int per = (n + kChunks - 1) / kChunks;
    per = (per + proj_rows(nrhs) - 1) / proj_rows(nrhs) * proj_rows(nrhs);
    DG_CUDA(cudaMemsetAsync(c->dsmall + 160, 0, sizeof(double) * 32, c->stream));
    double* mean = c->dsmall + 128;
    for (int k = 0; k < kChunks; ++k) {
        const int r0 = std::min(n, k * per), r1 = std::min(n, r0 + per);
        if (r1 > r0) {
            const size_t off = static_cast<size_t>(r0) * nrhs;
            DG_CUDA(cudaMemcpyAsync(dst + off, h_b + off, sizeof(double) * (r1 - r0) * nrhs, cudaMemcpyHostToDevice,
                                    c->io_stream));
        }
        DG_CUDA(cudaEventRecord(c->io_events[k], c->io_stream));
        DG_CUDA(cudaStreamWaitEvent(c->stream, c->io_events[k], 0));
        if (r1 > r0 || k == kChunks - 1) DG_TRY(project_chain(c, nrhs, dst, r0, r1, k == kChunks - 1 ? mean : nullptr));
    }
    return project_subtract(c, nrhs, mean, dst);
}

// Device-side gmg_solve loop: one CUDA graph per (plan, batch width, buffer
// state) holding a WHILE node whose body is one cycle with the convergence
// check in the middle -- [first level-0 sweep with the fused residual norm of
// the current iterate, k_solve_check, copy of finished lanes] then an IF node
// [rest of the cycle]. The host launches it once instead of synchronising on
// every cycle's residual; every kernel and argument is the host loop's, so the
// iterates and histories are the same bits. The body is captured from
// Driver::one_cycle itself: the fused-norm hook adds the check kernels and
// the IF node to the capture and redirects the rest of the cycle into the IF
// body. One captured cycle is valid for every iteration only if the cycle
// preserves level 0's ping-pong parity (coarser levels restart from zero on
// every descent); a cycle that flips it (an odd number of level-0 Jacobi
// sweeps, e.g. V(2,1)) is detected after the capture and *graphed stays false,
// so solve() runs the host loop. The key includes every level's parity.
Status solve_graph(decmg_gpu_ctx* c, Driver& dr, const Plan& plan, int nrhs, unsigned all, double tol,
                   int max_cycles, double* denom, double* dres, int64_t total, bool* graphed) {
    *graphed = false;
    if (!c->gstate_raw) DG_TRY(dalloc(c, &c->gstate_raw, (sizeof(SolveState) + 7) / 8));
    SolveState* gst = reinterpret_cast<SolveState*>(c->gstate_raw);

    // omega by its exact bits: two omegas that print alike must not share a graph
    uint64_t omega_bits = 0;
    std::memcpy(&omega_bits, &plan.omega, sizeof omega_bits);
    std::string key = plan.walk + "|" + std::to_string(plan.smoother) + "|" + std::to_string(omega_bits) + "|" +
                      std::to_string(nrhs) + "|" + std::to_string(reinterpret_cast<uintptr_t>(dr.b0)) + "|" +
                      std::to_string(reinterpret_cast<uintptr_t>(c->hist_dev)) + "|" +
                      std::to_string(reinterpret_cast<uintptr_t>(c->tstamp_dev)) + "|" +
                      std::to_string(reinterpret_cast<uintptr_t>(c->red)) + "|" + (dr.use_pairs ? "p|" : "s|");
    for (size_t k = 0; k < c->lv.size(); ++k)
        key += std::to_string(plan.pre[k]) + "," + std::to_string(plan.post[k]) + "," +
               std::to_string(c->lv[k].cur) + std::to_string(c->lv[k].x_zero ? 1 : 0) + ";";
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
    for (auto& e : c->graphs)
        if (e.key == key) {
            exec = e.exec;
            kernels = e.kernels;
        }
    if (!exec) {
        const int64_t lc0 = c->launch_count;
        cudaGraph_t g = nullptr;
        DG_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle hw;
        DG_CUDA(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams wp = {};
        wp.type = cudaGraphNodeTypeConditional;
        wp.conditional.handle = hw;
        wp.conditional.type = cudaGraphCondTypeWhile;
        wp.conditional.size = 1;
        cudaGraphNode_t wn;
        DG_CUDA(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
        cudaGraph_t body = wp.conditional.phGraph_out[0];
        if (!c->cap_stream) DG_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        const cudaStream_t main = c->stream;
        bool split = false;
        Status hs;
        DG_CUDA(cudaStreamBeginCaptureToGraph(main, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        dr.fuse_hist = dres;
        dr.fuse_denom = denom;
        dr.fuse_hook = [&](const double* xprev, bool* stop) -> Status {
            *stop = false;
            cudaStreamCaptureStatus cs;
            cudaGraph_t cg = nullptr;
            const cudaGraphNode_t* deps = nullptr;
            size_t nd = 0;
            DG_CUDA(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cg, &deps, &nd));
            cudaGraphConditionalHandle hif;
            DG_CUDA(cudaGraphConditionalHandleCreate(&hif, cg, 0, cudaGraphCondAssignDefault));
            DG_TRY(launch(c, kNorms, 0.0, [&] {
                k_solve_check<<<1, 32, 0, c->stream>>>(nrhs, dres, gst, c->hist_dev, c->tstamp_dev, hif, hw);
            }));
            DG_TRY(launch(c, kNorms, 16.0 * static_cast<double>(total), [&] {
                k_copy_lanes_dev<<<grid_for(total, kBlock), kBlock, 0, c->stream>>>(total, nrhs, gst, xprev,
                                                                                   c->xsol);
            }));
            DG_CUDA(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cg, &deps, &nd));
            cudaGraphNodeParams ip = {};
            ip.type = cudaGraphNodeTypeConditional;
            ip.conditional.handle = hif;
            ip.conditional.type = cudaGraphCondTypeIf;
            ip.conditional.size = 1;
            cudaGraphNode_t in;
            DG_CUDA(cudaGraphAddNode(&in, cg, deps, nd, &ip));
            DG_CUDA(cudaStreamUpdateCaptureDependencies(c->stream, &in, 1, cudaStreamSetCaptureDependencies));
            DG_CUDA(cudaStreamBeginCaptureToGraph(c->cap_stream, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal));
            c->stream = c->cap_stream;  // the rest of the cycle goes into the IF body
            split = true;
            return Status::Ok();
        };
        // host view of the ping-pong state before the captured cycle: the graph
        // replays one cycle with fixed buffer pointers, which is valid only if
        // the cycle leaves level 0's parity unchanged (an even number of level-0
        // Jacobi sweeps; coarser levels restart from zero on every descent)
        std::vector<std::pair<int, bool>> st0;
        for (const Level& L : c->lv) st0.emplace_back(L.cur, L.x_zero);
        hs = dr.one_cycle(plan);
        dr.fuse_hook = nullptr;
        dr.fuse_hist = nullptr;
        kernels = c->launch_count - lc0;  // one loop iteration's kernels, recorded not run
        c->launch_count = lc0;
        cudaGraph_t tmp = nullptr;
        if (split) {
            const cudaError_t e1 = cudaStreamEndCapture(c->cap_stream, &tmp);
            if (hs.ok() && e1 != cudaSuccess) hs = cuda_status(e1, "graph capture (if body)");
        }
        c->stream = main;
        const cudaError_t e2 = cudaStreamEndCapture(main, &tmp);
        if (hs.ok() && e2 != cudaSuccess) hs = cuda_status(e2, "graph capture (loop body)");
        if (hs.ok() && !split) hs = Status::Err(DECMG_RUNTIME, "graph capture: the cycle has no fused residual");
        if (!hs.ok()) {
            cudaGraphDestroy(g);
            return hs;
        }
        if (c->lv[0].cur != st0[0].first) {
            // parity-changing cycle (e.g. V(2,1) Jacobi): nothing was executed,
            // so restore the host state and let the caller run the host loop
            cudaGraphDestroy(g);
            for (size_t k = 0; k < c->lv.size(); ++k) {
                c->lv[k].cur = st0[k].first;
                c->lv[k].x_zero = st0[k].second;
            }
            return Status::Ok();
        }
        DG_CUDA(cudaGraphInstantiate(&exec, g, 0));
        c->graphs.push_back({key, g, exec, kernels});
    }
    DG_TRY(launch(c, kNorms, 0.0, [&] { k_solve_init<<<1, 1, 0, c->stream>>>(gst, 1, all, max_cycles, tol); }));
    DG_CUDA(cudaGraphLaunch(exec, c->stream));
    c->last_graph_kernels = kernels;  // solve() multiplies by the iterations the device loop ran
    *graphed = true;
    return Status::Ok();
}

// A few device scalars -> c->hsmall, written by a kernel through the mapped
// pinned buffer rather than a copy engine (a 16-double copy would queue behind
// a concurrent 1.3 GB download in solve_batches), then synchronise.
Status small_to_host(decmg_gpu_ctx* c, const double* d_src, int n) {
    if (!c->hsmall_dev) {
        void* p = nullptr;
        DG_CUDA(cudaHostGetDevicePointer(&p, c->hsmall, 0));
        c->hsmall_dev = static_cast<double*>(p);
    }
    DG_TRY(launch(c, kNorms, 16.0 * n, [&] { k_small_copy<<<1, 32, 0, c->stream>>>(n, d_src, c->hsmall_dev); }));
    DG_CUDA(cudaStreamSynchronize(c->stream));
    return Status::Ok();
}

// gmg_solve (proj/src/solvers.cpp:251-279), batched: each RHS stops at its
// own cycle count; its solution is the iterate of that cycle.
Status solve(decmg_gpu_ctx* c, const Plan& plan, int nrhs, const double* d_b, const double* d_x0,
             double tol, int max_cycles, double* d_x, double* h_hist, int* cycles_done,
             double* h_final, bool staged, const double* bsrc) {
    DG_TRY(check_nrhs(c, nrhs));
    if (max_cycles < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_solve: max_cycles >= 0");
    const auto t_host0 = std::chrono::steady_clock::now();
    c->last_times.clear();
    if (max_cycles > c->hist_cap) {
        if (c->hist_dev) cudaFree(c->hist_dev);
        if (c->tstamp_dev) cudaFree(c->tstamp_dev);
        c->hist_dev = nullptr;
        c->tstamp_dev = nullptr;
        c->hist_cap = 0;
        DG_CUDA(cudaMalloc(&c->hist_dev, sizeof(double) * max_cycles * 32));
        DG_CUDA(cudaMalloc(&c->tstamp_dev, sizeof(unsigned long long) * (max_cycles + 1)));
        c->hist_cap = max_cycles;
    }
    if (!c->tstamp_dev) DG_CUDA(cudaMalloc(&c->tstamp_dev, sizeof(unsigned long long) * 1));
    // device clock at the start (cumulative_seconds of the graph-driven cycles)
    DG_TRY(launch(c, kNorms, 0.0, [&] { k_stamp<<<1, 1, 0, c->stream>>>(c->tstamp_dev); }));
    const double t_launch0 = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host0).count();
    auto host_elapsed = [&]() {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host0).count();
    };
    Level& L0 = c->lv[0];
    if (!bsrc) bsrc = c->bproj;
    if (!staged) {  // staged: stage_rhs already left the projected RHS in bsrc
        const size_t nbytes = sizeof(double) * L0.nv * nrhs;
        DG_CUDA(cudaMemcpyAsync(c->bproj, d_b, nbytes, cudaMemcpyDeviceToDevice, c->stream));
        if (!c->dirichlet) DG_TRY(project_compatible(c, nrhs, c->bproj));  // in the reference numbering
        bsrc = c->bproj;
    }
    Driver dr{c, nrhs, bp_of(nrhs), L0.ord ? L0.b : bsrc};
    // a batch stream stages the next batch on other streams while this one cycles: the two-sweep
    // pass is a cooperative launch (every CTA resident), which would wait for those kernels to drain
    dr.use_pairs = !c->batch_overlap || c->pair_ctas_overlap > 0;
    DG_TRY(dr.init());
    if (L0.ord) DG_TRY(dr.to_internal(bsrc, L0.b));
    double* denom = c->dsmall;
    double* dres = c->dsmall + 256;
    DG_TRY(dr.load_x0(d_x0));
    DG_TRY(dr.make_denom(denom));
    std::vector<int> done(nrhs, 0);
    std::vector<double> final_res(nrhs, 0.0);
    const unsigned all = nrhs == 32 ? 0xffffffffu : ((1u << nrhs) - 1u);
    unsigned active = all;
    const int64_t total = static_cast<int64_t>(L0.nv) * nrhs;
    int cyc = 0;
    if (max_cycles == 0) {
        DG_TRY(dr.resnorm(dres, denom));
        DG_TRY(small_to_host(c, dres, nrhs));
        for (int l = 0; l < nrhs; ++l) final_res[l] = c->hsmall[l];
    }
    // Record the residual of the iterate after `cyc` cycles (in dres) and
    // retire the right-hand sides that reached tol; xsrc holds that iterate.
    auto check = [&](const double* xsrc) -> Status {
        DG_TRY(small_to_host(c, dres, nrhs));
        unsigned fin = 0;
        for (int l = 0; l < nrhs; ++l) {
            if (!(active & (1u << l))) continue;
            const double res = c->hsmall[l];
            if (h_hist) h_hist[static_cast<int64_t>(cyc - 1) * nrhs + l] = res;
            final_res[l] = res;
            done[l] = cyc;
            if (res <= tol || cyc == max_cycles || !std::isfinite(res)) fin |= 1u << l;
        }
        if (cyc >= 1) c->last_times.push_back(host_elapsed());
        if (fin) {
            DG_TRY(launch(c, kNorms, 16.0 * L0.nv * nrhs, [&] {
                k_copy_lanes<<<grid_for(total, kBlock), kBlock, 0, c->stream>>>(total, nrhs, fin, xsrc, c->xsol);
            }));
            active &= ~fin;
        }
        return Status::Ok();
    };
    bool graphed = false;
    if (c->graph && !c->timing.enabled && max_cycles >= 2 && c->lv.size() > 1) {
        DG_TRY(dr.one_cycle(plan));  // cycle 0 (from x0; its first sweep carries no residual)
        cyc = 1;
        bool on_device = false;
        if (dr.can_fuse(plan))  // cycles 1.. on the device
            DG_TRY(solve_graph(c, dr, plan, nrhs, all, tol, max_cycles, denom, dres, total, &on_device));
        if (on_device) {
            SolveState st;
            std::vector<double> hist(static_cast<size_t>(max_cycles) * nrhs);
            std::vector<unsigned long long> ts(static_cast<size_t>(max_cycles) + 1);
            DG_CUDA(cudaMemcpyAsync(&st, c->gstate_raw, sizeof(SolveState), cudaMemcpyDeviceToHost, c->stream));
            DG_CUDA(cudaMemcpyAsync(hist.data(), c->hist_dev, sizeof(double) * hist.size(), cudaMemcpyDeviceToHost,
                                    c->stream));
            DG_CUDA(cudaMemcpyAsync(ts.data(), c->tstamp_dev, sizeof(unsigned long long) * ts.size(),
                                    cudaMemcpyDeviceToHost, c->stream));
            DG_CUDA(cudaStreamSynchronize(c->stream));
            int maxdone = 0;
            for (int l = 0; l < nrhs; ++l) maxdone = std::max(maxdone, st.done[l]);
            c->launch_count += c->last_graph_kernels * std::max(maxdone - 1, 1);  // the loop's iterations
            for (int k = 1; k <= maxdone; ++k)  // device clock of each check, offset by the host's launch delay
                c->last_times.push_back(t_launch0 + 1e-9 * static_cast<double>(ts[k] - ts[0]));
            for (int l = 0; l < nrhs; ++l) {
                done[l] = st.done[l];
                final_res[l] = st.final_res[l];
                if (h_hist)
                    for (int k = 0; k < done[l]; ++k)
                        h_hist[static_cast<int64_t>(k) * nrhs + l] = hist[static_cast<size_t>(k) * nrhs + l];
            }
            active = 0;
            graphed = true;
        }
    }
    while (!graphed && cyc < max_cycles && active) {
        if (cyc > 0 && dr.can_fuse(plan)) {
            // the first level-0 sweep of the next cycle yields the residual of
            // the current iterate; stop there if every RHS has converged
            dr.fuse_hist = dres;
            dr.fuse_denom = denom;
            dr.fuse_hook = [&](const double* xprev, bool* stop) -> Status {
                DG_TRY(check(xprev));
                *stop = active == 0;
                return Status::Ok();
            };
            dr.stopped = false;
            DG_TRY(dr.one_cycle(plan));
            dr.fuse_hook = nullptr;
            if (dr.stopped) break;
        } else {
            if (cyc > 0) {
                DG_TRY(dr.resnorm(dres, denom));
                DG_TRY(check(L0.x[L0.cur]));
                if (!active) break;
            }
            DG_TRY(dr.one_cycle(plan));
        }
        ++cyc;
    }
    if (active && cyc > 0) {  // residual of the last iterate (cycle cap or last cycle)
        DG_TRY(dr.ensure_x(0));
        DG_TRY(dr.resnorm(dres, denom));
        DG_TRY(check(L0.x[L0.cur]));
    }
    if (active) {  // max_cycles == 0: the solution is x0
        DG_TRY(dr.ensure_x(0));
        const double* src = L0.x[L0.cur];
        DG_TRY(launch(c, kNorms, 16.0 * L0.nv * nrhs, [&] {
            k_copy_lanes<<<grid_for(total, kBlock), kBlock, 0, c->stream>>>(total, nrhs, active, src, c->xsol);
        }));
    }
    DG_TRY(dr.from_internal(c->xsol, d_x));
    DG_CUDA(cudaStreamSynchronize(c->stream));
    for (int l = 0; l < nrhs; ++l) {
        if (cycles_done) cycles_done[l] = done[l];
        if (h_final) h_final[l] = final_res[l];
    }
    // NaN/Inf guard on the per-cycle residual: the lane stopped at
    // the first non-finite residual instead of cycling on to max_cycles
    for (int l = 0; l < nrhs; ++l)
        if (!std::isfinite(final_res[l]))
            return Status::Err(DECMG_RUNTIME, "gmg_solve: non-finite residual (right-hand side " + std::to_string(l) +
                                                  ", cycle " + std::to_string(done[l]) + ")");
    return Status::Ok();
}

// A stream of independent gmg_solve batches (extension x6):
// batch k+1's host-to-device copy and projection chain run on their own
// streams while batch k cycles, and batch k's solution goes back to the host
// while batch k+1 cycles. Each batch is exactly one gmg_solve (same kernels,
// same bits); only the copies and the projection overlap other batches' work.
Status solve_batches(decmg_gpu_ctx* c, const Plan& plan, int nrhs, int nbatch, const double* const* h_b, double tol,
                     int max_cycles, double* const* h_x, double* h_hist, int* cycles_done, double* h_final) {
    DG_TRY(check_nrhs(c, nrhs));
    if (nbatch < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_solve_batches: nbatch >= 0");
    if (max_cycles < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_solve: max_cycles >= 0");
    const int n0 = c->lv[0].nv;
    const size_t n = static_cast<size_t>(n0) * nrhs;
    for (int k = 0; k < nbatch; ++k)
        if (!h_b || !h_b[k]) return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_solve_batches: rhs is null");
    if (!c->bproj2) {
        DG_TRY(dalloc(c, &c->bproj2, static_cast<size_t>(n0) * c->max_nrhs));
        DG_TRY(dalloc(c, &c->io_x2, static_cast<size_t>(n0) * c->max_nrhs));
        int prio_lo = 0, prio_hi = 0;
        DG_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        DG_CUDA(cudaStreamCreateWithPriority(&c->aux_stream, cudaStreamNonBlocking, prio_lo));
        DG_CUDA(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            DG_CUDA(cudaEventCreateWithFlags(&c->ev_stage[i], cudaEventDisableTiming));
            DG_CUDA(cudaEventCreateWithFlags(&c->ev_d2h[i], cudaEventDisableTiming));
        }
        DG_CUDA(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
    }
    double* bp[2] = {c->bproj, c->bproj2};
    double* xo[2] = {c->io_x, c->io_x2};
    const bool project = !c->dirichlet;
    // staging of batch k on the auxiliary stream (its kernels are launched on
    // c->stream, so the context stream is swapped for the duration)
    auto stage = [&](int k) -> Status {
        if (c->proj_seq) {  // the literal chain uses the residual scratch: no overlap
            DG_TRY(stage_rhs(c, nrhs, h_b[k], project, bp[k & 1]));
            return cuda_status(cudaEventRecord(c->ev_stage[k & 1], c->stream), "stage event");
        }
        cudaStream_t keep = c->stream;
        c->stream = c->aux_stream;
        Status s = stage_rhs(c, nrhs, h_b[k], project, bp[k & 1]);
        if (s.ok()) s = cuda_status(cudaEventRecord(c->ev_stage[k & 1], c->aux_stream), "stage event");
        c->stream = keep;
        return s;
    };
    struct Overlap {  // the solves of this call run beside the staging of the next batch
        decmg_gpu_ctx* c;
        explicit Overlap(decmg_gpu_ctx* cc, bool on) : c(cc) { c->batch_overlap = on; }
        ~Overlap() { c->batch_overlap = false; }
    } overlap(c, nbatch > 1 && !c->proj_seq);
    DG_CUDA(cudaEventRecord(c->ev_start, c->stream));  // after everything already queued on the context
    DG_CUDA(cudaStreamWaitEvent(c->aux_stream, c->ev_start, 0));
    DG_CUDA(cudaStreamWaitEvent(c->d2h_stream, c->ev_start, 0));
    if (nbatch > 0) DG_TRY(stage(0));
    for (int k = 0; k < nbatch; ++k) {
        if (k + 1 < nbatch) DG_TRY(stage(k + 1));  // overlaps batch k's cycles
        DG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_stage[k & 1], 0));
        if (k >= 2) DG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_d2h[k & 1], 0));  // xo[k & 1] copied out
        const size_t ho = static_cast<size_t>(k) * (max_cycles > 0 ? max_cycles : 1) * nrhs;
        const auto t_solve = std::chrono::steady_clock::now();
        DG_TRY(solve(c, plan, nrhs, nullptr, nullptr, tol, max_cycles, xo[k & 1], h_hist ? h_hist + ho : nullptr,
                     cycles_done ? cycles_done + static_cast<size_t>(k) * nrhs : nullptr,
                     h_final ? h_final + static_cast<size_t>(k) * nrhs : nullptr, true, bp[k & 1]));
        // solve returned after synchronising the context stream: xo[k & 1] holds batch k
        if (std::getenv("DECMG_DEBUG"))
            std::fprintf(stderr, "solve_batches: batch %d solve %.2f ms\n", k,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_solve).count());
        if (h_x && h_x[k])
            DG_CUDA(cudaMemcpyAsync(h_x[k], xo[k & 1], n * sizeof(double), cudaMemcpyDeviceToHost, c->d2h_stream));
        DG_CUDA(cudaEventRecord(c->ev_d2h[k & 1], c->d2h_stream));
    }
    DG_CUDA(cudaStreamSynchronize(c->d2h_stream));
    DG_CUDA(cudaStreamSynchronize(c->aux_stream));
    return Status::Ok();
}

// smooth (multigrid.hpp:66-68, multigrid.cpp:95-120) on level k's operator:
// x = d_x (reference numbering) -> iters sweeps -> d_out. weighted: the CG
// smoother's inner product uses the level's dual areas (what cycle_once
// passes); otherwise plain dots (smooth's default `weights = {}`).
Status smooth_level(decmg_gpu_ctx* c, int k, const Plan& plan, int iters, int nrhs, const double* d_x,
                    const double* d_b, double* d_out, bool weighted) {
    DG_TRY(check_nrhs(c, nrhs));
    const int L = static_cast<int>(c->lv.size());
    if (k < 0 || k >= L) return Status::Err(DECMG_INVALID_ARGUMENT, "smooth: level out of range");
    if (iters < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "smooth: negative iteration count");
    Level& m = c->lv[k];
    if ((plan.smoother == DECMG_SMOOTHER_GS || plan.smoother == DECMG_SMOOTHER_SGS) && !m.gsf_rows)
        DG_TRY(build_gs_schedule(c, m));  // the coarsest level has none until asked
    Driver dr{c, nrhs, bp_of(nrhs), c->lv[0].b};
    DG_TRY(dr.init());
    const int64_t t = static_cast<int64_t>(m.nv) * nrhs;
    auto perm = [&](const double* src, double* dst, bool scatter) -> Status {
        if (!m.ord) {
            DG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * t, cudaMemcpyDeviceToDevice, c->stream));
            return Status::Ok();
        }
        return launch(c, kNorms, 16.0 * t, [&] {
            if (scatter)
                k_permute<true><<<grid_for(t, kBlock), kBlock, 0, c->stream>>>(m.nv, nrhs, m.ord, src, dst);
            else
                k_permute<false><<<grid_for(t, kBlock), kBlock, 0, c->stream>>>(m.nv, nrhs, m.ord, src, dst);
        });
    };
    DG_TRY(perm(d_b, m.b, false));
    DG_TRY(perm(d_x, m.x[m.cur], false));
    m.x_zero = false;
    double* ones = nullptr;
    if (plan.smoother == DECMG_SMOOTHER_CG && !weighted) {
        DG_CUDA(cudaMalloc(&ones, sizeof(double) * m.nv));
        DG_TRY(launch(c, kNorms, 8.0 * m.nv, [&] {
            k_fill<<<grid_for(m.nv, kBlock), kBlock, 0, c->stream>>>(m.nv, 1.0, ones);
        }));
        dr.cg_weights = ones;
    }
    Status s = dr.smooth(k, iters, plan);
    if (s.ok()) s = perm(m.x[m.cur], d_out, true);
    if (ones) {
        cudaStreamSynchronize(c->stream);
        cudaFree(ones);
    }
    return s;
}

Status apply_op(decmg_gpu_ctx* c, int level, char op, const double* d_x, double* d_y) {
    const int L = static_cast<int>(c->lv.size());
    if (level < 0 || level >= L) return Status::Err(DECMG_INVALID_ARGUMENT, "apply: level out of range");
    Level& m = c->lv[level];
    const int *rp, *ci;
    const double* v;
    int rows;
    if (op == 'L') {
        rp = m.L_rp; ci = m.L_ci; v = m.L_v; rows = m.nv;
    } else if ((op == 'P' || op == 'R') && level + 1 < L) {
        if (op == 'P') { rp = m.P_rp; ci = m.P_ci; v = m.P_v; rows = m.nv; }
        else { rp = m.R_rp; ci = m.R_ci; v = m.R_v; rows = c->lv[level + 1].nv; }
    } else {
        return Status::Err(DECMG_INVALID_ARGUMENT, "apply: unknown operator for this level");
    }
    DG_TRY(launch(c, kNorms, 0.0, [&] {
        k_spmv<1, 1, 0><<<grid_for(rows, kBlock), kBlock, 0, c->stream>>>(rows, 1, rp, ci, v, nullptr, d_x, d_y, nullptr);
    }));
    return Status::Ok();
}

}  // namespace decmg_gpu
