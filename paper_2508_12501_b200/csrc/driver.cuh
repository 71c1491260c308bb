// Single-GPU V-cycle driver (shared by cycle.cu and dist.cu, which reuses it
// for the replicated coarse levels and for launching the row kernels on a
// rank's local operators).
#pragma once

#include "rowkernels.cuh"

#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <functional>
#include <string>
#include <type_traits>

namespace decmg_gpu {
namespace {

// Dispatch the pipelined kernel on the ELL width of an operator (7 or 8).
#define PIPE_W(w, OP, ...) ((w) == 7 ? pipe<OP, 7>(__VA_ARGS__) : pipe<OP, 8>(__VA_ARGS__))

struct Driver {
    decmg_gpu_ctx* c;
    int nrhs, bp;
    const double* b0;  // level-0 right-hand side
    int key = 0;       // DISPATCH_BP key of the row kernels (10 * BP + RPT)
    int tpr = 1;       // threads per row
    // Fused residual norm: when set, the next level-0 sweep also writes
    // ||b - A x|| / denom of the x it reads into fuse_hist, then calls
    // fuse_hook(xprev, &stop); stop == true undoes the sweep's buffer flip and
    // abandons the rest of the cycle (gmg_solve's convergence exit).
    double* fuse_hist = nullptr;
    const double* fuse_denom = nullptr;
    std::function<Status(const double*, bool*)> fuse_hook;
    bool stopped = false;
    const double* cg_weights = nullptr;  // CG smoother inner-product weights (nullptr: the level's dual areas)
    bool use_pairs = true;  // two Jacobi sweeps per pass where planned (the partitioned path exchanges halos between sweeps)

    Status init() {
        const bool vec = nrhs == bp && bp >= 2;
        int rpt = vec ? (bp < c->rpt ? bp : c->rpt) : 1;
        key = 10 * bp + rpt;
        tpr = bp / rpt;
        return prepare_pairs();
    }

    // ---- two Jacobi sweeps per pass (rowkernels.cuh k_sweep_pair) ----------
    // Grid and plan of the pass for level k at this driver's tile shape, built on
    // first use and cached in the level: called from the API entry points before
    // any capture (it allocates and synchronises). pair_rows stays 0 where the
    // level has too few rounds or no ELL operator.
    template <int BP, int RPT, int W>
    Status prepare_pair_level(Level& L) {
        using G = PipeGeom<BP, RPT, W>;
        Level::PairPlan P;
        P.rows = G::ROWS;
        P.ctas = pair_ctas();
        auto kern = k_sweep_pair<BP, RPT, W, false>;
        auto kern_n = k_sweep_pair<BP, RPT, W, true>;
        for (const void* fn : {reinterpret_cast<const void*>(kern), reinterpret_cast<const void*>(kern_n)})
            if (first_on_device(c, fn)) {
                DG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(G::PSMEM)));
                if (c->carveout >= 0 && kPipeCtasPerSm * (G::PSMEM + 1024.0) <= c->carveout / 100.0 * kSmemPerSm)
                    DG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, c->carveout));
            }
        const int occ = std::min(block_occupancy(c, reinterpret_cast<const void*>(kern_n), kPipeThreads, G::PSMEM),
                                 block_occupancy(c, reinterpret_cast<const void*>(kern), kPipeThreads, G::PSMEM));
        const int grid = std::min(occ, pair_ctas()) * c->num_sms;
        // a round (grid * group tiles, both sweeps' traffic) of about 45 MB: sweep 2 finds b, the
        // operator tiles and sweep 1's output of its round still in L2 (measured: 112 rows per
        // group with 16 right-hand sides, 448 with one)
        const double round_bytes = 2.0 * (24.0 * nrhs + 12.0 * W + 4.0) * G::ROWS * std::max(grid, 1);
        const int group = c->pair_group > 0 ? c->pair_group : std::max(1, static_cast<int>(45.0e6 / round_bytes + 0.5));
        const int ntiles = (L.nv + G::ROWS - 1) / G::ROWS;
        const int per_round = std::max(grid, 1) * group;
        const int rounds = (ntiles + per_round - 1) / per_round;
        if (grid < 1 || rounds < c->pair_min_rounds) {
            L.pair_plans.push_back(P);  // grid == 0: separate sweeps
            return Status::Ok();
        }
        const int npad = (L.nv + 223) / 224 * 224;
        DG_TRY(dalloc(c, &P.ord2, npad));
        DG_TRY(dalloc(c, &P.count, rounds));
        unsigned char* flag = nullptr;
        int *nsel = nullptr, *sel = nullptr;
        void* tmp = nullptr;
        DG_CUDA(cudaMalloc(&flag, npad));
        DG_CUDA(cudaMalloc(&nsel, sizeof(int)));
        DG_CUDA(cudaMalloc(&sel, sizeof(int) * npad));
        k_pair_plan<<<grid_for(npad, kBlock), kBlock, 0, c->stream>>>(npad, W, per_round * G::ROWS, c->pair_ahead, L.Le_ci,
                                                                     L.Le_row, P.ord2, flag);
        size_t bytes = 0;
        cub::CountingInputIterator<int> ids(0);
        DG_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, ids, flag, sel, nsel, npad, c->stream));
        DG_CUDA(cudaMalloc(&tmp, bytes ? bytes : 1));
        DG_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, ids, flag, sel, nsel, npad, c->stream));
        int nd = 0;
        DG_CUDA(cudaMemcpyAsync(&nd, nsel, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        DG_CUDA(cudaStreamSynchronize(c->stream));
        DG_TRY(dalloc(c, &P.defer, std::max(nd, 1)));
        DG_CUDA(cudaMemcpyAsync(P.defer, sel, sizeof(int) * nd, cudaMemcpyDeviceToDevice, c->stream));
        DG_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(tmp);
        cudaFree(sel);
        cudaFree(nsel);
        cudaFree(flag);
        P.ndefer = nd;
        P.grid = grid;
        P.group = group;
        P.ahead = c->pair_ahead;
        P.rounds = rounds;
        L.pair_plans.push_back(P);
        if (std::getenv("DECMG_DEBUG"))
            std::fprintf(stderr, "[decmg] pair plan: %d rows, %d rows/tile, grid %d, group %d, %d rounds, %d deferred rows\n",
                         L.nv, G::ROWS, grid, group, rounds, nd);
        return Status::Ok();
    }
    // resident CTAs per SM of the two-sweep pass: one fewer beside a batch stream's staging kernels, so
    // that the cooperative launch finds room without waiting for them to drain
    int pair_ctas() const { return std::max(1, std::min(kPipeCtasPerSm, c->batch_overlap ? c->pair_ctas_overlap : c->pair_ctas)); }
    int pair_tile_rows() const {
        int rows = 0;
        DISPATCH_BP(key, { rows = PipeGeom<BP, RPT, 7>::ROWS; })
        return rows;
    }
    const Level::PairPlan* pair_plan(const Level& L) const {
        if (!use_pairs || !c->pair || tpr > 8) return nullptr;
        const int rows = pair_tile_rows();
        for (const Level::PairPlan& P : L.pair_plans)
            if (P.rows == rows && P.ctas == pair_ctas()) return P.grid > 0 ? &P : nullptr;
        return nullptr;
    }
    Status prepare_pairs() {
        if (!use_pairs || !c->pair || tpr > 8) return Status::Ok();
        const int rows = pair_tile_rows();
        for (size_t k = 0; k + 1 < c->lv.size(); ++k) {
            Level& L = c->lv[k];
            if (!L.Le_ci || !L.Le_row || L.zero_diag_row >= 0) continue;
            bool have = false;
            for (const Level::PairPlan& P : L.pair_plans) have = have || (P.rows == rows && P.ctas == pair_ctas());
            if (have) continue;
            Status st;
            DISPATCH_BP(key, { st = L.Le_w == 7 ? prepare_pair_level<BP, RPT, 7>(L) : prepare_pair_level<BP, RPT, 8>(L); })
            DG_TRY(st);
        }
        return Status::Ok();
    }
    // x[cur] -> (c->r) -> x[cur ^ 1]: two sweeps, one flip. norm: OP_SWEEP_NORM's partials of the incoming x.
    Status sweep_pair(int k, const Level::PairPlan& P, const Plan& plan, bool norm) {
        Level& L = c->lv[k];
        const double R = nrhs;
        const double bytes = 2.0 * (12.0 * L.nnzL + 4.0 * (L.nv + 1) + 24.0 * L.nv * R);
        DG_CUDA(cudaMemsetAsync(P.count, 0, sizeof(unsigned) * P.rounds, c->stream));
        Status st;
        DISPATCH_BP(key, {
            PairArgs a{};
            a.ntiles = (L.nv + P.rows - 1) / P.rows;
            a.nrhs = nrhs;
            a.eci = L.Le_ci;
            a.ev = L.Le_v;
            a.ord = L.Le_row;
            a.ord2 = P.ord2;
            a.x = xcur(L);
            a.b = bptr(k);
            a.mid = c->r;
            a.out = L.x[L.cur ^ 1];
            a.partial = c->red;
            a.defer = P.defer;
            a.ndefer = P.ndefer;
            a.count = P.count;
            a.omega = plan.omega;
            a.n = L.nv;
            a.pf = c->pf;
            a.group = P.group;
            a.ahead = P.ahead;
            st = launch(c, k == 0 ? kFineSweep : kCoarseLevels, bytes, [&] {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(P.grid);
                cfg.blockDim = dim3(kPipeThreads);
                cfg.stream = c->stream;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                if (L.Le_w == 7) {
                    cfg.dynamicSmemBytes = PipeGeom<BP, RPT, 7>::PSMEM;
                    if (norm) cudaLaunchKernelEx(&cfg, k_sweep_pair<BP, RPT, 7, true>, a);
                    else cudaLaunchKernelEx(&cfg, k_sweep_pair<BP, RPT, 7, false>, a);
                } else {
                    cfg.dynamicSmemBytes = PipeGeom<BP, RPT, 8>::PSMEM;
                    if (norm) cudaLaunchKernelEx(&cfg, k_sweep_pair<BP, RPT, 8, true>, a);
                    else cudaLaunchKernelEx(&cfg, k_sweep_pair<BP, RPT, 8, false>, a);
                }
            });
        })
        DG_TRY(st);
        L.cur ^= 1;
        L.x_zero = false;
        return Status::Ok();
    }

    const double* bptr(int k) const { return k == 0 ? b0 : c->lv[k].b; }
    static double* xcur(Level& L) { return L.x[L.cur]; }

    unsigned rows_grid(int n) const { return grid_for(static_cast<int64_t>(n) * tpr, kBlock); }

    // Launch the pipelined persistent row kernel on an ELL operator.
    // Returns the grid size in *grid (the number of norm partials for OP_RES_NORM).
    template <int OP, int W>
    Status pipe(int cls, double bytes, int nrows, const int* eci, const double* ev, const int* erow,
                const double* x, const double* b, double* out, double* partial, const int* zr, double omega,
                int* grid = nullptr) {
        Status st;
        DISPATCH_BP(key, {
            PipeArgs a{0, nrhs, eci, ev, erow, x, b, out, partial, zr, omega, nrows, c->pf, c->pfl, c->tile_group};
            // default: groups of ~224 rows (16 right-hand sides) / ~448 rows (a single one)
            if (a.group < 0) a.group = std::max(1, (nrhs >= 8 ? 224 : 448) / PipeGeom<BP, RPT, W>::ROWS);
            // beside a batch stream's staging kernels the contiguous ranges measured faster (e2e 18.7 vs 18.3 G)
            if (c->batch_overlap) a.group = 0;
            // pipelined kernel for the 7/8-wide operators (L, R), the
            // high-occupancy kernel for P (2-wide rows); env DECMG_KERNEL forces one
            const bool ell = c->kmode == 1 || (c->kmode == 2 && W == 2);
            if (ell) {
                const unsigned g = grid_for(static_cast<int64_t>(nrows) * (BP / RPT), kBlock);
                if (c->carveout >= 0 && first_on_device(c, reinterpret_cast<const void*>(k_rowop_ell<BP, RPT, W, OP>)))
                    cudaFuncSetAttribute(k_rowop_ell<BP, RPT, W, OP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         c->carveout);
                st = launch(c, cls, bytes, [&] { k_rowop_ell<BP, RPT, W, OP><<<g, kBlock, 0, c->stream>>>(a, nrows); });
                if (grid) *grid = static_cast<int>(g);
            } else {  // persistent pipelined kernel with the TMA-bulk index ring
                using G = PipeGeom<BP, RPT, W>;
                static_assert((G::ROWS * 4 % 16 == 0 && G::CI_BYTES % 16 == 0) || BP / RPT > 8, "pipe tile");
                const int ntiles = (nrows + G::ROWS - 1) / G::ROWS;
                const int per_sm = kPipeCtasPerSm;
                const int g = ntiles < per_sm * c->num_sms ? ntiles : per_sm * c->num_sms;
                if (first_on_device(c, reinterpret_cast<const void*>(k_rowop_pipe<BP, RPT, W, OP>))) {
                    cudaFuncSetAttribute(k_rowop_pipe<BP, RPT, W, OP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(G::PSMEM));
                    // the common carve-out only where all per_sm CTAs still fit in it (the
                    // single-RHS tiles need ~80 KB each: the driver's choice keeps them resident)
                    if (c->carveout >= 0 &&
                        per_sm * (G::PSMEM + 1024.0) <= c->carveout / 100.0 * kSmemPerSm)
                        cudaFuncSetAttribute(k_rowop_pipe<BP, RPT, W, OP>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout, c->carveout);
                }
                a.ntiles = ntiles;
                // round-robin tile groups only where every CTA gets many of them (small
                // levels keep one contiguous range per CTA: a short last round would unbalance them)
                if (a.group > 0 && static_cast<int64_t>(ntiles) < 16ll * a.group * g) a.group = 0;
                st = launch(c, cls, bytes, [&] {
                    k_rowop_pipe<BP, RPT, W, OP><<<g, kPipeThreads, G::PSMEM, c->stream>>>(a);
                });
                if (grid) *grid = g;
            }
        })
        return st;
    }

    template <int OP, class... A>
    Status pipe_w(int w, A... a) {
        return w == 7 ? pipe<OP, 7>(a...) : pipe<OP, 8>(a...);
    }

    Status ensure_x(int k) {
        Level& L = c->lv[k];
        if (L.x_zero) {
            DG_CUDA(cudaMemsetAsync(xcur(L), 0, sizeof(double) * L.nv * nrhs, c->stream));
            L.x_zero = false;
        }
        return Status::Ok();
    }

    // One exact Gauss-Seidel sweep on level k: its phases in order, x in place.
    Status gs_sweep(int k, bool reverse) {
        DG_TRY(ensure_x(k));
        Level& L = c->lv[k];
        const std::vector<int>& ptr = reverse ? L.gsr_ptr : L.gsf_ptr;
        const int* rows = reverse ? L.gsr_rows : L.gsf_rows;
        if (!rows) return Status::Err(DECMG_RUNTIME, "gauss_seidel: no schedule on this level");
        double* x = xcur(L);
        const double* b = bptr(k);
        const bool ell = L.Le_ci && tpr <= 8;
        const int cls = k == 0 ? kFineSweep : kCoarseLevels;
        for (size_t p = 0; p + 1 < ptr.size(); ++p) {
            const int nr = ptr[p + 1] - ptr[p];
            if (nr == 0) continue;
            const double bytes = 12.0 * L.nnzL * nr / L.nv + 8.0 * nr + 24.0 * nr * nrhs;
            const int* rp = rows + ptr[p];
            DG_TRY(launch(c, cls, bytes, [&] {
                const unsigned g = grid_for(static_cast<int64_t>(nr) * tpr, kBlock);
                DISPATCH_BP(key, {
                    if (ell && L.Le_w == 7)
                        k_gs_phase<BP, RPT, 7><<<g, kBlock, 0, c->stream>>>(nr, rp, nrhs, nullptr, L.Le_ci, L.Le_v,
                                                                            L.Le_row, x, b);
                    else if (ell)
                        k_gs_phase<BP, RPT, 8><<<g, kBlock, 0, c->stream>>>(nr, rp, nrhs, nullptr, L.Le_ci, L.Le_v,
                                                                            L.Le_row, x, b);
                    else
                        k_gs_phase<BP, RPT, 0><<<g, kBlock, 0, c->stream>>>(nr, rp, nrhs, L.Lo_rp, L.Lo_ci, L.Lo_v,
                                                                            nullptr, x, b);
                })
            }));
        }
        L.x_zero = false;
        return Status::Ok();
    }

    // cg_fixed (multigrid.cpp:63-91) on level k with the level's dual areas as
    // weights (smooth's `weights`, cycle_once passes lvl.ops.dual_areas):
    // iters CG steps from the current x, per lane, no convergence exit. The
    // weighted dots are fixed-shape trees (the reference's are sequential).
    Status cg_smooth(int k, int iters) {
        DG_TRY(ensure_x(k));
        Level& L = c->lv[k];
        const int n = L.nv;
        const size_t nv0 = static_cast<size_t>(c->lv[0].nv) * c->max_nrhs;
        if (!c->cgs_buf) {
            DG_TRY(dalloc(c, &c->cgs_buf, 3 * nv0));
            DG_TRY(dalloc(c, &c->cgs_s, 8 * 32));
        }
        double* r = c->cgs_buf;
        double* p = r + nv0;
        double* ap = p + nv0;
        double* rr = c->cgs_s;
        double* curv = c->cgs_s + 32;
        double* alpha = c->cgs_s + 64;
        double* rrn = c->cgs_s + 96;
        double* beta = c->cgs_s + 128;
        int* done = reinterpret_cast<int*>(c->cgs_s + 160);
        double* x = xcur(L);
        const double* b = bptr(k);
        const double* w = cg_weights ? cg_weights : L.area_i;
        const int cls = k == 0 ? kFineSweep : kCoarseLevels;
        const unsigned g = rows_grid(n);
        const double mbytes = 12.0 * L.nnzL + 4.0 * (n + 1) + 16.0 * n * nrhs;
        auto spmv = [&](const double* v, const double* bb, double* y, int op) -> Status {
            if (L.Le_ci && tpr <= 8) {
                if (op == OP_RES_STORE)
                    return pipe_w<OP_RES_STORE>(L.Le_w, cls, mbytes, n, L.Le_ci, L.Le_v, L.Le_row, v, bb, y, nullptr,
                                                nullptr, 0.0, nullptr);
                return pipe_w<OP_SPMV>(L.Le_w, cls, mbytes, n, L.Le_ci, L.Le_v, L.Le_row, v, nullptr, y, nullptr,
                                       nullptr, 0.0, nullptr);
            }
            return launch(c, cls, mbytes, [&] {
                if (op == OP_RES_STORE) {
                    DISPATCH_BP(key, (k_residual<BP, RPT, 0, true><<<g, kBlock, 0, c->stream>>>(
                                        n, nrhs, L.Lo_rp, L.Lo_ci, L.Lo_v, nullptr, v, bb, y, nullptr)))
                } else {
                    DISPATCH_BP(key, (k_spmv<BP, RPT, 0><<<g, kBlock, 0, c->stream>>>(n, nrhs, L.Lo_rp, L.Lo_ci, L.Lo_v,
                                                                                      nullptr, v, y, nullptr)))
                }
            });
        };
        auto wdot = [&](const double* a, const double* bb, double* out) -> Status {
            DG_TRY(launch(c, cls, 24.0 * n * nrhs, [&] {
                DISPATCH_BP(key, k_wdot<BP, RPT><<<g, kBlock, 0, c->stream>>>(n, nrhs, w, a, bb, c->red));
            }));
            return reduce_partials(partial_blocks(n), out, 0, nullptr);
        };
        const size_t vb = sizeof(double) * static_cast<size_t>(n) * nrhs;
        DG_TRY(spmv(x, b, r, OP_RES_STORE));  // r = b - A x
        DG_CUDA(cudaMemcpyAsync(p, r, vb, cudaMemcpyDeviceToDevice, c->stream));
        DG_CUDA(cudaMemsetAsync(done, 0, sizeof(int) * 32, c->stream));
        DG_TRY(wdot(r, r, rr));
        for (int it = 0; it < iters; ++it) {
            DG_TRY(launch(c, kNorms, 0.0, [&] { k_cgs_start<<<1, 32, 0, c->stream>>>(nrhs, rr, done); }));
            DG_TRY(spmv(p, nullptr, ap, OP_SPMV));
            DG_TRY(wdot(p, ap, curv));
            DG_TRY(launch(c, kNorms, 0.0, [&] { k_cgs_alpha<<<1, 32, 0, c->stream>>>(nrhs, rr, curv, alpha, done); }));
            DG_TRY(launch(c, cls, 48.0 * n * nrhs, [&] {
                DISPATCH_BP(key, (k_cgs_update<BP, RPT, false><<<g, kBlock, 0, c->stream>>>(n, nrhs, alpha, done, x, r,
                                                                                          p, ap)));
            }));
            DG_TRY(wdot(r, r, rrn));
            DG_TRY(launch(c, kNorms, 0.0, [&] { k_cgs_beta<<<1, 32, 0, c->stream>>>(nrhs, rr, rrn, beta, done); }));
            DG_TRY(launch(c, cls, 24.0 * n * nrhs, [&] {
                DISPATCH_BP(key, (k_cgs_update<BP, RPT, true><<<g, kBlock, 0, c->stream>>>(n, nrhs, beta, done, nullptr,
                                                                                         r, p, nullptr)));
            }));
        }
        L.x_zero = false;
        return Status::Ok();
    }

    Status smooth(int k, int iters, const Plan& plan) {
        Level& L = c->lv[k];
        if (iters <= 0) return Status::Ok();
        if (plan.smoother == DECMG_SMOOTHER_CG) return cg_smooth(k, iters);
        if (plan.smoother != DECMG_SMOOTHER_JACOBI) {  // smooth (multigrid.cpp:95-120)
            if (L.zero_diag_row >= 0)
                return Status::Err(DECMG_RUNTIME,
                                   "gauss_seidel: zero diagonal at row " + std::to_string(L.zero_diag_row));
            for (int it = 0; it < iters; ++it) {
                DG_TRY(gs_sweep(k, false));
                if (plan.smoother == DECMG_SMOOTHER_SGS) DG_TRY(gs_sweep(k, true));
            }
            return Status::Ok();
        }
        if (L.zero_diag_row >= 0)
            return Status::Err(DECMG_RUNTIME, "jacobi: zero diagonal at row " + std::to_string(L.zero_diag_row));
        const double R = nrhs;
        for (int it = 0; it < iters;) {
            const bool fuse_norm = k == 0 && it == 0 && fuse_hist && !L.x_zero;
            double* xo = L.x[L.cur ^ 1];
            const double* b = bptr(k);
            if (L.x_zero) {
                const double bytes = 8.0 * L.nv + 16.0 * L.nv * R;
                if (c->carveout >= 0) {
                    DISPATCH_BP(key, {
                        if (first_on_device(c, reinterpret_cast<const void*>(k_sweep_zero<BP, RPT>)))
                            cudaFuncSetAttribute(k_sweep_zero<BP, RPT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                 c->carveout);
                    })
                }
                DG_TRY(launch(c, kZeroSweep, bytes, [&] {
                    DISPATCH_BP(key, k_sweep_zero<BP, RPT><<<rows_grid(L.nv), kBlock, 0, c->stream>>>(
                                        L.nv, nrhs, L.diag_i, b, xo, plan.omega));
                }));
            } else if (const Level::PairPlan* P = it + 2 <= iters ? pair_plan(L) : nullptr) {
                // two sweeps in one pass; the fused norm is of the x that enters the pair
                const double* xprev = xcur(L);
                DG_TRY(sweep_pair(k, *P, plan, fuse_norm));
                it += 2;
                if (fuse_norm) {
                    DG_TRY(reduce_partials(P->grid, fuse_hist, 2, fuse_denom));
                    fuse_hist = nullptr;
                    if (fuse_hook) {
                        bool stop = false;
                        DG_TRY(fuse_hook(xprev, &stop));
                        if (stop) {
                            L.cur ^= 1;  // x_prev stays the current iterate
                            stopped = true;
                            return Status::Ok();
                        }
                    }
                }
                continue;
            } else {
                const double bytes = 12.0 * L.nnzL + 4.0 * (L.nv + 1) + 24.0 * L.nv * R;
                const double* x = xcur(L);
                if (fuse_norm && L.Le_ci && tpr <= 8) {
                    int g = 0;
                    DG_TRY(PIPE_W(L.Le_w, OP_SWEEP_NORM, kFineSweep, bytes, L.nv, L.Le_ci, L.Le_v, L.Le_row, x, b,
                                  xo, c->red, nullptr, plan.omega, &g));
                    DG_TRY(reduce_partials(g, fuse_hist, 2, fuse_denom));
                    fuse_hist = nullptr;
                    L.cur ^= 1;
                    L.x_zero = false;
                    ++it;
                    if (fuse_hook) {
                        bool stop = false;
                        DG_TRY(fuse_hook(L.x[L.cur ^ 1], &stop));
                        if (stop) {
                            L.cur ^= 1;  // x_prev stays the current iterate
                            stopped = true;
                            return Status::Ok();
                        }
                    }
                    continue;
                } else if (L.Le_ci && tpr <= 8) {
                    DG_TRY(PIPE_W(L.Le_w, OP_SWEEP, k == 0 ? kFineSweep : kCoarseLevels, bytes, L.nv, L.Le_ci,
                                  L.Le_v, L.Le_row, x, b, xo, nullptr, nullptr, plan.omega, nullptr));
                } else {
                    DG_TRY(launch(c, k == 0 ? kFineSweep : kCoarseLevels, bytes, [&] {
                        DISPATCH_BP(key, (k_sweep<BP, RPT, 0><<<rows_grid(L.nv), kBlock, 0, c->stream>>>(
                                            L.nv, nrhs, L.Lo_rp, L.Lo_ci, L.Lo_v, nullptr, x, b, xo, plan.omega)))
                    }));
                }
            }
            L.cur ^= 1;
            L.x_zero = false;
            ++it;
        }
        return Status::Ok();
    }

    // r = b - A x on level k, then b_{k+1} = R r (multigrid.cpp:263-267)
    Status residual_restrict(int k) {
        DG_TRY(ensure_x(k));
        Level& L = c->lv[k];
        Level& C = c->lv[k + 1];
        const double R = nrhs;
        const double* x = xcur(L);
        const double* b = bptr(k);
        const double rbytes = 12.0 * L.nnzL + 4.0 * (L.nv + 1) + 24.0 * L.nv * R;
        if (L.Le_ci && tpr <= 8) {
            DG_TRY(PIPE_W(L.Le_w, OP_RES_STORE, k == 0 ? kFineResidual : kCoarseLevels, rbytes, L.nv, L.Le_ci,
                          L.Le_v, L.Le_row, x, b, c->r, nullptr, nullptr, 0.0, nullptr));
        } else {
            DG_TRY(launch(c, k == 0 ? kFineResidual : kCoarseLevels, rbytes, [&] {
                DISPATCH_BP(key, (k_residual<BP, RPT, 0, true><<<rows_grid(L.nv), kBlock, 0, c->stream>>>(
                                    L.nv, nrhs, L.Lo_rp, L.Lo_ci, L.Lo_v, nullptr, x, b, c->r, nullptr)))
            }));
        }
        const double tbytes = 12.0 * L.nnzR + 4.0 * (C.nv + 1) + 8.0 * L.nv * R + 8.0 * C.nv * R;
        const int* zr = c->dirichlet ? C.bd_i : nullptr;
        if (L.Re_ci && tpr <= 8) {
            DG_TRY(PIPE_W(L.Re_w, OP_SPMV, k == 0 ? kRestrict : kCoarseLevels, tbytes, C.nv, L.Re_ci, L.Re_v,
                          L.Re_row, c->r, nullptr, C.b, nullptr, zr, 0.0, nullptr));
        } else {
            DG_TRY(launch(c, k == 0 ? kRestrict : kCoarseLevels, tbytes, [&] {
                DISPATCH_BP(key, (k_spmv<BP, RPT, 0><<<rows_grid(C.nv), kBlock, 0, c->stream>>>(
                                    C.nv, nrhs, L.Ro_rp, L.Ro_ci, L.Ro_v, nullptr, c->r, C.b, zr)))
            }));
        }
        return Status::Ok();
    }

    // x_k += P_k x_{k+1}
    Status prolong(int k) {
        DG_TRY(ensure_x(k));
        DG_TRY(ensure_x(k + 1));
        Level& L = c->lv[k];
        Level& C = c->lv[k + 1];
        const double R = nrhs;
        const double bytes = 12.0 * L.nnzP + 4.0 * (L.nv + 1) + 8.0 * C.nv * R + 16.0 * L.nv * R;
        const double* xc = xcur(C);
        double* xf = xcur(L);
        if (L.Pe_ci && tpr <= 8) {
            DG_TRY((pipe<OP_PROLONG, 2>(k == 0 ? kProlong : kCoarseLevels, bytes, L.nv, L.Pe_ci, L.Pe_v, L.Le_row,
                                        xc, nullptr, xf, nullptr, nullptr, 0.0)));
        } else {
            DG_TRY(launch(c, k == 0 ? kProlong : kCoarseLevels, bytes, [&] {
                DISPATCH_BP(key, (k_prolong_add<BP, RPT, 0><<<rows_grid(L.nv), kBlock, 0, c->stream>>>(
                                    L.nv, nrhs, L.Po_rp, L.Po_ci, L.Po_v, nullptr, xc, xf)))
            }));
        }
        return Status::Ok();
    }

    Status coarse_solve(int k) {
        Level& L = c->lv[k];
        double* x = xcur(L);
        const double* b = bptr(k);
        const int project = c->dirichlet ? 0 : 1;
        if (L.nv <= 32) {  // one warp per right-hand side
            DG_TRY(launch(c, kCoarseSolve, 0.0, [&] {
                k_coarse_cg_warp<<<(nrhs + 7) / 8, 256, 0, c->stream>>>(L.nv, nrhs, L.L_rp, L.L_ci, L.L_v, L.area,
                                                                         L.wtot, project, b, x);
            }));
        } else {  // the tree-sum CG over a cooperative grid
            const int nchunks = (L.nv + kCgChunk - 1) / kCgChunk;
            if (!c->cg_grid_buf) DG_TRY(dalloc(c, &c->cg_grid_buf, 2 * static_cast<size_t>(nchunks) * 32 + 256));
            const size_t nv = static_cast<size_t>(L.nv) * nrhs;
            CoarseGridArgs a{L.nv, nrhs, project, L.L_rp, L.L_ci, L.L_v, L.area, L.wtot, b, x,
                             c->coarse_scratch, c->coarse_scratch + nv, c->coarse_scratch + 2 * nv,
                             c->coarse_scratch + 3 * nv, c->cg_grid_buf + 256, c->cg_grid_buf};
            const size_t smem = static_cast<size_t>(kCgChunk) * nrhs * sizeof(double);
            const void* fn = reinterpret_cast<const void*>(k_coarse_cg_grid);
            if (first_on_device(c, fn))
                DG_CUDA(cudaFuncSetAttribute(k_coarse_cg_grid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kCgChunk * 32 * sizeof(double))));
            const int per_sm = block_occupancy(c, fn, kCgChunk, kCgChunk * 32 * sizeof(double));
            if (per_sm < 1) return Status::Err(DECMG_CUDA, "coarse CG kernel does not fit on an SM");
            const int g = std::min(nchunks, per_sm * c->num_sms);
            DG_TRY(launch(c, kCoarseSolve, 0.0, [&] {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(g);
                cfg.blockDim = dim3(kCgChunk);
                cfg.dynamicSmemBytes = smem;
                cfg.stream = c->stream;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, k_coarse_cg_grid, a);
            }));
        }
        L.x_zero = false;
        return Status::Ok();
    }

    // The bottom of a V from `level` (walk[w] == 'd') in one cooperative kernel
    // (rowkernels.cuh k_vtail) when every pass below is small: the walk from w
    // must be d^m u^m down to the coarsest, Jacobi, ELL operators everywhere,
    // at least one pre-sweep per level. Returns false (nothing launched) if not.
    bool tail_ok(const Plan& plan, int w, int level) const {
        const int Lc = static_cast<int>(c->lv.size());
        const int m = Lc - 1 - level;
        if (!c->vtail || level < 1 || m < 1 || m >= kTailMax || tpr > 8 || fuse_hist) return false;
        if (c->lv.back().nv > 32) return false;  // larger coarse solves run the tree-sum grid CG
        if (plan.smoother != DECMG_SMOOTHER_JACOBI) return false;
        if (static_cast<int64_t>(c->lv[level].nv) * tpr > c->vtail_items) return false;  // (row, lane group) thread items
        if (w + 2 * m > static_cast<int>(plan.walk.size())) return false;
        for (int i = 0; i < m; ++i)
            if (plan.walk[w + i] != 'd' || plan.walk[w + m + i] != 'u') return false;
        for (int k = level; k < Lc - 1; ++k) {
            const Level& L = c->lv[k];
            if (!L.Le_ci || !L.Re_ci || !L.Pe_ci || !L.Le_row || !L.Re_row || plan.pre[k] < 1 ||
                L.zero_diag_row >= 0)
                return false;
        }
        return true;
    }

    Status run_tail(const Plan& plan, int level) {
        const int Lc = static_cast<int>(c->lv.size());
        const int nl = Lc - level;
        TailArgs a{};
        a.nl = nl;
        a.nrhs = nrhs;
        a.project = c->dirichlet ? 0 : 1;
        a.omega = plan.omega;
        const Level& Cst = c->lv[Lc - 1];
        a.crp = Cst.L_rp;
        a.cci = Cst.L_ci;
        a.cv = Cst.L_v;
        a.carea = Cst.area;
        a.cwtot = Cst.wtot;
        a.cta_items = c->vtail_cta_items;
        a.trace = c->vtail_trace;
        for (int i = 0; i < nl; ++i) {
            const Level& L = c->lv[level + i];
            TailLevel& T = a.lv[i];
            T.nv = L.nv;
            T.Lw = L.Le_w;
            T.Rw = L.Re_w;
            T.pre = plan.pre[level + i];
            T.post = plan.post[level + i];
            T.cur = L.cur;
            T.xzero = L.x_zero ? 1 : 0;
            T.Lci = L.Le_ci;
            T.Lv = L.Le_v;
            T.Lrow = L.Le_row;
            T.Rci = L.Re_ci;
            T.Rv = L.Re_v;
            T.Rrow = L.Re_row;
            T.Pci = L.Pe_ci;
            T.Pv = L.Pe_v;
            T.diag = L.diag_i;
            T.bdc = (c->dirichlet && i + 1 < nl) ? c->lv[level + i + 1].bd_i : nullptr;
            T.x[0] = L.x[0];
            T.x[1] = L.x[1];
            T.b = const_cast<double*>(bptr(level + i));
        }
        Status st;
        DISPATCH_BP(key, {
            auto kern = k_vtail<BP, RPT>;
            // every resident CTA (the passes of mid-size levels are latency-bound)
            const int per_sm = std::min(block_occupancy(c, reinterpret_cast<const void*>(kern), kBlock, 0),
                                        c->vtail_ctas_per_sm);
            const int blocks = per_sm >= 1 ? per_sm * c->num_sms : 0;
            if (blocks == 0) {
                st = Status::Err(DECMG_CUDA, "bottom-of-V kernel does not fit on an SM");
            } else {
                st = launch(c, kCoarseLevels, 0.0, [&] {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(blocks);
                    cfg.blockDim = dim3(kBlock);
                    cfg.dynamicSmemBytes = 0;
                    cfg.stream = c->stream;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeCooperative;
                    at[0].val.cooperative = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    cudaLaunchKernelEx(&cfg, kern, a);
                });
            }
        })
        DG_TRY(st);
        // the host's view of the levels after the tail: each sweep flipped the ping-pong buffer
        for (int i = 0; i < nl; ++i) {
            Level& L = c->lv[level + i];
            if (i + 1 < nl) L.cur ^= (plan.pre[level + i] + plan.post[level + i]) & 1;
            L.x_zero = false;
        }
        return Status::Ok();
    }

    // MultigridHierarchy::cycle_once (multigrid.cpp:252-285)
    Status cycle_once(const Plan& plan) {
        const int nw = static_cast<int>(plan.walk.size());
        const int Lc = static_cast<int>(c->lv.size());
        int level = 0;
        for (int w = 0; w < nw; ++w) {
            if (plan.walk[w] == 'd' && tail_ok(plan, w, level)) {
                DG_TRY(run_tail(plan, level));
                w += 2 * (Lc - 1 - level) - 1;  // the walk resumes with the 'u' out of `level`
                continue;
            }
            if (plan.walk[w] == 'd') {
                DG_TRY(smooth(level, plan.pre[level], plan));
                if (stopped) return Status::Ok();
                DG_TRY(residual_restrict(level));
                ++level;
                c->lv[level].x_zero = true;  // kernels::fill(0.0, xs[level])
                if (level == Lc - 1) {
                    DG_TRY(coarse_solve(level));
                } else if (w + 1 < nw && plan.walk[w + 1] == 'u') {
                    DG_TRY(smooth(level, plan.pre[level], plan));
                }
            } else {
                DG_TRY(prolong(level - 1));
                --level;
                DG_TRY(smooth(level, plan.post[level], plan));
            }
        }
        return Status::Ok();
    }

    int partial_blocks(int n) const { return static_cast<int>(rows_grid(n)); }

    // Fold nrows partial rows ([nrows][bp] in c->red) down to one row.
    Status reduce_partials(int64_t nrows, double* out, int mode, const double* denom) {
        double* in = c->red;
        double* nxt = c->red + c->red_cap / 2;
        while (nrows > 1) {
            const int64_t threads = nrows * bp;
            const unsigned g = grid_for(threads, kBlock);
            DG_TRY(launch(c, kNorms, 8.0 * threads, [&] {
                DISPATCH_B1(bp, k_fold<BP><<<g, kBlock, 0, c->stream>>>(nrows, in, nxt));
            }));
            nrows = g;
            std::swap(in, nxt);
        }
        DG_TRY(launch(c, kNorms, 0.0, [&] { k_finalize<<<1, 32, 0, c->stream>>>(nrhs, in, out, mode, denom); }));
        return Status::Ok();
    }

    // out[lane] = ||b||_2 over level-0 rows of vector v (mode 1) or sum (0)
    Status sumsq(const double* v, double* out, int mode) {
        const int n = c->lv[0].nv;
        DG_TRY(launch(c, kNorms, 8.0 * n * nrhs, [&] {
            DISPATCH_BP(key, k_sumsq<BP, RPT><<<rows_grid(n), kBlock, 0, c->stream>>>(n, nrhs, v, c->red));
        }));
        return reduce_partials(partial_blocks(n), out, mode, nullptr);
    }

    // hist[lane] = ||b - A x||_2 / denom[lane] on level 0 (multigrid.cpp:317-319)
    Status resnorm(double* hist, const double* denom) {
        DG_TRY(ensure_x(0));
        Level& L = c->lv[0];
        const double* x = xcur(L);
        const double bytes = 12.0 * L.nnzL + 4.0 * (L.nv + 1) + 16.0 * L.nv * nrhs;
        if (L.Le_ci && tpr <= 8) {
            int g = 0;
            DG_TRY(PIPE_W(L.Le_w, OP_RES_NORM, kFineResidual, bytes, L.nv, L.Le_ci, L.Le_v, L.Le_row, x, b0,
                          nullptr, c->red, nullptr, 0.0, &g));
            return reduce_partials(g, hist, 2, denom);
        }
        DG_TRY(launch(c, kFineResidual, bytes, [&] {
            DISPATCH_BP(key, (k_residual<BP, RPT, 0, false><<<rows_grid(L.nv), kBlock, 0, c->stream>>>(
                                L.nv, nrhs, L.Lo_rp, L.Lo_ci, L.Lo_v, nullptr, x, b0, nullptr, c->red)))
        }));
        return reduce_partials(partial_blocks(L.nv), hist, 2, denom);
    }

    // denom[lane] = ||b|| > 0 ? ||b|| : 1   (multigrid.cpp:307-308)
    Status make_denom(double* denom) {
        double* bn = c->dsmall + 64;
        DG_TRY(sumsq(b0, bn, 1));
        DG_TRY(launch(c, kNorms, 0.0, [&] { k_denom<<<1, 32, 0, c->stream>>>(nrhs, bn, denom); }));
        return Status::Ok();
    }

    // Can the next cycle's first level-0 sweep carry the residual norm of the
    // current iterate? (walk starts with a level-0 pre-smoothing on the
    // pipelined path and x is materialized)
    bool can_fuse(const Plan& plan) const {
        const Level& L = c->lv[0];
        return c->lv.size() > 1 && plan.smoother == DECMG_SMOOTHER_JACOBI && !plan.walk.empty() &&
               plan.walk[0] == 'd' && plan.pre[0] >= 1 && !L.x_zero &&
               L.Le_ci && tpr <= 8 && L.zero_diag_row < 0;
    }

    Status one_cycle(const Plan& plan) {
        if (c->lv.size() == 1) return coarse_solve(0);
        return cycle_once(plan);
    }

    // Level-0 vectors between the reference numbering (API) and the internal
    // one (common.cuh Level::ord): dst[q] = src[ord[q]] / dst[ord[q]] = src[q].
    Status to_internal(const double* src, double* dst) {
        const Level& L = c->lv[0];
        const int64_t t = static_cast<int64_t>(L.nv) * nrhs;
        if (!L.ord) {
            DG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * t, cudaMemcpyDeviceToDevice, c->stream));
            return Status::Ok();
        }
        const bool v4 = nrhs % 4 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 31) == 0;
        return launch(c, kNorms, 16.0 * t, [&] {
            if (v4)
                k_permute4<false><<<grid_for(t / 4, kBlock), kBlock, 0, c->stream>>>(L.nv, nrhs, L.ord, src, dst);
            else
                k_permute<false><<<grid_for(t, kBlock), kBlock, 0, c->stream>>>(L.nv, nrhs, L.ord, src, dst);
        });
    }
    Status from_internal(const double* src, double* dst) {
        const Level& L = c->lv[0];
        const int64_t t = static_cast<int64_t>(L.nv) * nrhs;
        if (!L.ord) {
            DG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * t, cudaMemcpyDeviceToDevice, c->stream));
            return Status::Ok();
        }
        const bool v4 = nrhs % 4 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 31) == 0;
        return launch(c, kNorms, 16.0 * t, [&] {
            if (v4)
                k_permute4<true><<<grid_for(t / 4, kBlock), kBlock, 0, c->stream>>>(L.nv, nrhs, L.ord, src, dst);
            else
                k_permute<true><<<grid_for(t, kBlock), kBlock, 0, c->stream>>>(L.nv, nrhs, L.ord, src, dst);
        });
    }

    Status load_x0(const double* d_x0) {
        Level& L = c->lv[0];
        if (d_x0) {
            DG_TRY(to_internal(d_x0, xcur(L)));
            L.x_zero = false;
        } else {
            L.x_zero = true;
        }
        return Status::Ok();
    }
};

Status check_nrhs(const decmg_gpu_ctx* c, int nrhs) {
    if (nrhs < 1 || nrhs > c->max_nrhs || nrhs > 32)
        return Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs] (max 32)");
    return Status::Ok();
}

}  // namespace
}  // namespace decmg_gpu
