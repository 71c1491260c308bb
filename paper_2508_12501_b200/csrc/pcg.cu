// GMG-preconditioned CG: gmg_preconditioned_cg (proj/src/solvers.cpp:118-130)
// = weighted_cg (solvers.cpp:56-116) on the level-0 operator with the dual
// areas as weights and run_cycle(inner plan, r, 0) as the preconditioner,
// after project_compatible(b). Batched: every right-hand side is one lane with
// its own alpha, beta and stopping iteration; a lane that has stopped keeps
// its x and r.
//
// Arithmetic per element is the reference's (x += alpha p, r -= alpha Ap,
// p = z + beta p, (w a) c products, alpha = rz / curv, beta = rz_new / rz);
// the weighted dots and norms are fixed-shape trees (deterministic run to run)
// instead of the reference's sequential sums, so iterates agree to rounding
// and residual histories within the 1e-10 bar (tests/test_gpu_pcg.py).
// Vectors live in the internal numbering (common.cuh Level::ord).
#include "driver.cuh"

#include <chrono>

#include <cmath>
#include <string>
#include <vector>

namespace decmg_gpu {

Status pcg(decmg_gpu_ctx* c, const Plan& inner, int inner_cycles, int nrhs, const double* d_b, double tol,
           int maxiter, double* d_x, double* h_hist, int* iters, int* converged, double* h_final, bool staged) {
    DG_TRY(check_nrhs(c, nrhs));
    const auto t_host0 = std::chrono::steady_clock::now();
    auto host_elapsed = [&]() {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host0).count();
    };
    c->last_times.clear();
    if (c->dirichlet)
        return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_pcg: Neumann hierarchies only (the reference projects b)");
    if (maxiter < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_pcg: maxiter >= 0");
    if (inner_cycles < 1) return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_pcg: inner plan needs cycles >= 1");
    Level& L0 = c->lv[0];
    const int n = L0.nv;
    const size_t nv = static_cast<size_t>(n) * c->max_nrhs;
    if (!c->pcg_buf) {
        DG_TRY(dalloc(c, &c->pcg_buf, 5 * nv));
        DG_TRY(dalloc(c, &c->pcg_s, 8 * 32));
    }
    double* bc = c->pcg_buf;
    double* x = bc + nv;
    double* r = x + nv;
    double* p = r + nv;
    double* ap = p + nv;
    double* denom = c->pcg_s;
    double* rz = c->pcg_s + 32;
    double* curv = c->pcg_s + 64;
    double* alpha = c->pcg_s + 96;
    double* rzn = c->pcg_s + 128;
    double* beta = c->pcg_s + 160;
    double* res = c->pcg_s + 192;
    const size_t vb = sizeof(double) * static_cast<size_t>(n) * nrhs;
    cudaStream_t st = c->stream;

    // bc = project_compatible(b) (reference numbering), then internal; staged:
    // stage_rhs already left the projected right-hand side in c->bproj
    if (!staged) {
        DG_CUDA(cudaMemcpyAsync(c->bproj, d_b, vb, cudaMemcpyDeviceToDevice, st));
        DG_TRY(project_compatible(c, nrhs, c->bproj));
    }
    Driver dr{c, nrhs, bp_of(nrhs), r};
    DG_TRY(dr.init());
    DG_TRY(dr.to_internal(c->bproj, bc));
    // x = 0, r = bc - A 0 = bc exactly
    DG_CUDA(cudaMemsetAsync(x, 0, vb, st));
    DG_CUDA(cudaMemcpyAsync(r, bc, vb, cudaMemcpyDeviceToDevice, st));
    const double* w = L0.area_i;

    auto wdot = [&](const double* a, const double* b, double* out) -> Status {
        DG_TRY(launch(c, kNorms, 24.0 * n * nrhs, [&] {
            DISPATCH_BP(dr.key, k_wdot<BP, RPT><<<dr.rows_grid(n), kBlock, 0, st>>>(n, nrhs, w, a, b, c->red));
        }));
        return dr.reduce_partials(dr.partial_blocks(n), out, 0, nullptr);
    };
    auto norm = [&](const double* v, double* out, int mode, const double* den) -> Status {
        DG_TRY(launch(c, kNorms, 8.0 * n * nrhs, [&] {
            DISPATCH_BP(dr.key, k_sumsq<BP, RPT><<<dr.rows_grid(n), kBlock, 0, st>>>(n, nrhs, v, c->red));
        }));
        return dr.reduce_partials(dr.partial_blocks(n), out, mode, den);
    };
    // y = A v (level-0 operator, reference entry order)
    auto apply = [&](const double* v, double* y) -> Status {
        const double bytes = 12.0 * L0.nnzL + 4.0 * (n + 1) + 16.0 * n * nrhs;
        if (L0.Le_ci && dr.tpr <= 8)
            return dr.pipe_w<OP_SPMV>(L0.Le_w, kFineResidual, bytes, n, L0.Le_ci, L0.Le_v, L0.Le_row, v, nullptr, y,
                                      nullptr, nullptr, 0.0, nullptr);
        return launch(c, kFineResidual, bytes, [&] {
            DISPATCH_BP(dr.key, (k_spmv<BP, RPT, 0><<<dr.rows_grid(n), kBlock, 0, st>>>(
                                    n, nrhs, L0.Lo_rp, L0.Lo_ci, L0.Lo_v, nullptr, v, y, nullptr)))
        });
    };
    // z = run_cycle(inner, r, 0).x: inner_cycles cycles from zero with b = r
    auto precondition = [&](const double** z) -> Status {
        dr.b0 = r;
        DG_TRY(dr.load_x0(nullptr));
        for (int k = 0; k < inner_cycles; ++k) DG_TRY(dr.one_cycle(inner));
        DG_TRY(dr.ensure_x(0));
        *z = L0.x[L0.cur];
        return Status::Ok();
    };
    auto fetch = [&](const double* dev, std::vector<double>& h) -> Status {
        DG_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, st));
        DG_CUDA(cudaStreamSynchronize(st));
        return Status::Ok();
    };

    DG_TRY(norm(bc, res, 1, nullptr));  // ||bc||
    DG_TRY(launch(c, kNorms, 0.0, [&] { k_denom<<<1, 32, 0, st>>>(nrhs, res, denom); }));
    const double* z = nullptr;
    DG_TRY(precondition(&z));
    DG_CUDA(cudaMemcpyAsync(p, z, vb, cudaMemcpyDeviceToDevice, st));
    DG_TRY(wdot(r, z, rz));
    DG_TRY(norm(r, res, 2, denom));
    std::vector<double> hres(nrhs), hres_g(34);
    double* guard = res + 32;  // [kind, iteration] of the first breakdown (pcg_s + 224)
    DG_CUDA(cudaMemsetAsync(guard, 0, sizeof(double) * 2, st));
    DG_TRY(fetch(res, hres));
    c->last_times.push_back(host_elapsed());  // weighted_cg records the initial residual's time too
    unsigned active = 0;
    for (int l = 0; l < nrhs; ++l) {
        if (h_hist) h_hist[l] = hres[l];
        iters[l] = 0;
        converged[l] = hres[l] <= tol;
        if (hres[l] > tol && maxiter > 0) active |= 1u << l;
    }
    const unsigned g = dr.rows_grid(n);
    int it = 0;
    while (active) {
        DG_TRY(apply(p, ap));
        DG_TRY(wdot(p, ap, curv));
        DG_TRY(launch(c, kNorms, 0.0, [&] { k_lane_div<<<1, 32, 0, st>>>(nrhs, rz, curv, alpha); }));
        // breakdown checks (solvers.cpp) on the device, read with this iteration's residuals
        DG_TRY(launch(c, kNorms, 0.0, [&] { k_pcg_guard<<<1, 32, 0, st>>>(nrhs, active, it, curv, alpha, guard); }));
        DG_TRY(launch(c, kNorms, 48.0 * n * nrhs, [&] {
            DISPATCH_BP(dr.key, k_cg_xr<BP, RPT><<<g, kBlock, 0, st>>>(n, nrhs, alpha, active, x, r, p, ap));
        }));
        DG_TRY(precondition(&z));
        DG_TRY(wdot(r, z, rzn));
        DG_TRY(launch(c, kNorms, 0.0, [&] { k_lane_div<<<1, 32, 0, st>>>(nrhs, rzn, rz, beta); }));
        DG_CUDA(cudaMemcpyAsync(rz, rzn, sizeof(double) * nrhs, cudaMemcpyDeviceToDevice, st));
        DG_TRY(launch(c, kNorms, 24.0 * n * nrhs, [&] {
            DISPATCH_BP(dr.key, k_cg_p<BP, RPT><<<g, kBlock, 0, st>>>(n, nrhs, beta, active, p, z));
        }));
        ++it;
        DG_TRY(norm(r, res, 2, denom));
        DG_CUDA(cudaMemcpyAsync(hres_g.data(), res, sizeof(double) * 34, cudaMemcpyDeviceToHost, st));
        DG_CUDA(cudaStreamSynchronize(st));
        if (hres_g[32] != 0.0)
            return Status::Err(DECMG_RUNTIME, std::string(hres_g[32] == 1.0 ? "cg: breakdown (zero curvature)"
                                                                           : "cg: breakdown (non-finite step)") +
                                                  " at iteration " + std::to_string(static_cast<int>(hres_g[33])));
        for (int l = 0; l < nrhs; ++l) hres[l] = hres_g[l];
        c->last_times.push_back(host_elapsed());
        for (int l = 0; l < nrhs; ++l) {
            if (!(active & (1u << l))) continue;
            if (h_hist) h_hist[static_cast<size_t>(it) * nrhs + l] = hres[l];
            iters[l] = it;
            converged[l] = hres[l] <= tol;
            if (hres[l] <= tol || it >= maxiter) active &= ~(1u << l);
        }
    }
    // final_relative_residual = relative_residual(A, x, bc) (solvers.cpp:20-27)
    if (h_final) {
        if (L0.Le_ci && dr.tpr <= 8) {
            DG_TRY(dr.pipe_w<OP_RES_STORE>(L0.Le_w, kNorms, 0.0, n, L0.Le_ci, L0.Le_v, L0.Le_row, x, bc, ap, nullptr,
                                            nullptr, 0.0, nullptr));
        } else {
            DG_TRY(launch(c, kNorms, 0.0, [&] {
                DISPATCH_BP(dr.key, (k_residual<BP, RPT, 0, true><<<dr.rows_grid(n), kBlock, 0, st>>>(
                                        n, nrhs, L0.Lo_rp, L0.Lo_ci, L0.Lo_v, nullptr, x, bc, ap, nullptr)))
            }));
        }
        DG_TRY(norm(ap, res, 2, denom));
        DG_TRY(fetch(res, hres));
        for (int l = 0; l < nrhs; ++l) h_final[l] = hres[l];
    }
    DG_TRY(dr.from_internal(x, d_x));
    DG_CUDA(cudaStreamSynchronize(st));
    return Status::Ok();
}

}  // namespace decmg_gpu
