// Two weighted-Jacobi sweeps in one persistent pass (jacobi_sweep twice,
// proj/src/multigrid.cpp:36-56), with the intermediate iterate handed from
// the first sweep to the second through L2 instead of a full HBM round trip.
//
// Two separate sweeps move x, b, x' (write) + L, then x', b, x'' (write) + L
// again: 9.9 GB per pair at config 4. Here each CTA walks its tiles (56-row
// ELL tiles of the Morton-ordered level, ch consecutive tiles per step,
// chunks dealt round-robin to the CTAs) as a wavefront: at step i it runs
// sweep 1 on its chunk i and sweep 2 on its chunk i - lag. All CTAs advance
// together, so the x' rows a sweep-2 tile gathers were written a few steps
// earlier and are still in L2, as are its b rows and its ELL tile; HBM sees
// x, b and L once, x' and x'' written once (6.3 GB). Sweep 2 overwrites x
// with x'' in place.
//
// Correctness (bit-identical to two separate sweeps): every row's arithmetic
// is the sweep kernel's (same ELL entry order, same division). Sweep 2 of
// tile t may start only when sweep 1 has finished on every tile holding a
// neighbour of t's rows (and on t): then all x' it gathers are final, and no
// later sweep-1 gather reads the x rows it overwrites (the neighbour relation
// of L is symmetric, padding entries point at the row itself). Each consumer
// warp publishes its part of a sweep-1 tile with fence + atomic increment of
// the tile's counter; the producer warp waits (acquire loads) for the
// counters of a tile's dependencies before issuing its sweep-2 work, and
// sweep-2 gathers bypass L1 (ld.global.cg). A tile with a dependency further
// ahead than the current step is deferred to the end of the CTA's schedule
// (a wait on a later step could deadlock); waits only ever target tiles of
// the current step or earlier, which every co-resident CTA reaches without
// waiting on anyone, and the launch is cooperative so all CTAs are resident.
//
// Measured (B200, config 4, 16 RHS): bit-identical, DRAM
// traffic per level-0 pair 6.9 GB (from 9.9 GB), but 2.44 ms against 1.72 ms
// for two k_rowop_pipe sweeps: dealing tiles round-robin costs the L1 reuse
// of the contiguous per-CTA ranges (L1 hit 28 % vs 74 %), sweep 2's gathers
// wait on L2, and publishing each tile costs a release fence per warp (2.03
// ms with the synchronisation removed). Contiguous ranges would keep L1, but
// 86 % of 56-row tiles have a neighbour 4 or more tiles ahead (Morton jumps),
// so tile-granular dependencies defer almost everything. Opt-in: DECMG_PAIR=1.
#include "driver.cuh"

namespace decmg_gpu {

constexpr int kPairDeps = 15;  // dependency tiles kept per tile (slot 15: count, -1 = more)
constexpr int kPairDepStride = kPairDeps + 1;
constexpr int kPairWarps = kPipeConsumers / 32;  // counter increments per sweep-1 tile

namespace {

// Distinct neighbour tiles of every tile (excluding itself), ascending.
// One warp per tile.
__global__ void k_pair_deps(int ntiles, int rows_per_tile, int W, const int* __restrict__ eci,
                            const int* __restrict__ erow, int* __restrict__ deps) {
    const int t = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= ntiles) return;
    const int n = rows_per_tile * W;
    const int64_t base = static_cast<int64_t>(t) * rows_per_tile;
    int last = -1, cnt = 0;
    int* out = deps + static_cast<int64_t>(t) * kPairDepStride;
    for (;;) {
        int best = 0x7fffffff;
        for (int i = lane; i < n; i += 32) {
            const int r = i / W;
            if (erow[base + r] < 0) continue;  // padding row
            const int u = eci[(base + r) * W + (i - r * W)] / rows_per_tile;
            if (u != t && u > last && u < best) best = u;
        }
        for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (best == 0x7fffffff) break;
        if (cnt == kPairDeps) {
            cnt = -1;
            break;
        }
        if (lane == 0) out[cnt] = best;
        ++cnt;
        last = best;
    }
    if (lane == 0) out[kPairDeps] = cnt;
}

struct PairArgs {
    int ntiles, nrhs;
    const int* eci;
    const double* ev;
    const int* ord;
    double* x;         // in: x; out: x'' (tile by tile)
    double* xp;        // x'
    const double* b;
    double* partial;   // NORM: per-CTA partials of ||b - A x||^2
    double omega;
    int n, pf, ch, lag;
    const int* deps;
    unsigned* flags;             // per tile: sweep-1 completions (kPairWarps per launch)
    unsigned long long* done;    // sweep-1 tiles completed (all launches)
    unsigned target;             // epoch * kPairWarps
    unsigned long long done_target;  // epoch * ntiles
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <int RPT>
__device__ __forceinline__ void ldv_cg(const double* __restrict__ p, double (&o)[RPT]) {
    if constexpr (RPT == 4) {
        asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
                     : "l"(p));
    } else if constexpr (RPT == 1) {
        o[0] = __ldcg(p);
    } else {
#pragma unroll
        for (int j = 0; j < RPT / 2; ++j) {
            const double2 t = __ldcg(reinterpret_cast<const double2*>(p + 2 * j));
            o[2 * j] = t.x;
            o[2 * j + 1] = t.y;
        }
    }
}

// L2 eviction-priority hints: the sweep-1 outputs and b stay (evict_last)
// until sweep 2 of the neighbourhood has read them.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
template <int RPT>
__device__ __forceinline__ void ldv_hint(const double* __restrict__ p, double (&o)[RPT], uint64_t pol) {
    if constexpr (RPT == 4) {
        asm volatile("ld.global.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                     : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
                     : "l"(p), "l"(pol));
    } else {
        ldv<RPT>(p, o);
    }
}
template <int RPT>
__device__ __forceinline__ void stv_hint(double* __restrict__ p, const double (&o)[RPT], uint64_t pol) {
    if constexpr (RPT == 4) {
        asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(o[0]), "d"(o[1]),
                     "d"(o[2]), "d"(o[3]), "l"(pol)
                     : "memory");
    } else {
        stv<RPT>(p, o);
    }
}

// spin bound: ~seconds; a dependency that never completes traps instead of hanging the GPU
constexpr long long kPairSpin = 1ll << 24;

template <int BP, int RPT, int W, bool NORM>
__global__ void __launch_bounds__(kPipeThreads, kPipeCtasPerSm) k_rowop_pair(PairArgs a) {
    using G = PipeGeom<BP, RPT, W>;
    constexpr int TPR = G::TPR;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kPipeStages], empty[kPipeStages];
    __shared__ int item[kPipeStages];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < kPipeStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kPipeConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int Gn = gridDim.x, cta = blockIdx.x;
    const int ch = a.ch, lag = a.lag;
    const int nst = (a.ntiles + ch - 1) / ch;
    const int nsteps = nst > cta ? (nst - cta + Gn - 1) / Gn : 0;
    double acc[RPT];
#pragma unroll
    for (int l = 0; l < RPT; ++l) acc[l] = 0.0;

    if (tid >= kPipeConsumers) {
        // producer warp: schedule, dependency waits (all lanes), TMA issue (lane 0)
        const int lane = tid - kPipeConsumers;
        int it = 0;
        auto step_of = [&](int u) { return (u / ch) / Gn; };
        auto regular = [&](int t, int i) -> bool {
            const int* d = a.deps + static_cast<int64_t>(t) * kPairDepStride;
            const int nd = d[kPairDeps];
            if (nd < 0) return false;
            bool ok = true;
            for (int k = 0; k < nd; ++k) ok &= step_of(d[k]) <= i;
            return ok;
        };
        auto wait_deps = [&](int t) {
            const int* d = a.deps + static_cast<int64_t>(t) * kPairDepStride;
            const int nd = d[kPairDeps];
            long long spins = 0;
            if (nd < 0) {
                while (ld_acquire64(a.done) < a.done_target)
                    if (++spins > kPairSpin) __trap();
                return;
            }
            // lane k waits for dependency k; lane nd for the tile itself
            const int u = lane < nd ? d[lane] : (lane == nd ? t : -1);
            if (u >= 0)
                while (ld_acquire(a.flags + u) < a.target)
                    if (++spins > kPairSpin) {
                        printf("pair: CTA %d waits for tile %d (for tile %d): counter %u, target %u\n", blockIdx.x, u,
                               t, ld_acquire(a.flags + u), a.target);
                        __trap();
                    }
            __syncwarp();
        };
        auto push = [&](int t, int phase) {
            const int s = it % kPipeStages;
            if (phase == 2) wait_deps(t);
            if (lane == 0) {
                if (it >= kPipeStages) mbar_wait(&empty[s], ((it / kPipeStages) - 1) & 1);
                item[s] = t < 0 ? -1 : (t | (phase == 2 ? 1 << 30 : 0));  // bit 30: sweep 2
                if (t < 0) {
                    mbar_arrive(&full[s]);
                } else {
                    unsigned char* st = smem_raw + static_cast<size_t>(s) * G::STAGE_BYTES;
                    mbar_expect_tx(&full[s], G::STAGE_BYTES);
                    tma_bulk_g2s(st, a.ev + static_cast<int64_t>(t) * G::ROWS * W, G::V_BYTES, &full[s]);
                    tma_bulk_g2s(st + G::V_BYTES, a.eci + static_cast<int64_t>(t) * G::ROWS * W, G::CI_BYTES,
                                 &full[s]);
                    tma_bulk_g2s(st + G::V_BYTES + G::CI_BYTES, a.ord + static_cast<int64_t>(t) * G::ROWS,
                                 G::ORD_BYTES, &full[s]);
                }
            }
            __syncwarp();
            ++it;
        };
        for (int i = 0; i < nsteps + lag; ++i) {
            if (i < nsteps) {
                const int s0 = (i * Gn + cta) * ch;
                for (int t = s0; t < s0 + ch && t < a.ntiles; ++t) push(t, 1);
            }
            if (i >= lag) {
                const int s0 = ((i - lag) * Gn + cta) * ch;
                for (int t = s0; t < s0 + ch && t < a.ntiles; ++t)
                    if (regular(t, i)) push(t, 2);
            }
        }
        for (int j = 0; j < nsteps; ++j) {  // deferred sweep-2 tiles
            const int s0 = (j * Gn + cta) * ch;
            for (int t = s0; t < s0 + ch && t < a.ntiles; ++t)
                if (!regular(t, j + lag)) push(t, 2);
        }
        push(-1, 0);
    } else {
        const int q = tid / TPR;
        const int lane0 = (tid % TPR) * RPT;
        const int nrhs = a.nrhs;
        const uint64_t keep = policy_evict_last();
        for (int i = 0;; ++i) {
            const int s = i % kPipeStages;
            mbar_wait(&full[s], (i / kPipeStages) & 1);
            const int itm = item[s];
            if (itm < 0) break;
            const int t = itm & ((1 << 30) - 1);
            const bool second = (itm >> 30) & 1;
            const unsigned char* st = smem_raw + static_cast<size_t>(s) * G::STAGE_BYTES;
            const double* vs = reinterpret_cast<const double*>(st);
            const int* cs = reinterpret_cast<const int*>(st + G::V_BYTES);
            const int* os = reinterpret_cast<const int*>(st + G::V_BYTES + G::CI_BYTES);
            const int* cq = cs + q * W;
            const double* vq = vs + q * W;
            const int e = os[q];
            const bool active = e >= 0 && lane0 < nrhs;
            const int64_t row = erow_id(e);
            const int64_t o = row * nrhs + lane0;
            double pre[RPT], xv[W][RPT], sum[RPT], xr[RPT], d = 0.0;
            if (active) {
                if (!second) ldv_hint<RPT>(a.b + o, pre, keep);  // sweep 1 leaves b in L2 for sweep 2
                else ldv<RPT>(a.b + o, pre);
                if (!second) {
                    if (a.pf && row + a.pf < a.n) {
                        const int64_t po = (row + a.pf) * nrhs + lane0;
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.x + po));
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.b + po));
                    }
#pragma unroll
                    for (int j = 0; j < W; ++j) ldv<RPT>(a.x + static_cast<int64_t>(cq[j]) * nrhs + lane0, xv[j]);
                } else if (BP * 8 >= 128) {
                    // one row per 128-byte line: a line this SM caches holds only a finished x' row
                    // (L1 starts each launch empty), so sweep 2 may use L1
#pragma unroll
                    for (int j = 0; j < W; ++j) ldv<RPT>(a.xp + static_cast<int64_t>(cq[j]) * nrhs + lane0, xv[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < W; ++j) ldv_cg<RPT>(a.xp + static_cast<int64_t>(cq[j]) * nrhs + lane0, xv[j]);
                }
#pragma unroll
                for (int l = 0; l < RPT; ++l) sum[l] = 0.0;
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    const double vj = vq[j];
#pragma unroll
                    for (int l = 0; l < RPT; ++l) sum[l] = __dadd_rn(sum[l], __dmul_rn(vj, xv[j][l]));
                }
                d = vq[erow_slot(e)];
                if (!second) ldv<RPT>(a.x + o, xr);
                else if (BP * 8 >= 128) ldv<RPT>(a.xp + o, xr);
                else ldv_cg<RPT>(a.xp + o, xr);
            }
            const double y = active ? div_seed(d) : 0.0;  // consumes the stage's d before the release
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty[s]);  // stage consumed
            if (active) {
                double res[RPT];
#pragma unroll
                for (int l = 0; l < RPT; ++l) {
                    if constexpr (NORM) {
                        if (!second) {
                            const double rl = __dsub_rn(pre[l], sum[l]);
                            acc[l] = __dadd_rn(acc[l], __dmul_rn(rl, rl));
                        }
                    }
                    res[l] = __dadd_rn(xr[l], div_rn(__dmul_rn(a.omega, __dsub_rn(pre[l], sum[l])), d, y));
                }
                if (!second) stv_hint<RPT>(a.xp + o, res, keep);  // stays in L2 for sweep 2
                else stv_cs<RPT>(a.x + o, res);
            }
            if (!second) {  // publish this warp's part of sweep-1 tile t (release, cumulative over the warp)
                __syncwarp();
                if ((tid & 31) == 0) {
                    unsigned old;
                    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.flags + t) : "memory");
                    if (old + 1 == a.target) atomicAdd(a.done, 1ull);
                }
            }
        }
    }
    if constexpr (NORM) {
        // the consumers' accumulators folded as in k_rowop_pipe (fixed tree)
        constexpr int ROWS = G::ROWS;
        constexpr int RP2 = ROWS <= 1 ? 1 : (ROWS <= 2 ? 2 : (ROWS <= 4 ? 4 : (ROWS <= 8 ? 8 : (ROWS <= 16 ? 16 :
                            (ROWS <= 32 ? 32 : (ROWS <= 64 ? 64 : (ROWS <= 128 ? 128 : 256)))))));
        __shared__ double sh[RP2 * BP];
        for (int idx = kPipeConsumers * RPT + tid; idx < RP2 * BP; idx += kPipeThreads) sh[idx] = 0.0;
        if (tid < kPipeConsumers)
#pragma unroll
            for (int l = 0; l < RPT; ++l) sh[tid * RPT + l] = acc[l];
        __syncthreads();
        for (int sft = RP2 / 2; sft >= 1; sft >>= 1) {
            for (int idx = tid; idx < sft * BP; idx += kPipeThreads) sh[idx] = __dadd_rn(sh[idx], sh[idx + sft * BP]);
            __syncthreads();
        }
        for (int idx = tid; idx < BP; idx += kPipeThreads)
            a.partial[static_cast<int64_t>(blockIdx.x) * BP + idx] = sh[idx];
    }
}

template <int BP, int RPT, int W, bool NORM>
Status launch_pair(decmg_gpu_ctx* c, const PairArgs& a0, int* grid_out) {
    using G = PipeGeom<BP, RPT, W>;
    auto kern = k_rowop_pair<BP, RPT, W, NORM>;
    static int per_sm = -1;
    if (per_sm < 0) {
        DG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(G::SMEM)));
        int nb = 0;
        DG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kPipeThreads, G::SMEM));
        per_sm = nb < kPipeCtasPerSm ? nb : kPipeCtasPerSm;
        if (per_sm < 1) return Status::Err(DECMG_CUDA, "pair sweep: kernel does not fit on an SM");
    }
    PairArgs a = a0;
    const int nst = (a.ntiles + a.ch - 1) / a.ch;
    int g = per_sm * c->num_sms;
    if (g > nst) g = nst;
    if (grid_out) *grid_out = g;
    void* args[] = {&a};
    // cooperative: all CTAs co-resident (the dependency waits assume it)
    return cuda_status(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(g), dim3(kPipeThreads),
                                                   args, G::SMEM, c->stream),
                       "pair sweep launch");
}

}  // namespace

// Two Jacobi sweeps on level k: x (L.x[L.cur]) -> x'' in place, x' in
// L.x[L.cur ^ 1]. partial != nullptr: also the per-CTA norm partials of
// b - A x for the incoming x (the fused cycle residual; *grid = partial rows).
Status pair_sweeps(decmg_gpu_ctx* c, int k, int key, int nrhs, double omega, const double* b, double* partial,
                   int* grid, double bytes, int cls) {
    Level& L = c->lv[k];
    Status st;
    DISPATCH_BP(key, {
        using G7 = PipeGeom<BP, RPT, 7>;
        constexpr int ROWS = G7::ROWS;
        const int ntiles = (L.nv + ROWS - 1) / ROWS;
        if (!L.pr_deps || L.pr_rows != ROWS) {  // (re)built when the tile size changes with nrhs
            DG_TRY(dalloc(c, &L.pr_deps, static_cast<size_t>(ntiles) * kPairDepStride));
            DG_TRY(dalloc(c, &L.pr_flags, static_cast<size_t>(ntiles)));
            DG_TRY(dalloc(c, &L.pr_done, 1));
            DG_CUDA(cudaMemsetAsync(L.pr_flags, 0, sizeof(unsigned) * ntiles, c->stream));
            DG_CUDA(cudaMemsetAsync(L.pr_done, 0, sizeof(unsigned long long), c->stream));
            L.pr_epoch = 0;
            L.pr_rows = ROWS;
            const int64_t threads = static_cast<int64_t>(ntiles) * 32;
            DG_TRY(launch(c, kNorms, 0.0, [&] {
                k_pair_deps<<<grid_for(threads, 256), 256, 0, c->stream>>>(ntiles, ROWS, L.Le_w, L.Le_ci, L.Le_row,
                                                                        L.pr_deps);
            }));
        }
        ++L.pr_epoch;
        PairArgs a{};
        a.ntiles = ntiles;
        a.nrhs = nrhs;
        a.eci = L.Le_ci;
        a.ev = L.Le_v;
        a.ord = L.Le_row;
        a.x = L.x[L.cur];
        a.xp = L.x[L.cur ^ 1];
        a.b = b;
        a.partial = partial;
        a.omega = omega;
        a.n = L.nv;
        a.pf = c->pf;
        a.ch = c->pair_ch;
        a.lag = c->pair_lag;
        a.deps = L.pr_deps;
        a.flags = L.pr_flags;
        a.done = L.pr_done;
        a.target = L.pr_epoch * static_cast<unsigned>(kPairWarps);
        a.done_target = static_cast<unsigned long long>(L.pr_epoch) * static_cast<unsigned long long>(ntiles);
        Status s2;
        st = launch(c, cls, bytes, [&] {
            if (L.Le_w == 7)
                s2 = partial ? launch_pair<BP, RPT, 7, true>(c, a, grid) : launch_pair<BP, RPT, 7, false>(c, a, grid);
            else
                s2 = partial ? launch_pair<BP, RPT, 8, true>(c, a, grid) : launch_pair<BP, RPT, 8, false>(c, a, grid);
        });
        if (!s2.ok()) return s2;
    })
    return st;
}

}  // namespace decmg_gpu
