// Vertex-partitioned multi-GPU V-cycle.
//
// Every rank builds the full hierarchy (deterministic, bit-identical on all
// ranks), then takes a partition of the finer levels:
//  * ownership: level-0 vertices are split into N contiguous ranges of the
//    level's internal (Morton) row order; a coarse vertex is the fine vertex
//    with the same id (subdivision keeps coarse ids first, subdivision.cpp:
//    30-40), so it has the same owner on every level and restriction and
//    prolongation stay almost entirely rank-local;
//  * levels 0 .. ka-1 are distributed: rank p owns the vertices of its range
//    and keeps a 1-ring halo (every vertex its owned rows of L_k, its owned
//    coarse rows of R_k and its owned fine rows of P_{k-1} reference); local
//    vectors are [owned (internal order) | halo (grouped by owner rank, then
//    global id)], so the halo values a peer sends land in one contiguous slice;
//  * levels ka .. L-1 (fewer than `agglomerate` vertices per rank) run
//    replicated on every rank after the restricted right-hand side of level ka
//    is all-gathered (the coarsest solve included: "coarsest levels
//    agglomerated").
// Every row's arithmetic is the single-GPU one (same entries, same order), so
// iterates are bit-identical to the 1-GPU solve for any rank count. The owned
// rows of each operator are split into interior rows (every column owned) and
// boundary rows: the interior pass runs while the halo is in flight, the
// boundary pass after it lands. Norms are per-rank partial sums, all-gathered
// and added in rank order on the device (deterministic for a rank count; a few
// ulps from the single-GPU tree).
//
// Transports (one exchange schedule, three ways to move the bytes):
//  * NCCL: one process per GPU, grouped ncclSend/ncclRecv on a communication
//    stream (the interior pass overlaps it), ncclAllGather for the norms;
//    capturable, so cycles run as CUDA graphs;
//  * emulation: all ranks of a world in one process on one device and stream,
//    device copies in place of NCCL (no kernel ever waits on another rank's
//    kernel, so it is safe on one GPU); also captured as graphs;
//  * host staging ("shm"): one process per rank, any devices (several ranks may
//    share one GPU): packed halos go device -> shared host mapping -> device,
//    with a host barrier between the write and the reads. No kernel waits on
//    another process -- the host synchronises its own stream before the
//    barrier -- so it is the multi-process test of the per-process setup on a
//    single GPU. Not capturable (host synchronisation per exchange).
#include "driver.cuh"

#include <nccl.h>

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <numeric>

namespace decmg_gpu {
namespace {

// buf[t] = v[idx[i]] (rows of nrhs values)
__global__ void k_pack(int n, int nrhs, const int* __restrict__ idx, const double* __restrict__ v,
                       double* __restrict__ buf) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * nrhs) return;
    const int64_t i = t / nrhs;
    const int l = static_cast<int>(t % nrhs);
    buf[t] = v[static_cast<int64_t>(idx[i]) * nrhs + l];
}

// v[idx[i]] = buf[t]
__global__ void k_unpack(int n, int nrhs, const int* __restrict__ idx, const double* __restrict__ buf,
                         double* __restrict__ v) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * nrhs) return;
    const int64_t i = t / nrhs;
    const int l = static_cast<int>(t % nrhs);
    v[static_cast<int64_t>(idx[i]) * nrhs + l] = buf[t];
}

// Per-lane residual norms from the all-gathered per-rank sums [N][nrhs]:
// out[l] = sqrt(sum_p all[p][l]) / denom[l], ranks added in order.
__global__ void k_rank_fold(int N, int nrhs, const double* __restrict__ all, const double* __restrict__ denom,
                            double* __restrict__ out) {
    const int l = threadIdx.x;
    if (l >= nrhs) return;
    double t = 0.0;
    for (int p = 0; p < N; ++p) t = __dadd_rn(t, all[static_cast<int64_t>(p) * nrhs + l]);
    out[l] = __ddiv_rn(__dsqrt_rn(t), denom[l]);
}

// hist[(*cnt) * nrhs + l] = res[l]; ++*cnt (run_cycle's history inside a
// replayed graph: the slot comes from a device counter)
__global__ void k_hist_put(int nrhs, const double* __restrict__ res, double* __restrict__ hist, int* cnt) {
    const int l = threadIdx.x;
    const int c = *cnt;
    if (l < nrhs) hist[static_cast<int64_t>(c) * nrhs + l] = res[l];
    __syncwarp();
    if (l == 0) *cnt = c + 1;
}

// gmg_solve's convergence check of the iterate after st->cyc cycles (the
// partitioned variant of k_solve_check, without graph conditionals): finished
// lanes are recorded and flagged for the snapshot kernel; the outcome is
// published to the host through mapped pinned memory as {cycle, all done}.
struct DistSolveState {
    int cyc;
    unsigned active;
    unsigned fin;
    int max_cycles;
    double tol;
    int done[32];
    double final_res[32];
};

__global__ void k_dist_check(int nrhs, const double* __restrict__ res, DistSolveState* st, double* __restrict__ hist,
                             volatile int* hflag) {
    const int l = threadIdx.x;
    const int cyc = st->cyc;
    const unsigned active = st->active;
    bool fin = false;
    if (l < nrhs && ((active >> l) & 1u)) {
        const double r = res[l];
        if (cyc >= 1) hist[static_cast<int64_t>(cyc - 1) * nrhs + l] = r;
        st->final_res[l] = r;
        st->done[l] = cyc;
        // NaN/Inf residual: finishes the lane (the host reports DECMG_RUNTIME)
        fin = r <= st->tol || cyc >= st->max_cycles || !isfinite(r);
    }
    const unsigned finmask = __ballot_sync(0xffffffffu, fin);
    if (l == 0) {
        const unsigned left = active & ~finmask;
        st->fin = finmask;
        st->active = left;
        st->cyc = cyc + 1;
        __threadfence_system();
        hflag[1] = left ? 0 : 1;
        __threadfence_system();
        hflag[0] = cyc;
    }
}

__global__ void k_dist_copy_lanes(int64_t total, int nrhs, const DistSolveState* __restrict__ st,
                                  const double* __restrict__ src, double* __restrict__ dst) {
    const unsigned mask = st->fin;
    if (!mask) return;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int lane = static_cast<int>(t % nrhs);
    if (mask & (1u << lane)) dst[t] = src[t];
}

__global__ void k_dist_state_init(DistSolveState* st, int cyc, unsigned active, int max_cycles, double tol) {
    st->cyc = cyc;
    st->active = active;
    st->fin = 0;
    st->max_cycles = max_cycles;
    st->tol = tol;
}

// One exchange plan: what this rank sends (owned rows, packed per peer) and
// receives. Halo plans receive straight into the vector's halo slice of each
// peer; all-gather plans receive into rbuf and scatter through ridx.
struct Xch {
    std::vector<int> peer;        // peer ranks with traffic either way, ascending
    std::vector<int> soff, scnt;  // rows sent to peer j: sbuf rows [soff, soff + scnt)
    std::vector<int> roff, rcnt;  // rows received from peer j: slots [roff, roff + rcnt)
    std::vector<int64_t> rsrc;    // host staging: row offset of this rank's slice in peer j's packed buffer
    int nsend = 0, nrecv = 0;
    int* sidx = nullptr;          // [nsend] local rows to pack
    double* sbuf = nullptr;       // [nsend][max_nrhs]
    bool gather = false;          // all-gather: receive into rbuf, scatter by ridx
    int* ridx = nullptr;          // [nrecv]
    double* rbuf = nullptr;       // [nrecv][max_nrhs]
    int recv_base = 0;            // halo plans: local row of the first halo slot (= nown)
};

// An ELL row set (interior or boundary rows of one operator).
struct Ell {
    int rows = 0;  // real rows (the arrays are padded to a multiple of 224 rows)
    int* ci = nullptr;
    double* v = nullptr;
    int* row = nullptr;  // local row id | diagonal slot << kRowBits, -1 padding
};

struct DLevel {
    int k = 0;
    int nown = 0, nloc = 0;
    int* d_own = nullptr;  // global vertex ids of the owned rows (local 0..nown-1)
    int Lw = 0, Rw = 0;
    Ell Li, Lb;            // L_k rows: interior / boundary
    Ell Ri, Rb;            // R_k rows (owned vertices of level k+1)
    Ell Pi, Pb;            // P_k rows (owned fine rows), ELL-2
    double* diag = nullptr;  // [nown]
    int* bd = nullptr;       // [nown] Dirichlet flags of the owned rows (extension x1)
    int zero_diag_row = -1;
    Xch hx;                // halo plan of level k (x and r)
    double* x[2] = {nullptr, nullptr};
    double* b = nullptr;
    double* r = nullptr;
    int cur = 0;
    bool x_zero = false;
};

struct DRank {
    int rank = 0;
    std::vector<DLevel> lv;  // distributed levels 0 .. ka-1
    Xch bx;                  // all-gather of the restricted right-hand side of level ka
    Xch sx;                  // all-gather of the level-0 solution (reference numbering)
    double* red = nullptr;   // norm partials (two halves for the fold ping-pong)
    size_t red_cap = 0;
    double* dsum = nullptr;  // this rank's per-lane partial sum [32]
    double* xsol = nullptr;  // solve snapshot of the owned level-0 rows [nown][max_nrhs]
};

// Host-staged transport: a shared file mapping [header | 2 parities x N ranks x slot].
struct ShmHeader {
    std::atomic<int> count;
    std::atomic<int> gen;
    std::atomic<int> abort;
};

}  // namespace
}  // namespace decmg_gpu

struct decmg_gpu_dist {
    int world = 1, ka = 0, L = 0, max_nrhs = 1;
    int kind = DECMG_DIST_EMULATE;
    ncclComm_t comm = nullptr;
    std::vector<decmg_gpu::DRank> ranks;  // local ranks (emulation: all; otherwise one)
    std::unique_ptr<decmg_gpu_ctx, void (*)(decmg_gpu_ctx*)> g{nullptr, nullptr};
    std::string err;
    std::vector<void*> allocs;
    cudaStream_t comm_stream = nullptr;     // NCCL transfers (overlap the interior passes)
    cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
    double* all = nullptr;                  // all-gathered per-rank sums [N][32]
    double* res = nullptr;                  // per-lane relative residuals [32] (device)
    double* hist = nullptr;                 // device history [hist_cap][32]
    int hist_cap = 0;
    int* hcnt = nullptr;                    // device history counter (run_cycle graphs)
    decmg_gpu::DistSolveState* st = nullptr;
    int* hflag = nullptr;                   // mapped pinned {cycle, all done}
    int* hflag_dev = nullptr;
    float last_cycle_ms = 0.f;              // device time of the last run's cycle loop
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // graphs of one cycle body, by key
    struct GraphEntry {
        std::string key;
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        std::vector<std::pair<int, bool>> post;  // host ping-pong state after one body
        int64_t kernels = 0;                     // launches recorded into one replay
    };
    std::vector<GraphEntry> graphs;
    // host staging
    int shm_fd = -1;
    size_t shm_bytes = 0, shm_slot = 0;
    unsigned char* shm = nullptr;
    int shm_parity = 0;
    double* shm_stage = nullptr;            // pinned staging of this rank's packed rows
};

namespace decmg_gpu {
namespace {

thread_local std::string g_dist_create_error;

template <class T>
Status dmalloc(decmg_gpu_dist* D, T** p, size_t n) {
    void* q = nullptr;
    DG_CUDA(cudaMalloc(&q, (n ? n : 1) * sizeof(T)));
    D->allocs.push_back(q);
    *p = static_cast<T*>(q);
    return Status::Ok();
}
template <class T>
Status upload(decmg_gpu_dist* D, T** p, const std::vector<T>& h) {
    DG_TRY(dmalloc(D, p, h.size()));
    if (!h.empty()) DG_CUDA(cudaMemcpy(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return Status::Ok();
}
template <class T>
Status download(const T* d, size_t n, std::vector<T>* h) {
    h->resize(n);
    if (n) DG_CUDA(cudaMemcpy(h->data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
    return Status::Ok();
}

inline int ncclcheck(ncclResult_t r, std::string* msg) {
    if (r == ncclSuccess) return 0;
    *msg = std::string("NCCL: ") + ncclGetErrorString(r);
    return 1;
}
#define DG_NCCL(call)                                                              \
    do {                                                                           \
        std::string _m;                                                            \
        if (ncclcheck((call), &_m)) return Status::Err(DECMG_NCCL, _m);            \
    } while (0)

// ---------------------------------------------------------- host staging ----
Status shm_open_map(decmg_gpu_dist* D, const char* path, size_t slot) {
    D->shm_slot = (slot + 255) / 256 * 256;
    D->shm_bytes = 4096 + 2 * static_cast<size_t>(D->world) * D->shm_slot;
    D->shm_fd = ::open(path, O_RDWR | O_CREAT, 0600);
    if (D->shm_fd < 0) return Status::Err(DECMG_INVALID_ARGUMENT, std::string("dist shm: cannot open ") + path);
    // every rank extends the file to the same size (idempotent); a fresh file is zero-filled
    struct stat sb;
    if (::fstat(D->shm_fd, &sb) != 0) return Status::Err(DECMG_RUNTIME, "dist shm: fstat failed");
    if (static_cast<size_t>(sb.st_size) < D->shm_bytes && ::ftruncate(D->shm_fd, D->shm_bytes) != 0)
        return Status::Err(DECMG_RUNTIME, "dist shm: ftruncate failed");
    void* p = ::mmap(nullptr, D->shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, D->shm_fd, 0);
    if (p == MAP_FAILED) return Status::Err(DECMG_RUNTIME, "dist shm: mmap failed");
    D->shm = static_cast<unsigned char*>(p);
    DG_CUDA(cudaMallocHost(&D->shm_stage, D->shm_slot));
    return Status::Ok();
}

ShmHeader* shm_hdr(decmg_gpu_dist* D) { return reinterpret_cast<ShmHeader*>(D->shm); }
double* shm_region(decmg_gpu_dist* D, int parity, int rank) {
    return reinterpret_cast<double*>(D->shm + 4096 + (static_cast<size_t>(parity) * D->world + rank) * D->shm_slot);
}

// Sense-reversing barrier of the world's processes on the shared mapping.
Status shm_barrier(decmg_gpu_dist* D) {
    ShmHeader* h = shm_hdr(D);
    const int gen = h->gen.load(std::memory_order_acquire);
    if (h->count.fetch_add(1, std::memory_order_acq_rel) == D->world - 1) {
        h->count.store(0, std::memory_order_relaxed);
        h->gen.fetch_add(1, std::memory_order_release);
        return Status::Ok();
    }
    const auto t0 = std::chrono::steady_clock::now();
    while (h->gen.load(std::memory_order_acquire) == gen) {
        if (h->abort.load(std::memory_order_relaxed))
            return Status::Err(DECMG_RUNTIME, "dist shm: a peer process aborted");
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300))
            return Status::Err(DECMG_RUNTIME, "dist shm: barrier timed out (a peer process is gone)");
        sched_yield();
    }
    return Status::Ok();
}

// ---------------------------------------------------------------- setup ----
struct HostCSR {
    std::vector<int> rp, ci;
    std::vector<double> v;
};

Status fetch_csr(const int* rp, const int* ci, const double* v, int nrows, int64_t nnz, HostCSR* h) {
    DG_TRY(download(rp, static_cast<size_t>(nrows) + 1, &h->rp));
    DG_TRY(download(ci, static_cast<size_t>(nnz), &h->ci));
    DG_TRY(download(v, static_cast<size_t>(nnz), &h->v));
    return Status::Ok();
}

// ELL of the given rows (global row ids, in order) with columns mapped by
// colmap. Same layout as setup.cu k_ell_fill: padding entries are a real
// column with value 0.0 (the row's diagonal column for L, diag = true; its
// first column otherwise) and the row id carries the diagonal slot above
// kRowBits.
Status build_local_ell(decmg_gpu_dist* D, const HostCSR& A, const std::vector<int>& rows,
                       const std::vector<int>& rowid, const std::vector<int>& colmap, int W, bool diag, Ell* out) {
    const size_t npad = (rows.size() + 223) / 224 * 224;
    std::vector<int> ci(npad * W, 0), rid(npad, -1);
    std::vector<double> v(npad * W, 0.0);
    for (size_t q = 0; q < rows.size(); ++q) {
        const int g = rows[q];
        const int k0 = A.rp[g], len = A.rp[g + 1] - k0;
        if (len > W) return Status::Err(DECMG_RUNTIME, "dist: row longer than the ELL width");
        if (rowid[q] >= (1 << kRowBits)) return Status::Err(DECMG_RUNTIME, "dist: row id beyond the ELL row-id bits");
        int slot = 0, padc = -1;
        for (int j = 0; j < len; ++j) {
            const int lc = colmap[A.ci[k0 + j]];
            if (lc < 0) return Status::Err(DECMG_RUNTIME, "dist: column outside owned + halo");
            ci[q * W + j] = lc;
            v[q * W + j] = A.v[k0 + j];
            if (A.ci[k0 + j] == g) {
                slot = j;
                if (diag) padc = lc;
            }
            if (!diag && j == 0) padc = lc;
        }
        if (padc < 0 && len > 0) padc = ci[q * W];
        for (int j = len; j < W; ++j) ci[q * W + j] = padc < 0 ? 0 : padc;
        rid[q] = rowid[q] | (diag ? slot << kRowBits : 0);
    }
    out->rows = static_cast<int>(rows.size());
    DG_TRY(upload(D, &out->ci, ci));
    DG_TRY(upload(D, &out->v, v));
    DG_TRY(upload(D, &out->row, rid));
    return Status::Ok();
}

int maxlen(const HostCSR& A) {
    int m = 0;
    for (size_t i = 0; i + 1 < A.rp.size(); ++i) m = std::max(m, A.rp[i + 1] - A.rp[i]);
    return m;
}

// Split `rows` (with their local ids) into interior rows (every column
// satisfies own(col)) and boundary rows, keeping the order, and build both ELLs.
template <class Own>
Status build_split_ell(decmg_gpu_dist* D, const HostCSR& A, const std::vector<int>& rows,
                       const std::vector<int>& rowid, const std::vector<int>& colmap, int W, bool diag, Own own,
                       Ell* in, Ell* bd) {
    std::vector<int> ri, rb, ii, ib;
    for (size_t q = 0; q < rows.size(); ++q) {
        const int g = rows[q];
        bool interior = true;
        for (int e = A.rp[g]; e < A.rp[g + 1]; ++e)
            if (!own(A.ci[e])) interior = false;
        (interior ? ri : rb).push_back(g);
        (interior ? ii : ib).push_back(rowid[q]);
    }
    DG_TRY(build_local_ell(D, A, ri, ii, colmap, W, diag, in));
    DG_TRY(build_local_ell(D, A, rb, ib, colmap, W, diag, bd));
    return Status::Ok();
}

Status build_dist(decmg_gpu_dist* D, int agglomerate) {
    decmg_gpu_ctx* g = D->g.get();
    const int L = static_cast<int>(g->lv.size());
    const int N = D->world;
    D->L = L;
    if (L < 2) return Status::Err(DECMG_INVALID_ARGUMENT, "dist: the hierarchy needs at least two levels");
    // agglomeration level: first level with fewer than `agglomerate` vertices per rank
    int ka = L - 1;
    for (int k = 0; k < L; ++k)
        if (static_cast<int64_t>(g->lv[k].nv) < static_cast<int64_t>(agglomerate) * N) {
            ka = k;
            break;
        }
    if (ka < 1) ka = 1;  // level 0 is always distributed
    if (ka > L - 1) ka = L - 1;
    D->ka = ka;

    // ownership: contiguous ranges of the level-0 internal order; coarse
    // vertices inherit the owner of the fine vertex with the same id
    std::vector<std::vector<int>> owner(ka + 1), order(ka + 1);
    for (int k = 0; k <= ka; ++k) {
        const Level& m = g->lv[k];
        if (m.ord) {
            DG_TRY(download(m.ord, m.nv, &order[k]));
        } else {
            order[k].resize(m.nv);
            std::iota(order[k].begin(), order[k].end(), 0);
        }
        if (k > 0 && m.nv > g->lv[k - 1].nv) return Status::Err(DECMG_RUNTIME, "dist: levels must coarsen");
    }
    {
        const int n0 = g->lv[0].nv;
        owner[0].assign(n0, 0);
        for (int p = 0; p < N; ++p) {
            const int64_t a = static_cast<int64_t>(n0) * p / N, b = static_cast<int64_t>(n0) * (p + 1) / N;
            for (int64_t q = a; q < b; ++q) owner[0][order[0][q]] = p;
        }
        for (int k = 1; k <= ka; ++k) owner[k].assign(owner[k - 1].begin(), owner[k - 1].begin() + g->lv[k].nv);
    }
    // the replicated levels (>= ka) run on the shared hierarchy in its internal numbering
    std::vector<int> inv_ka(g->lv[ka].nv);
    if (g->lv[ka].inv) {
        DG_TRY(download(g->lv[ka].inv, g->lv[ka].nv, &inv_ka));
    } else {
        std::iota(inv_ka.begin(), inv_ka.end(), 0);
    }
    // reference-layout operators of the distributed levels
    std::vector<HostCSR> Lh(ka), Rh(ka), Ph(ka);
    for (int k = 0; k < ka; ++k) {
        const Level& m = g->lv[k];
        DG_TRY(fetch_csr(m.L_rp, m.L_ci, m.L_v, m.nv, m.nnzL, &Lh[k]));
        DG_TRY(fetch_csr(m.R_rp, m.R_ci, m.R_v, g->lv[k + 1].nv, m.nnzR, &Rh[k]));
        DG_TRY(fetch_csr(m.P_rp, m.P_ci, m.P_v, m.nv, m.nnzP, &Ph[k]));
    }
    // owned lists (internal order of the level) and halo sets of every rank,
    // the halo sorted by (owner, id)
    std::vector<std::vector<std::vector<int>>> own(ka + 1, std::vector<std::vector<int>>(N));
    for (int k = 0; k <= ka; ++k)
        for (int v : order[k]) own[k][owner[k][v]].push_back(v);
    std::vector<std::vector<std::vector<int>>> halo(ka, std::vector<std::vector<int>>(N));
    for (int k = 0; k < ka; ++k) {
        std::vector<int> mark(g->lv[k].nv, -1);
        for (int q = 0; q < N; ++q) {
            std::vector<int>& H = halo[k][q];
            auto add = [&](int v) {
                if (owner[k][v] != q && mark[v] != q) {
                    mark[v] = q;
                    H.push_back(v);
                }
            };
            for (int v : own[k][q])  // L_k rows
                for (int e = Lh[k].rp[v]; e < Lh[k].rp[v + 1]; ++e) add(Lh[k].ci[e]);
            for (int u : own[k + 1][q])  // R_k rows (level k+1 vertices owned by q)
                for (int e = Rh[k].rp[u]; e < Rh[k].rp[u + 1]; ++e) add(Rh[k].ci[e]);
            if (k > 0)
                for (int v : own[k - 1][q])  // P_{k-1} rows reference level k
                    for (int e = Ph[k - 1].rp[v]; e < Ph[k - 1].rp[v + 1]; ++e) add(Ph[k - 1].ci[e]);
            const std::vector<int>& ow = owner[k];
            std::sort(H.begin(), H.end(), [&](int a, int b) { return ow[a] != ow[b] ? ow[a] < ow[b] : a < b; });
        }
    }
    // halo traffic matrix cnt[k][q][p] = rows rank q sends to rank p at level k
    std::vector<std::vector<std::vector<int>>> cnt(ka, std::vector<std::vector<int>>(N, std::vector<int>(N, 0)));
    for (int k = 0; k < ka; ++k)
        for (int p = 0; p < N; ++p)
            for (int v : halo[k][p]) ++cnt[k][owner[k][v]][p];
    // host staging slot: the largest packed buffer of any rank (halo or all-gather)
    size_t slot_rows = 0;
    for (int k = 0; k < ka; ++k)
        for (int q = 0; q < N; ++q) {
            size_t s = 0;
            for (int p = 0; p < N; ++p) s += cnt[k][q][p];
            slot_rows = std::max(slot_rows, s);
        }
    for (int q = 0; q < N; ++q) slot_rows = std::max({slot_rows, own[0][q].size(), own[ka][q].size()});
    const size_t slot_bytes = std::max<size_t>(slot_rows * D->max_nrhs, 32) * sizeof(double);

    for (DRank& R : D->ranks) {
        const int p = R.rank;
        R.lv.resize(ka);
        std::vector<std::vector<int>> g2l(ka);
        for (int k = 0; k < ka; ++k) {
            g2l[k].assign(g->lv[k].nv, -1);
            int i = 0;
            for (int v : own[k][p]) g2l[k][v] = i++;
            for (int v : halo[k][p]) g2l[k][v] = i++;
        }
        for (int k = 0; k < ka; ++k) {
            DLevel& d = R.lv[k];
            const Level& m = g->lv[k];
            d.k = k;
            d.nown = static_cast<int>(own[k][p].size());
            d.nloc = d.nown + static_cast<int>(halo[k][p].size());
            DG_TRY(upload(D, &d.d_own, own[k][p]));
            const std::vector<int>& owk = owner[k];
            auto mine_k = [&](int v) { return owk[v] == p; };
            // L rows
            std::vector<int> lrow(d.nown);
            std::iota(lrow.begin(), lrow.end(), 0);
            const int lm = maxlen(Lh[k]);
            if (lm > 8) return Status::Err(DECMG_RUNTIME, "dist: vertex valence above 7 is not supported");
            d.Lw = lm <= 7 ? 7 : 8;
            DG_TRY(build_split_ell(D, Lh[k], own[k][p], lrow, g2l[k], d.Lw, true, mine_k, &d.Li, &d.Lb));
            std::vector<double> dg(d.nown, 0.0);
            d.zero_diag_row = -1;
            for (int q = 0; q < d.nown; ++q) {
                const int v = own[k][p][q];
                for (int e = Lh[k].rp[v]; e < Lh[k].rp[v + 1]; ++e)
                    if (Lh[k].ci[e] == v) dg[q] = Lh[k].v[e];
                if (dg[q] == 0.0 && d.zero_diag_row < 0) d.zero_diag_row = v;
            }
            DG_TRY(upload(D, &d.diag, dg));
            {
                std::vector<int> bdg, bdl(d.nown, 0);
                DG_TRY(download(m.bd, m.nv, &bdg));
                for (int q = 0; q < d.nown; ++q) bdl[q] = bdg[own[k][p][q]];
                DG_TRY(upload(D, &d.bd, bdl));
            }
            // R rows: owned level-(k+1) vertices (local rows when k+1 is distributed,
            // internal rows of the shared level otherwise)
            const bool next_dist = k + 1 < ka;
            std::vector<int> rrow;
            for (size_t q = 0; q < own[k + 1][p].size(); ++q)
                rrow.push_back(next_dist ? static_cast<int>(q) : inv_ka[own[k + 1][p][q]]);
            const int rm = maxlen(Rh[k]);
            if (rm > 8) return Status::Err(DECMG_RUNTIME, "dist: restriction row longer than 8");
            d.Rw = rm <= 7 ? 7 : 8;
            DG_TRY(build_split_ell(D, Rh[k], own[k + 1][p], rrow, g2l[k], d.Rw, false, mine_k, &d.Ri, &d.Rb));
            // P rows: owned level-k vertices, columns at level k+1
            std::vector<int> pmap;
            if (next_dist) {
                pmap.assign(g->lv[k + 1].nv, -1);
                int i = 0;
                for (int v : own[k + 1][p]) pmap[v] = i++;
                for (int v : halo[k + 1][p]) pmap[v] = i++;
            } else {
                pmap = inv_ka;
            }
            if (maxlen(Ph[k]) > 2) return Status::Err(DECMG_RUNTIME, "dist: prolongation row longer than 2");
            const std::vector<int>& ow1 = owner[k + 1];
            auto mine_k1 = [&](int v) { return !next_dist || ow1[v] == p; };
            DG_TRY(build_split_ell(D, Ph[k], own[k][p], lrow, pmap, 2, false, mine_k1, &d.Pi, &d.Pb));
            // halo exchange plan of level k: peers ascending; this rank's halo
            // slice from peer q is contiguous (halo sorted by owner)
            Xch& x = d.hx;
            x.recv_base = d.nown;
            std::vector<int> sidx;
            int roff = 0;
            for (int q = 0; q < N; ++q) {
                if (q == p || (cnt[k][p][q] == 0 && cnt[k][q][p] == 0)) continue;
                x.peer.push_back(q);
                x.soff.push_back(static_cast<int>(sidx.size()));
                for (int v : halo[k][q])
                    if (owner[k][v] == p) sidx.push_back(g2l[k][v]);
                x.scnt.push_back(static_cast<int>(sidx.size()) - x.soff.back());
                x.roff.push_back(roff);
                x.rcnt.push_back(cnt[k][q][p]);
                roff += cnt[k][q][p];
                int64_t off = 0;  // p's slice in q's packed buffer: q's peers before p
                for (int r = 0; r < p; ++r)
                    if (r != q) off += cnt[k][q][r];
                x.rsrc.push_back(off);
            }
            x.nsend = static_cast<int>(sidx.size());
            x.nrecv = roff;
            DG_TRY(upload(D, &x.sidx, sidx));
            DG_TRY(dmalloc(D, &x.sbuf, static_cast<size_t>(x.nsend) * D->max_nrhs));
            const size_t nv = static_cast<size_t>(d.nloc) * D->max_nrhs;
            DG_TRY(dmalloc(D, &d.x[0], nv));
            DG_TRY(dmalloc(D, &d.x[1], nv));
            DG_TRY(dmalloc(D, &d.b, nv));
            DG_TRY(dmalloc(D, &d.r, nv));
        }
        // all-gather plans: every rank's owned entries to every other rank.
        // slots: internal rows of the shared level ka / reference ids at level 0.
        auto allgather_plan = [&](int k, Xch* x, const std::vector<int>& slotmap) -> Status {
            x->gather = true;
            std::vector<int> sidx, ridx;
            for (int v : own[k][p]) sidx.push_back(slotmap.empty() ? v : slotmap[v]);
            int roff = 0;
            for (int q = 0; q < N; ++q) {
                if (q == p) continue;
                x->peer.push_back(q);
                x->soff.push_back(0);
                x->scnt.push_back(static_cast<int>(sidx.size()));
                x->roff.push_back(roff);
                x->rcnt.push_back(static_cast<int>(own[k][q].size()));
                x->rsrc.push_back(0);
                roff += static_cast<int>(own[k][q].size());
                for (int v : own[k][q]) ridx.push_back(slotmap.empty() ? v : slotmap[v]);
            }
            x->nsend = static_cast<int>(sidx.size());
            x->nrecv = roff;
            DG_TRY(upload(D, &x->sidx, sidx));
            DG_TRY(upload(D, &x->ridx, ridx));
            DG_TRY(dmalloc(D, &x->sbuf, static_cast<size_t>(x->nsend) * D->max_nrhs));
            DG_TRY(dmalloc(D, &x->rbuf, static_cast<size_t>(x->nrecv) * D->max_nrhs));
            return Status::Ok();
        };
        DG_TRY(allgather_plan(ka, &R.bx, inv_ka));
        // the level-0 solution is gathered from the internal numbering (xsol rows
        // = owned rows in internal order) into reference ids
        {
            Xch* x = &R.sx;
            x->gather = true;
            std::vector<int> sidx(own[0][p].size()), ridx;
            std::iota(sidx.begin(), sidx.end(), 0);  // xsol is already packed: rows 0..nown-1
            int roff = 0;
            for (int q = 0; q < N; ++q) {
                if (q == p) continue;
                x->peer.push_back(q);
                x->soff.push_back(0);
                x->scnt.push_back(static_cast<int>(sidx.size()));
                x->roff.push_back(roff);
                x->rcnt.push_back(static_cast<int>(own[0][q].size()));
                x->rsrc.push_back(0);
                roff += static_cast<int>(own[0][q].size());
                for (int v : own[0][q]) ridx.push_back(v);
            }
            x->nsend = static_cast<int>(sidx.size());
            x->nrecv = roff;
            DG_TRY(upload(D, &x->sidx, sidx));
            DG_TRY(upload(D, &x->ridx, ridx));
            DG_TRY(dmalloc(D, &x->sbuf, static_cast<size_t>(x->nsend) * D->max_nrhs));
            DG_TRY(dmalloc(D, &x->rbuf, static_cast<size_t>(x->nrecv) * D->max_nrhs));
        }
        // norm partials: up to 2 launches x (kPipeCtasPerSm * SMs or the ELL grid)
        const int bp = bp_of(D->max_nrhs);
        R.red_cap = 2 * ((static_cast<size_t>(R.lv[0].nown) * bp / 256 + 4 * 3 * g->num_sms + 64) * bp);
        DG_TRY(dmalloc(D, &R.red, R.red_cap));
        DG_TRY(dmalloc(D, &R.dsum, 32));
        DG_TRY(dmalloc(D, &R.xsol, static_cast<size_t>(R.lv[0].nown) * D->max_nrhs));
    }
    DG_TRY(dmalloc(D, &D->all, static_cast<size_t>(N) * 32));
    DG_TRY(dmalloc(D, &D->res, 32));
    DG_TRY(dmalloc(D, &D->hcnt, 1));
    {
        double* s;
        DG_TRY(dmalloc(D, &s, (sizeof(DistSolveState) + 7) / 8));
        D->st = reinterpret_cast<DistSolveState*>(s);
    }
    DG_CUDA(cudaHostAlloc(&D->hflag, 2 * sizeof(int), cudaHostAllocMapped));
    void* fd = nullptr;
    DG_CUDA(cudaHostGetDevicePointer(&fd, D->hflag, 0));
    D->hflag_dev = static_cast<int*>(fd);
    D->shm_slot = slot_bytes;
    return Status::Ok();
}

// --------------------------------------------------------------- driver ----
struct DistDriver {
    decmg_gpu_dist* D;
    int nrhs;
    std::vector<Driver> drv;  // one single-GPU driver per local rank (replicated levels + launches)
    // fused cycle residual: the next level-0 sweep also folds the norm of the
    // incoming x; then `on_norm(xprev per rank)` enqueues the consumers
    bool fuse = false;
    std::function<Status()> on_norm;

    decmg_gpu_ctx* g() const { return D->g.get(); }
    cudaStream_t stream() const { return g()->stream; }
    unsigned grid(int64_t t) const { return grid_for(t, 256); }
    int bp() const { return drv[0].bp; }

    // ---- exchanges -----------------------------------------------------
    Status pack(DRank& R, Xch& x, const double* v) {
        if (!x.nsend) return Status::Ok();
        return launch(g(), 6, 16.0 * x.nsend * nrhs, [&] {
            k_pack<<<grid(static_cast<int64_t>(x.nsend) * nrhs), 256, 0, stream()>>>(x.nsend, nrhs, x.sidx, v, x.sbuf);
        });
    }
    double* recv_ptr(Xch& x, int j, double* v) {
        return x.gather ? x.rbuf + static_cast<int64_t>(x.roff[j]) * nrhs
                        : v + (static_cast<int64_t>(x.recv_base) + x.roff[j]) * nrhs;
    }

    // Start moving the values of `vec_of(R)` described by plan `plan_of(R)`:
    // packs on the main stream; NCCL transfers on the communication stream
    // (finish() joins them); emulation and host staging complete here.
    template <class PlanOf, class VecOf>
    Status start(PlanOf plan_of, VecOf vec_of) {
        if (D->world == 1) return Status::Ok();
        for (DRank& R : D->ranks) DG_TRY(pack(R, *plan_of(R), vec_of(R)));
        if (D->kind == DECMG_DIST_EMULATE) {
            for (DRank& R : D->ranks) {
                Xch& x = *plan_of(R);
                for (size_t j = 0; j < x.peer.size(); ++j) {
                    if (!x.rcnt[j]) continue;
                    DRank& Q = D->ranks[x.peer[j]];
                    Xch& y = *plan_of(Q);
                    const auto it = std::find(y.peer.begin(), y.peer.end(), R.rank);
                    if (it == y.peer.end()) return Status::Err(DECMG_RUNTIME, "dist: inconsistent plan");
                    const size_t jj = it - y.peer.begin();
                    if (y.scnt[jj] != x.rcnt[j]) return Status::Err(DECMG_RUNTIME, "dist: inconsistent plan");
                    DG_CUDA(cudaMemcpyAsync(recv_ptr(x, static_cast<int>(j), vec_of(R)),
                                            y.sbuf + static_cast<int64_t>(y.soff[jj]) * nrhs,
                                            sizeof(double) * x.rcnt[j] * nrhs, cudaMemcpyDeviceToDevice, stream()));
                }
            }
        } else if (D->kind == DECMG_DIST_NCCL) {
            DG_CUDA(cudaEventRecord(D->ev_pack, stream()));
            DG_CUDA(cudaStreamWaitEvent(D->comm_stream, D->ev_pack, 0));
            DRank& R = D->ranks[0];
            Xch& x = *plan_of(R);
            double* v = vec_of(R);
            DG_NCCL(ncclGroupStart());
            for (size_t j = 0; j < x.peer.size(); ++j) {
                if (x.scnt[j])
                    DG_NCCL(ncclSend(x.sbuf + static_cast<int64_t>(x.soff[j]) * nrhs,
                                     static_cast<size_t>(x.scnt[j]) * nrhs, ncclDouble, x.peer[j], D->comm,
                                     D->comm_stream));
                if (x.rcnt[j])
                    DG_NCCL(ncclRecv(recv_ptr(x, static_cast<int>(j), v), static_cast<size_t>(x.rcnt[j]) * nrhs,
                                     ncclDouble, x.peer[j], D->comm, D->comm_stream));
            }
            DG_NCCL(ncclGroupEnd());
            DG_CUDA(cudaEventRecord(D->ev_comm, D->comm_stream));
        } else {  // host staging
            DRank& R = D->ranks[0];
            Xch& x = *plan_of(R);
            double* v = vec_of(R);
            const size_t sb = sizeof(double) * x.nsend * nrhs;
            if (sb > D->shm_slot) return Status::Err(DECMG_RUNTIME, "dist shm: slot too small");
            double* mine = shm_region(D, D->shm_parity, R.rank);
            if (sb) DG_CUDA(cudaMemcpyAsync(D->shm_stage, x.sbuf, sb, cudaMemcpyDeviceToHost, stream()));
            DG_CUDA(cudaStreamSynchronize(stream()));
            if (sb) std::memcpy(mine, D->shm_stage, sb);
            DG_TRY(shm_barrier(D));
            for (size_t j = 0; j < x.peer.size(); ++j) {
                if (!x.rcnt[j]) continue;
                const double* src = shm_region(D, D->shm_parity, x.peer[j]) + x.rsrc[j] * nrhs;
                // stream-ordered: the next pass on this stream sees the halo; the
                // source half is rewritten only after the next barrier, which follows
                // a synchronisation of this stream
                DG_CUDA(cudaMemcpyAsync(recv_ptr(x, static_cast<int>(j), v), src, sizeof(double) * x.rcnt[j] * nrhs,
                                        cudaMemcpyHostToDevice, stream()));
            }
            D->shm_parity ^= 1;  // the next exchange writes the other half (no second barrier)
        }
        return Status::Ok();
    }
    template <class PlanOf, class VecOf>
    Status finish(PlanOf plan_of, VecOf vec_of) {
        if (D->world == 1) return Status::Ok();
        if (D->kind == DECMG_DIST_NCCL) DG_CUDA(cudaStreamWaitEvent(stream(), D->ev_comm, 0));
        for (DRank& R : D->ranks) {
            Xch& x = *plan_of(R);
            if (!x.gather || !x.nrecv) continue;
            double* v = vec_of(R);
            DG_TRY(launch(g(), 6, 16.0 * x.nrecv * nrhs, [&] {
                k_unpack<<<grid(static_cast<int64_t>(x.nrecv) * nrhs), 256, 0, stream()>>>(x.nrecv, nrhs, x.ridx,
                                                                                        x.rbuf, v);
            }));
        }
        return Status::Ok();
    }
    auto halo_plan(int k) {
        return [k](DRank& R) { return &R.lv[k].hx; };
    }
    auto xcur_of(int k) {
        return [k](DRank& R) { return R.lv[k].x[R.lv[k].cur]; };
    }

    // Per-rank sums of `partial` launches folded to dsum; then the world's
    // per-lane residual norms in rank order -> D->res.
    Status fold_rank(DRank& R, int rows) {
        Driver& dr = drv[0];
        double* in = R.red;
        double* nxt = R.red + R.red_cap / 2;
        int64_t nr = rows;
        while (nr > 1) {
            const int64_t threads = nr * dr.bp;
            const unsigned gsz = grid_for(threads, kBlock);
            DG_TRY(launch(g(), kNorms, 8.0 * threads, [&] {
                DISPATCH_B1(dr.bp, k_fold<BP><<<gsz, kBlock, 0, stream()>>>(nr, in, nxt));
            }));
            nr = gsz;
            std::swap(in, nxt);
        }
        if (nr == 0) DG_CUDA(cudaMemsetAsync(in, 0, sizeof(double) * dr.bp, stream()));
        return launch(g(), kNorms, 0.0, [&] { k_finalize<<<1, 32, 0, stream()>>>(nrhs, in, R.dsum, 0, nullptr); });
    }
    Status world_norm() {
        const int N = D->world;
        if (D->kind == DECMG_DIST_EMULATE || N == 1) {
            for (DRank& R : D->ranks)
                DG_CUDA(cudaMemcpyAsync(D->all + static_cast<int64_t>(R.rank) * nrhs, R.dsum, sizeof(double) * nrhs,
                                        cudaMemcpyDeviceToDevice, stream()));
        } else if (D->kind == DECMG_DIST_NCCL) {
            DG_NCCL(ncclAllGather(D->ranks[0].dsum, D->all, nrhs, ncclDouble, D->comm, stream()));
        } else {
            DRank& R = D->ranks[0];
            double* mine = shm_region(D, D->shm_parity, R.rank);
            DG_CUDA(cudaMemcpyAsync(D->shm_stage, R.dsum, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, stream()));
            DG_CUDA(cudaStreamSynchronize(stream()));
            std::memcpy(mine, D->shm_stage, sizeof(double) * nrhs);
            DG_TRY(shm_barrier(D));
            for (int q = 0; q < N; ++q)
                DG_CUDA(cudaMemcpyAsync(D->all + static_cast<int64_t>(q) * nrhs, shm_region(D, D->shm_parity, q),
                                        sizeof(double) * nrhs, cudaMemcpyHostToDevice, stream()));
            D->shm_parity ^= 1;
        }
        return launch(g(), kNorms, 0.0, [&] {
            k_rank_fold<<<1, 32, 0, stream()>>>(N, nrhs, D->all, g()->dsmall, D->res);
        });
    }

    Status ensure_x(DRank& R, int k) {
        DLevel& d = R.lv[k];
        if (d.x_zero) {
            DG_CUDA(cudaMemsetAsync(d.x[d.cur], 0, sizeof(double) * d.nloc * nrhs, stream()));
            d.x_zero = false;
        }
        return Status::Ok();
    }

    // ---- passes --------------------------------------------------------
    template <int OP>
    Status rowop(size_t i, int w, int cls, const Ell& e, const double* x, const double* b, double* out,
                 double* partial, const int* zr, double omega, int* gsz) {
        if (e.rows == 0) {
            if (gsz) *gsz = 0;
            return Status::Ok();
        }
        const double bytes = 12.0 * w * e.rows + 4.0 * e.rows + 24.0 * e.rows * nrhs;
        if (w == 2) return drv[i].pipe<OP, 2>(cls, bytes, e.rows, e.ci, e.v, e.row, x, b, out, partial, zr, omega, gsz);
        return drv[i].pipe_w<OP>(w, cls, bytes, e.rows, e.ci, e.v, e.row, x, b, out, partial, zr, omega, gsz);
    }

    Status smooth(int k, int iters, const Plan& plan) {
        if (iters <= 0) return Status::Ok();
        if (k >= D->ka) return drv[0].smooth(k, iters, plan);  // replicated: one full copy per process
        for (DRank& R : D->ranks)
            if (R.lv[k].zero_diag_row >= 0)
                return Status::Err(DECMG_RUNTIME,
                                   "jacobi: zero diagonal at row " + std::to_string(R.lv[k].zero_diag_row));
        const int cls = k == 0 ? kFineSweep : kCoarseLevels;
        for (int it = 0; it < iters; ++it) {
            const bool zero = D->ranks[0].lv[k].x_zero;
            const bool norm = k == 0 && it == 0 && fuse && !zero;
            if (zero) {
                for (size_t i = 0; i < D->ranks.size(); ++i) {
                    DLevel& d = D->ranks[i].lv[k];
                    const double bytes = 8.0 * d.nown + 16.0 * d.nown * nrhs;
                    Driver& dr = drv[i];
                    DG_TRY(launch(g(), kZeroSweep, bytes, [&] {
                        DISPATCH_BP(dr.key, k_sweep_zero<BP, RPT><<<dr.rows_grid(d.nown), kBlock, 0, stream()>>>(
                                                d.nown, nrhs, d.diag, d.b, d.x[d.cur ^ 1], plan.omega));
                    }));
                }
            } else {
                DG_TRY(start(halo_plan(k), xcur_of(k)));
                std::vector<int> g1(D->ranks.size(), 0);
                for (size_t i = 0; i < D->ranks.size(); ++i) {  // interior rows while the halo is in flight
                    DRank& R = D->ranks[i];
                    DLevel& d = R.lv[k];
                    if (norm)
                        DG_TRY(rowop<OP_SWEEP_NORM>(i, d.Lw, cls, d.Li, d.x[d.cur], d.b, d.x[d.cur ^ 1], R.red,
                                                    nullptr, plan.omega, &g1[i]));
                    else
                        DG_TRY(rowop<OP_SWEEP>(i, d.Lw, cls, d.Li, d.x[d.cur], d.b, d.x[d.cur ^ 1], nullptr, nullptr,
                                               plan.omega, nullptr));
                }
                DG_TRY(finish(halo_plan(k), xcur_of(k)));
                for (size_t i = 0; i < D->ranks.size(); ++i) {
                    DRank& R = D->ranks[i];
                    DLevel& d = R.lv[k];
                    if (norm) {
                        int g2 = 0;
                        DG_TRY(rowop<OP_SWEEP_NORM>(i, d.Lw, cls, d.Lb, d.x[d.cur], d.b, d.x[d.cur ^ 1],
                                                    R.red + static_cast<int64_t>(g1[i]) * bp(), nullptr, plan.omega,
                                                    &g2));
                        DG_TRY(fold_rank(R, g1[i] + g2));
                    } else {
                        DG_TRY(rowop<OP_SWEEP>(i, d.Lw, cls, d.Lb, d.x[d.cur], d.b, d.x[d.cur ^ 1], nullptr, nullptr,
                                               plan.omega, nullptr));
                    }
                }
                if (norm) {
                    DG_TRY(world_norm());
                    DG_TRY(on_norm());  // x[cur] is still the incoming iterate
                    fuse = false;
                }
            }
            for (DRank& R : D->ranks) {
                R.lv[k].cur ^= 1;
                R.lv[k].x_zero = false;
            }
        }
        return Status::Ok();
    }

    // r = b - A x on level k (owned rows), then b_{k+1} = R r on the owned coarse rows
    Status residual_restrict(int k, const Plan& plan) {
        if (k >= D->ka) return drv[0].residual_restrict(k);
        (void)plan;
        for (DRank& R : D->ranks) DG_TRY(ensure_x(R, k));
        const int cls = k == 0 ? kFineResidual : kCoarseLevels;
        DG_TRY(start(halo_plan(k), xcur_of(k)));
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DLevel& d = D->ranks[i].lv[k];
            DG_TRY(rowop<OP_RES_STORE>(i, d.Lw, cls, d.Li, d.x[d.cur], d.b, d.r, nullptr, nullptr, 0.0, nullptr));
        }
        DG_TRY(finish(halo_plan(k), xcur_of(k)));
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DLevel& d = D->ranks[i].lv[k];
            DG_TRY(rowop<OP_RES_STORE>(i, d.Lw, cls, d.Lb, d.x[d.cur], d.b, d.r, nullptr, nullptr, 0.0, nullptr));
        }
        auto rvec = [k](DRank& R) { return R.lv[k].r; };
        DG_TRY(start(halo_plan(k), rvec));
        const bool next_dist = k + 1 < D->ka;
        const int rcls = k == 0 ? kRestrict : kCoarseLevels;
        auto restrict_rows = [&](bool interior) -> Status {
            for (size_t i = 0; i < D->ranks.size(); ++i) {
                DRank& R = D->ranks[i];
                DLevel& d = R.lv[k];
                double* out = next_dist ? R.lv[k + 1].b : g()->lv[k + 1].b;
                const int* zr = nullptr;  // restricted RHS is zero on Dirichlet vertices (x1)
                if (g()->dirichlet) zr = next_dist ? R.lv[k + 1].bd : g()->lv[k + 1].bd_i;
                DG_TRY(rowop<OP_SPMV>(i, d.Rw, rcls, interior ? d.Ri : d.Rb, d.r, nullptr, out, nullptr, zr, 0.0,
                                      nullptr));
            }
            return Status::Ok();
        };
        DG_TRY(restrict_rows(true));
        DG_TRY(finish(halo_plan(k), rvec));
        DG_TRY(restrict_rows(false));
        if (!next_dist) {  // all-gather the owned entries of b_ka (replicated levels)
            auto bvec = [this](DRank&) { return g()->lv[D->ka].b; };
            auto bplan = [](DRank& R) { return &R.bx; };
            DG_TRY(start(bplan, bvec));
            DG_TRY(finish(bplan, bvec));
        }
        return Status::Ok();
    }

    // x_k += P_k x_{k+1} on the owned fine rows
    Status prolong(int k) {
        if (k >= D->ka) return drv[0].prolong(k);
        const bool next_dist = k + 1 < D->ka;
        const int cls = k == 0 ? kProlong : kCoarseLevels;
        if (next_dist) {
            for (DRank& R : D->ranks) DG_TRY(ensure_x(R, k + 1));
            DG_TRY(start(halo_plan(k + 1), xcur_of(k + 1)));
        } else {
            DG_TRY(drv[0].ensure_x(k + 1));
        }
        auto rows = [&](bool interior) -> Status {
            for (size_t i = 0; i < D->ranks.size(); ++i) {
                DRank& R = D->ranks[i];
                DG_TRY(ensure_x(R, k));
                DLevel& d = R.lv[k];
                const double* xc =
                    next_dist ? R.lv[k + 1].x[R.lv[k + 1].cur] : g()->lv[k + 1].x[g()->lv[k + 1].cur];
                DG_TRY(rowop<OP_PROLONG>(i, 2, cls, interior ? d.Pi : d.Pb, xc, nullptr, d.x[d.cur], nullptr,
                                         nullptr, 0.0, nullptr));
            }
            return Status::Ok();
        };
        DG_TRY(rows(true));
        if (next_dist) DG_TRY(finish(halo_plan(k + 1), xcur_of(k + 1)));
        DG_TRY(rows(false));
        return Status::Ok();
    }

    // MultigridHierarchy::cycle_once (multigrid.cpp:252-285) over the partition;
    // below ka the replicated driver runs (one cooperative kernel for the bottom
    // of the V when Driver::tail_ok allows).
    Status cycle_once(const Plan& plan) {
        const int nw = static_cast<int>(plan.walk.size());
        const int L = D->L;
        int level = 0;
        for (int w = 0; w < nw; ++w) {
            if (plan.walk[w] == 'd' && level >= D->ka && drv[0].tail_ok(plan, w, level)) {
                DG_TRY(drv[0].run_tail(plan, level));
                w += 2 * (L - 1 - level) - 1;
                continue;
            }
            if (plan.walk[w] == 'd') {
                DG_TRY(smooth(level, plan.pre[level], plan));
                DG_TRY(residual_restrict(level, plan));
                ++level;
                if (level < D->ka) {
                    for (DRank& R : D->ranks) R.lv[level].x_zero = true;
                } else {
                    g()->lv[level].x_zero = true;
                }
                if (level == L - 1) {
                    DG_TRY(drv[0].coarse_solve(level));
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

    // D->res[lane] = ||b - A x|| / ||b|| over all ranks' owned level-0 rows
    Status resnorm() {
        for (DRank& R : D->ranks) DG_TRY(ensure_x(R, 0));
        DG_TRY(start(halo_plan(0), xcur_of(0)));
        std::vector<int> g1(D->ranks.size(), 0);
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DRank& R = D->ranks[i];
            DLevel& d = R.lv[0];
            DG_TRY(rowop<OP_RES_NORM>(i, d.Lw, kFineResidual, d.Li, d.x[d.cur], d.b, nullptr, R.red, nullptr, 0.0,
                                      &g1[i]));
        }
        DG_TRY(finish(halo_plan(0), xcur_of(0)));
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DRank& R = D->ranks[i];
            DLevel& d = R.lv[0];
            int g2 = 0;
            DG_TRY(rowop<OP_RES_NORM>(i, d.Lw, kFineResidual, d.Lb, d.x[d.cur], d.b, nullptr,
                                      R.red + static_cast<int64_t>(g1[i]) * bp(), nullptr, 0.0, &g2));
            DG_TRY(fold_rank(R, g1[i] + g2));
        }
        return world_norm();
    }

};

}  // namespace

namespace {

// Host view of every ping-pong buffer (distributed levels of every local rank,
// then the shared hierarchy's levels).
std::vector<std::pair<int, bool>> host_state(const decmg_gpu_dist* D) {
    std::vector<std::pair<int, bool>> s;
    for (const DRank& R : D->ranks)
        for (const DLevel& d : R.lv) s.emplace_back(d.cur, d.x_zero);
    for (const Level& L : D->g->lv) s.emplace_back(L.cur, L.x_zero);
    return s;
}
void set_host_state(decmg_gpu_dist* D, const std::vector<std::pair<int, bool>>& s) {
    size_t i = 0;
    for (DRank& R : D->ranks)
        for (DLevel& d : R.lv) {
            d.cur = s[i].first;
            d.x_zero = s[i++].second;
        }
    for (Level& L : D->g->lv) {
        L.cur = s[i].first;
        L.x_zero = s[i++].second;
    }
}

// Level-0 Jacobi sweeps per cycle of the walk: a body replayed as a graph
// keeps level 0's ping-pong parity only if this is even (coarser levels
// restart from zero on every descent).
int level0_sweeps(const Plan& plan) {
    int sweeps = 0, level = 0;
    for (char t : plan.walk) {
        if (t == 'd') {
            if (level == 0) sweeps += plan.pre[0];
            ++level;
        } else {
            --level;
            if (level == 0) sweeps += plan.post[0];
        }
    }
    return sweeps;
}

}  // namespace

// run_cycle (solve == false: ncycles cycles, the residual after each) or
// gmg_solve (solve == true) over the partition; b (full, reference numbering)
// replicated on every rank. After the first cycle every cycle is a "body":
// its first level-0 sweep also yields the residual of the incoming iterate
// (fused norm, rank sums all-gathered and folded on the device), followed by
// the history store (run_cycle) or the convergence check and snapshot of the
// finished lanes (gmg_solve), then the rest of the cycle. Bodies are replayed
// as one CUDA graph (NCCL / emulation) when the cycle keeps level 0's parity.
// gmg_solve reads each check's outcome through mapped pinned memory while the
// rest of that body runs, so the host never drains the stream between cycles.
Status dist_run(decmg_gpu_dist* D, const Plan& plan, int nrhs, const double* h_b, const double* h_x0, int ncycles,
                bool solve, double tol, double* h_x, double* h_hist, int* cycles_done, double* h_final) {
    decmg_gpu_ctx* g = D->g.get();
    if (nrhs < 1 || nrhs > D->max_nrhs) return Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs]");
    if (ncycles < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "gmg_solve: max_cycles >= 0");
    const int n0 = g->lv[0].nv;
    const size_t nb = sizeof(double) * n0 * nrhs;
    DistDriver dd{D, nrhs, {}};
    for (size_t i = 0; i < D->ranks.size(); ++i) {
        Driver dr{g, nrhs, bp_of(nrhs), g->lv[0].b};
        dr.use_pairs = false;
        dr.init();
        dd.drv.push_back(dr);
    }
    cudaStream_t st = g->stream;
    // full right-hand side on this process (replicated), projected like gmg_solve
    DG_CUDA(cudaMemcpyAsync(g->io_b, h_b, nb, cudaMemcpyHostToDevice, st));
    if (solve && !g->dirichlet) DG_TRY(project_compatible(g, nrhs, g->io_b));
    {  // ||b|| over the internal numbering, exactly as the single-GPU run
        Driver d0{g, nrhs, bp_of(nrhs), g->lv[0].b};
        d0.use_pairs = false;
        d0.init();
        DG_TRY(d0.to_internal(g->io_b, g->lv[0].b));
        DG_TRY(d0.make_denom(g->dsmall));
    }
    if (h_x0) DG_CUDA(cudaMemcpyAsync(g->io_x0, h_x0, nb, cudaMemcpyHostToDevice, st));
    for (DRank& R : D->ranks) {
        DLevel& d = R.lv[0];
        const unsigned gr = grid_for(static_cast<int64_t>(d.nown) * nrhs, 256);
        DG_TRY(launch(g, 6, 0.0, [&] { k_pack<<<gr, 256, 0, st>>>(d.nown, nrhs, d.d_own, g->io_b, d.b); }));
        d.cur = 0;
        if (h_x0) {
            DG_TRY(launch(g, 6, 0.0, [&] { k_pack<<<gr, 256, 0, st>>>(d.nown, nrhs, d.d_own, g->io_x0, d.x[0]); }));
            d.x_zero = false;
        } else {
            d.x_zero = true;
        }
    }
    const int hist_rows = std::max(ncycles, 1);
    if (hist_rows > D->hist_cap) {
        DG_TRY(dmalloc(D, &D->hist, static_cast<size_t>(hist_rows) * 32));
        D->hist_cap = hist_rows;
    }
    DG_CUDA(cudaMemsetAsync(D->hcnt, 0, sizeof(int), st));
    const unsigned all = nrhs == 32 ? 0xffffffffu : ((1u << nrhs) - 1u);
    DG_TRY(launch(g, kNorms, 0.0, [&] {
        k_dist_state_init<<<1, 1, 0, st>>>(D->st, ncycles == 0 ? 0 : 1, all, ncycles, tol);
    }));
    DG_CUDA(cudaStreamSynchronize(st));
    D->hflag[0] = -1;
    D->hflag[1] = 0;

    // consumers of a cycle residual in D->res
    auto put_hist = [&]() -> Status {
        return launch(g, kNorms, 0.0, [&] { k_hist_put<<<1, 32, 0, st>>>(nrhs, D->res, D->hist, D->hcnt); });
    };
    auto check_snapshot = [&]() -> Status {
        DG_TRY(launch(g, kNorms, 0.0, [&] {
            k_dist_check<<<1, 32, 0, st>>>(nrhs, D->res, D->st, D->hist, D->hflag_dev);
        }));
        for (DRank& R : D->ranks) {
            DLevel& d = R.lv[0];
            const int64_t total = static_cast<int64_t>(d.nown) * nrhs;
            const double* xsrc = d.x[d.cur];
            DG_TRY(launch(g, kNorms, 16.0 * total, [&] {
                k_dist_copy_lanes<<<grid_for(total, 256), 256, 0, st>>>(total, nrhs, D->st, xsrc, R.xsol);
            }));
        }
        return Status::Ok();
    };
    auto wait_flag = [&](int cyc, bool* alldone) -> Status {
        const auto t0 = std::chrono::steady_clock::now();
        volatile int* f = D->hflag;
        while (f[0] != cyc) {
            const cudaError_t q = cudaStreamQuery(st);
            if (q == cudaSuccess) {
                if (f[0] == cyc) break;
                return Status::Err(DECMG_RUNTIME, "dist: convergence flag missing");
            }
            if (q != cudaErrorNotReady) return cuda_status(q, "dist: cycle stream");
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
                return Status::Err(DECMG_RUNTIME, "dist: convergence flag timed out");
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        *alldone = f[1] != 0;
        return Status::Ok();
    };

    // one body, eagerly
    auto body = [&]() -> Status {
        dd.fuse = true;
        dd.on_norm = solve ? std::function<Status()>(check_snapshot) : std::function<Status()>(put_hist);
        Status s = dd.cycle_once(plan);
        dd.fuse = false;
        dd.on_norm = nullptr;
        return s;
    };
    // the body as a graph (captured from `body` itself, so the same kernels and arguments)
    decmg_gpu_dist::GraphEntry* ge = nullptr;
    auto make_graph = [&]() -> Status {
        if (!g->graph || D->kind == DECMG_DIST_SHM || g->timing.enabled || level0_sweeps(plan) % 2) return Status::Ok();
        uint64_t ob = 0;
        std::memcpy(&ob, &plan.omega, sizeof ob);
        std::string key = plan.walk + "|" + std::to_string(ob) + "|" + std::to_string(nrhs) + "|" +
                          std::to_string(solve ? 1 : 0) + "|";
        for (size_t k = 0; k < plan.pre.size(); ++k)
            key += std::to_string(plan.pre[k]) + "," + std::to_string(plan.post[k]) + ";";
        const auto s0 = host_state(D);
        for (const auto& e : s0) key += std::to_string(e.first) + (e.second ? "z" : ".");
        for (auto& e : D->graphs)
            if (e.key == key) {
                ge = &e;
                return Status::Ok();
            }
        const int64_t lc0 = g->launch_count;
        DG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        Status s = body();
        cudaGraph_t gr = nullptr;
        const cudaError_t e = cudaStreamEndCapture(st, &gr);
        const int64_t kernels = g->launch_count - lc0;  // recorded, not run: counted per replay
        g->launch_count = lc0;
        const auto s1 = host_state(D);
        set_host_state(D, s0);  // nothing ran yet
        if (s.ok() && e != cudaSuccess) s = cuda_status(e, "dist graph capture");
        cudaGraphExec_t ex = nullptr;
        if (s.ok() && cudaGraphInstantiate(&ex, gr, 0) != cudaSuccess) s = Status::Err(DECMG_CUDA, "dist graph instantiate");
        if (!s.ok()) {
            // a transport whose calls cannot be captured (nothing has run: the host state is restored):
            // drop the graph for this context and run the cycles eagerly, as the first one did
            if (gr) cudaGraphDestroy(gr);
            cudaGetLastError();
            g->graph = 0;
            if (std::getenv("DECMG_DEBUG")) std::fprintf(stderr, "[decmg] dist: %s; cycles run eagerly\n", s.msg.c_str());
            return Status::Ok();
        }
        D->graphs.push_back({key, gr, ex, s1, kernels});
        ge = &D->graphs.back();
        return Status::Ok();
    };
    const bool fusable = ncycles >= 2 && !plan.walk.empty() && plan.walk[0] == 'd' && plan.pre[0] >= 1;
    // a cycle whose start yields the residual of the incoming iterate
    auto step = [&]() -> Status {
        if (ge) {
            DG_CUDA(cudaGraphLaunch(ge->exec, st));
            g->launch_count += ge->kernels;
            set_host_state(D, ge->post);
            return Status::Ok();
        }
        return body();
    };

    if (!D->ev[0]) {
        DG_CUDA(cudaEventCreate(&D->ev[0]));
        DG_CUDA(cudaEventCreate(&D->ev[1]));
    }
    DG_CUDA(cudaEventRecord(D->ev[0], st));
    if (!solve) {
        if (ncycles >= 1) DG_TRY(dd.cycle_once(plan));  // cycle 0, from x0
        if (fusable) DG_TRY(make_graph());
        for (int cyc = 1; cyc < ncycles; ++cyc) {
            if (fusable) {
                DG_TRY(step());  // hist[cyc - 1], then cycle cyc
            } else {
                DG_TRY(dd.resnorm());
                DG_TRY(put_hist());
                DG_TRY(dd.cycle_once(plan));
            }
        }
        if (ncycles >= 1) {
            DG_TRY(dd.resnorm());
            DG_TRY(put_hist());
        }
        DG_CUDA(cudaEventRecord(D->ev[1], st));
        for (DRank& R : D->ranks) {  // the solution: owned rows of x, gathered below
            DG_TRY(dd.ensure_x(R, 0));
            DLevel& d = R.lv[0];
            DG_CUDA(cudaMemcpyAsync(R.xsol, d.x[d.cur], sizeof(double) * d.nown * nrhs, cudaMemcpyDeviceToDevice, st));
        }
    } else {
        bool done = false;
        if (ncycles == 0) {  // the solution is x0
            DG_TRY(dd.resnorm());
            DG_TRY(check_snapshot());
            DG_TRY(wait_flag(0, &done));
        } else {
            DG_TRY(dd.cycle_once(plan));
            if (fusable) DG_TRY(make_graph());
            int cyc = 1;
            while (cyc < ncycles) {
                if (fusable) {
                    DG_TRY(step());  // check of the iterate after `cyc` cycles, then cycle cyc
                } else {
                    DG_TRY(dd.resnorm());
                    DG_TRY(check_snapshot());
                }
                // the check is early in the step: the host learns the outcome while
                // the rest of the step runs, and queues the next one behind it
                DG_TRY(wait_flag(cyc, &done));
                if (done) break;
                if (!fusable) DG_TRY(dd.cycle_once(plan));
                ++cyc;
            }
            if (!done) {  // the iterate after max_cycles cycles (every lane finishes)
                DG_TRY(dd.resnorm());
                DG_TRY(check_snapshot());
                DG_TRY(wait_flag(ncycles, &done));
            }
        }
        DG_CUDA(cudaEventRecord(D->ev[1], st));
    }
    DG_CUDA(cudaEventSynchronize(D->ev[1]));
    DG_CUDA(cudaEventElapsedTime(&D->last_cycle_ms, D->ev[0], D->ev[1]));
    // gather the solution: every rank's owned rows -> full vector (reference numbering)
    {
        auto splan = [](DRank& R) { return &R.sx; };
        DG_TRY(dd.start(splan, [](DRank& R) { return R.xsol; }));
        DG_TRY(dd.finish(splan, [g](DRank&) { return g->io_x; }));
        for (DRank& R : D->ranks) {
            DLevel& d = R.lv[0];
            DG_TRY(launch(g, 6, 0.0, [&] {
                k_unpack<<<grid_for(static_cast<int64_t>(d.nown) * nrhs, 256), 256, 0, st>>>(d.nown, nrhs, d.d_own,
                                                                                            R.xsol, g->io_x);
            }));
        }
    }
    DG_CUDA(cudaMemcpyAsync(h_x, g->io_x, nb, cudaMemcpyDeviceToHost, st));
    std::vector<double> hist(static_cast<size_t>(hist_rows) * nrhs);
    DG_CUDA(cudaMemcpyAsync(hist.data(), D->hist, sizeof(double) * hist.size(), cudaMemcpyDeviceToHost, st));
    DistSolveState hs;
    DG_CUDA(cudaMemcpyAsync(&hs, D->st, sizeof hs, cudaMemcpyDeviceToHost, st));
    double res_last[32];
    DG_CUDA(cudaMemcpyAsync(res_last, D->res, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, st));
    DG_CUDA(cudaStreamSynchronize(st));
    if (!solve) {
        if (h_hist) std::memcpy(h_hist, hist.data(), sizeof(double) * static_cast<size_t>(ncycles) * nrhs);
        for (int l = 0; l < nrhs; ++l) {
            if (cycles_done) cycles_done[l] = ncycles;
            if (h_final) h_final[l] = ncycles ? res_last[l] : 0.0;
        }
        return Status::Ok();
    }
    for (int l = 0; l < nrhs; ++l) {
        if (cycles_done) cycles_done[l] = hs.done[l];
        if (h_final) h_final[l] = hs.final_res[l];
        if (h_hist)
            for (int k = 0; k < hs.done[l]; ++k)
                h_hist[static_cast<int64_t>(k) * nrhs + l] = hist[static_cast<size_t>(k) * nrhs + l];
    }
    for (int l = 0; l < nrhs; ++l)
        if (!std::isfinite(hs.final_res[l]))
            return Status::Err(DECMG_RUNTIME, "gmg_solve: non-finite residual (right-hand side " + std::to_string(l) +
                                                  ", cycle " + std::to_string(hs.done[l]) + ")");
    return Status::Ok();
}

Status dist_create(decmg_gpu_dist* D, const double* pos, int nv, const int* tri, int nt, int nsub, unsigned flags,
                   const decmg_gpu_config* cfg, int agglomerate) {
    decmg_gpu_ctx* g = nullptr;
    const int rc = decmg_gpu_create_from_base(pos, nv, tri, nt, nsub, flags, cfg, &g);
    if (rc != DECMG_OK) return Status::Err(rc, decmg_gpu_last_error(nullptr));
    D->g = std::unique_ptr<decmg_gpu_ctx, void (*)(decmg_gpu_ctx*)>(g, decmg_gpu_destroy);
    D->max_nrhs = cfg ? cfg->max_nrhs : 1;
    DG_TRY(build_dist(D, agglomerate));
    return Status::Ok();
}

}  // namespace decmg_gpu

using namespace decmg_gpu;

extern "C" {

int decmg_gpu_nccl_unique_id(void* out, int bytes) {
    if (!out || bytes < static_cast<int>(sizeof(ncclUniqueId))) return DECMG_INVALID_ARGUMENT;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return DECMG_NCCL;
    std::memcpy(out, &id, sizeof id);
    return DECMG_OK;
}

int decmg_gpu_dist_create_ex(const double* positions, int nv, const int* corner_triples, int nt, int nsub,
                             unsigned flags, const decmg_gpu_config* cfg, int world_size, int rank,
                             const decmg_gpu_dist_transport* tr, int agglomerate_below, decmg_gpu_dist** out) {
    if (!out || world_size < 1) return DECMG_INVALID_ARGUMENT;
    *out = nullptr;
    const int kind = tr ? tr->kind : DECMG_DIST_EMULATE;
    if (kind != DECMG_DIST_EMULATE && kind != DECMG_DIST_NCCL && kind != DECMG_DIST_SHM) {
        g_dist_create_error = "dist: unknown transport";
        return DECMG_INVALID_ARGUMENT;
    }
    if (kind != DECMG_DIST_EMULATE && (rank < 0 || rank >= world_size)) {
        g_dist_create_error = "dist: rank out of range";
        return DECMG_INVALID_ARGUMENT;
    }
    if ((kind == DECMG_DIST_NCCL && !tr->nccl_id) || (kind == DECMG_DIST_SHM && !tr->shm_path)) {
        g_dist_create_error = "dist: transport needs its rendezvous (nccl_id / shm_path)";
        return DECMG_INVALID_ARGUMENT;
    }
    auto* D = new decmg_gpu_dist();
    D->world = world_size;
    D->kind = kind;
    if (kind == DECMG_DIST_EMULATE) {
        for (int p = 0; p < world_size; ++p) {
            DRank R;
            R.rank = p;
            D->ranks.push_back(R);
        }
    } else {
        DRank R;
        R.rank = rank;
        D->ranks.push_back(R);
    }
    Status s = dist_create(D, positions, nv, corner_triples, nt, nsub, flags, cfg,
                           agglomerate_below > 0 ? agglomerate_below : 65536);
    if (s.ok()) {
        const int dev = cfg ? cfg->device : 0;
        cudaSetDevice(dev);
        if (kind == DECMG_DIST_NCCL && world_size > 1) {
            ncclUniqueId id;
            std::memcpy(&id, tr->nccl_id, sizeof id);
            if (ncclCommInitRank(&D->comm, world_size, id, rank) != ncclSuccess)
                s = Status::Err(DECMG_NCCL, "ncclCommInitRank failed");
            if (s.ok()) s = cuda_status(cudaStreamCreateWithFlags(&D->comm_stream, cudaStreamNonBlocking), "stream");
            if (s.ok()) s = cuda_status(cudaEventCreateWithFlags(&D->ev_pack, cudaEventDisableTiming), "event");
            if (s.ok()) s = cuda_status(cudaEventCreateWithFlags(&D->ev_comm, cudaEventDisableTiming), "event");
        } else if (kind == DECMG_DIST_SHM && world_size > 1) {
            s = shm_open_map(D, tr->shm_path, D->shm_slot);
            if (s.ok()) s = shm_barrier(D);  // every process mapped the file
        }
    }
    if (!s.ok()) {
        decmg_gpu_dist_destroy(D);
        g_dist_create_error = s.msg;
        return s.code;
    }
    *out = D;
    return DECMG_OK;
}

int decmg_gpu_dist_create(const double* positions, int nv, const int* corner_triples, int nt, int nsub,
                          unsigned flags, const decmg_gpu_config* cfg, int world_size, int rank,
                          const void* nccl_id, int agglomerate_below, decmg_gpu_dist** out) {
    decmg_gpu_dist_transport t{nccl_id ? DECMG_DIST_NCCL : DECMG_DIST_EMULATE, nccl_id, nullptr};
    return decmg_gpu_dist_create_ex(positions, nv, corner_triples, nt, nsub, flags, cfg, world_size, rank, &t,
                                    agglomerate_below, out);
}

void decmg_gpu_dist_destroy(decmg_gpu_dist* D) {
    if (!D) return;
    if (D->g) cudaStreamSynchronize(D->g->stream);
    if (D->comm) ncclCommDestroy(D->comm);
    for (auto& e : D->graphs) {
        cudaGraphExecDestroy(e.exec);
        cudaGraphDestroy(e.graph);
    }
    for (cudaEvent_t e : D->ev)
        if (e) cudaEventDestroy(e);
    if (D->ev_pack) cudaEventDestroy(D->ev_pack);
    if (D->ev_comm) cudaEventDestroy(D->ev_comm);
    if (D->comm_stream) cudaStreamDestroy(D->comm_stream);
    for (void* p : D->allocs) cudaFree(p);
    if (D->hflag) cudaFreeHost(D->hflag);
    if (D->shm_stage) cudaFreeHost(D->shm_stage);
    if (D->shm) ::munmap(D->shm, D->shm_bytes);
    if (D->shm_fd >= 0) ::close(D->shm_fd);
    delete D;
}

decmg_gpu_ctx* decmg_gpu_dist_context(decmg_gpu_dist* D) { return D ? D->g.get() : nullptr; }

double decmg_gpu_dist_last_cycle_ms(const decmg_gpu_dist* D) { return D ? D->last_cycle_ms : -1.0; }

int64_t decmg_gpu_dist_launch_count(const decmg_gpu_dist* D) { return D && D->g ? D->g->launch_count : -1; }

const char* decmg_gpu_dist_last_error(const decmg_gpu_dist* D) {
    return D ? D->err.c_str() : g_dist_create_error.c_str();
}

int decmg_gpu_dist_info(const decmg_gpu_dist* D, int* agglomeration_level, int* levels, int64_t* owned0,
                        int64_t* halo0) {
    if (!D) return DECMG_INVALID_ARGUMENT;
    if (agglomeration_level) *agglomeration_level = D->ka;
    if (levels) *levels = D->L;
    if (owned0) *owned0 = D->ranks[0].lv[0].nown;
    if (halo0) *halo0 = D->ranks[0].lv[0].nloc - D->ranks[0].lv[0].nown;
    return DECMG_OK;
}

int decmg_gpu_dist_run(decmg_gpu_dist* D, const decmg_gpu_plan* plan, int nrhs, const double* b, const double* x0,
                       int max_cycles, int solve, double tol, double* x_out, double* hist_out, int* cycles_done,
                       double* final_out) {
    if (!D || !b || !x_out) return DECMG_INVALID_ARGUMENT;
    cudaSetDevice(D->g->device);
    Plan p;
    Status s = make_plan(D->g.get(), plan, &p);
    if (s.ok() && p.smoother != DECMG_SMOOTHER_JACOBI)
        s = Status::Err(DECMG_INVALID_ARGUMENT, "partitioned solve: only the weighted Jacobi smoother");
    if (s.ok())
        s = dist_run(D, p, nrhs, b, x0, max_cycles, solve != 0, tol, x_out, hist_out, cycles_done, final_out);
    if (!s.ok()) {
        D->err = s.msg;
        return s.code;
    }
    return DECMG_OK;
}

}  // extern "C"
