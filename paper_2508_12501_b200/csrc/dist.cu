// Vertex-partitioned multi-GPU V-cycle.
//
// Every rank builds the full hierarchy (deterministic, bit-identical on all
// ranks), then takes a partition of the finer levels:
//  * ownership: Morton key of the vertex position in the finest level's box,
//    split by key thresholds taken from the finest level's sorted keys, so a
//    coarse vertex and its fine copy share an owner on every level;
//  * levels 0 .. ka-1 are distributed: rank p owns the vertices of its key
//    range and keeps a 1-ring halo (every vertex its owned rows of L_k, its
//    owned coarse rows of R_k and its owned fine rows of P_{k-1} reference);
//    local vectors are [owned (Morton order) | halo (global id order)];
//  * levels ka .. L-1 (fewer than `agglomerate` vertices per rank) are
//    replicated: every rank runs them on its full copy, identically, after
//    the restricted right-hand side of level ka is all-gathered.
// Every row's arithmetic is the single-GPU one (same entries, same order), so
// iterates are bit-identical to the 1-GPU solve for any rank count. Halo
// exchanges are NCCL grouped send/recv on the rank's stream; norms are
// per-rank partial sums all-gathered and added in rank order (deterministic).
//
// Emulation mode runs all ranks of a world in one process on one device and
// one stream, with device copies in place of NCCL; nothing waits on another
// rank's kernel, so it is safe on a single GPU and is what the parity tests use.
#include "driver.cuh"

#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <numeric>

namespace decmg_gpu {
namespace {

__global__ void k_pack(int n, int nrhs, const int* __restrict__ idx, const double* __restrict__ v,
                       double* __restrict__ buf) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * nrhs) return;
    const int64_t i = t / nrhs;
    const int l = static_cast<int>(t % nrhs);
    buf[t] = v[static_cast<int64_t>(idx[i]) * nrhs + l];
}

__global__ void k_unpack(int n, int nrhs, const int* __restrict__ idx, const double* __restrict__ buf,
                         double* __restrict__ v) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * nrhs) return;
    const int64_t i = t / nrhs;
    const int l = static_cast<int>(t % nrhs);
    v[static_cast<int64_t>(idx[i]) * nrhs + l] = buf[t];
}

// dst[i] = src[map[i]] (rows of nrhs values)
__global__ void k_gather_rows(int n, int nrhs, const int* __restrict__ map, const double* __restrict__ src,
                              double* __restrict__ dst) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * nrhs) return;
    const int64_t i = t / nrhs;
    const int l = static_cast<int>(t % nrhs);
    dst[t] = src[static_cast<int64_t>(map[i]) * nrhs + l];
}

// dst[map[i]] = src[i]
__global__ void k_scatter_rows(int n, int nrhs, const int* __restrict__ map, const double* __restrict__ src,
                               double* __restrict__ dst) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * nrhs) return;
    const int64_t i = t / nrhs;
    const int l = static_cast<int>(t % nrhs);
    dst[static_cast<int64_t>(map[i]) * nrhs + l] = src[t];
}

struct XPeer {
    int rank = -1;
    int nsend = 0, nrecv = 0;
    int* d_send = nullptr;  // local indices packed for the peer
    int* d_recv = nullptr;  // local halo slots filled from the peer
    double* sbuf = nullptr;
    double* rbuf = nullptr;
};

struct DLevel {
    int k = 0;
    int nown = 0, nloc = 0;
    int* d_own = nullptr;   // global ids of the owned rows (local 0..nown-1)
    // operators in local numbering, padded ELL rows (multiple of 224)
    int Lw = 0;
    int* Lci = nullptr;
    double* Lv = nullptr;
    int* Lrow = nullptr;    // local row id (0..nown-1) | diag slot << kRowBits, -1 padding
    double* diag = nullptr; // [nown]
    int* bd = nullptr;      // [nown] Dirichlet flags of the owned rows (extension x1)
    int nR = 0;             // owned rows of R_k (vertices of level k+1)
    int Rw = 0;
    int* Rci = nullptr;
    double* Rv = nullptr;
    int* Rrow = nullptr;    // local id at level k+1 (internal row of the shared level when k+1 is replicated)
    int* Pci = nullptr;     // owned fine rows of P_k, ELL-2; cols local at k+1 (or global)
    double* Pv = nullptr;
    int zero_diag_row = -1;
    std::vector<XPeer> peers;
    double* x[2] = {nullptr, nullptr};
    double* b = nullptr;
    double* r = nullptr;
    int cur = 0;
    bool x_zero = false;
};

struct DRank {
    int rank = 0;
    decmg_gpu_ctx* g = nullptr;  // full hierarchy (shared by all local ranks in emulation)
    std::vector<DLevel> lv;      // distributed levels 0 .. ka-1
    XPeer* gather_peers = nullptr;
    std::vector<XPeer> bpeers;   // all-gather plan of level ka (owned coarse entries)
    std::vector<XPeer> xpeers;   // all-gather plan of level 0 (solution)
    double* red = nullptr;
    double* dsum = nullptr;      // per-rank partial sums [nrhs]
};

}  // namespace
}  // namespace decmg_gpu

struct decmg_gpu_dist {
    int world = 1, ka = 0, L = 0, max_nrhs = 1;
    bool emulate = true;
    ncclComm_t comm = nullptr;
    std::vector<decmg_gpu::DRank> ranks;  // local ranks (emulation: all; NCCL: one)
    std::unique_ptr<decmg_gpu_ctx, void (*)(decmg_gpu_ctx*)> g{nullptr, nullptr};
    std::string err;
    std::vector<void*> allocs;
    double* hsum = nullptr;               // pinned [world][32]
    float last_cycle_ms = 0.f;            // device time of the last run's cycle loop
    cudaEvent_t ev[2] = {nullptr, nullptr};
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
// colmap (-1 entries are a bug: every referenced column is owned or halo).
// Same layout as setup.cu k_ell_fill: padding entries are a real column with
// value 0.0 (the row's diagonal column for L, diag = true; its first column
// otherwise) and the row id carries the diagonal slot above kRowBits.
Status build_local_ell(decmg_gpu_dist* D, const HostCSR& A, const std::vector<int>& rows, const std::vector<int>& rowid,
                       const std::vector<int>& colmap, int W, bool diag, int** eci, double** ev, int** erow) {
    const size_t npad = (rows.size() + 223) / 224 * 224;
    std::vector<int> ci(npad * W, -1), rid(npad, -1);
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
    DG_TRY(upload(D, eci, ci));
    DG_TRY(upload(D, ev, v));
    if (erow) DG_TRY(upload(D, erow, rid));
    return Status::Ok();
}

int maxlen(const HostCSR& A) {
    int m = 0;
    for (size_t i = 0; i + 1 < A.rp.size(); ++i) m = std::max(m, A.rp[i + 1] - A.rp[i]);
    return m;
}

Status build_dist(decmg_gpu_dist* D, int agglomerate) {
    decmg_gpu_ctx* g = D->g.get();
    const int L = static_cast<int>(g->lv.size());
    const int N = D->world;
    D->L = L;
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
    for (int k = 0; k < L; ++k)
        if (!g->lv[k].pos) return Status::Err(DECMG_INVALID_ARGUMENT, "dist: hierarchy needs positions");

    // ownership by Morton key thresholds of the finest level
    double lo[3], sc[3];
    DG_TRY(level_bbox(g, g->lv[0], lo, sc));
    std::vector<std::vector<int>> owner(ka + 1), order(ka + 1);
    std::vector<unsigned long long> split(N, 0);
    for (int k = 0; k <= ka; ++k) {
        const Level& m = g->lv[k];
        unsigned long long* dk;
        DG_CUDA(cudaMalloc(&dk, sizeof(unsigned long long) * m.nv));
        Status s = morton_keys(g, m, lo, sc, dk, nullptr);
        std::vector<unsigned long long> key;
        if (s.ok()) s = download(dk, m.nv, &key);
        cudaFree(dk);
        DG_TRY(s);
        if (k == 0) {
            std::vector<int> ord;
            if (m.ord) {
                DG_TRY(download(m.ord, m.nv, &ord));
            } else {
                ord.resize(m.nv);
                std::iota(ord.begin(), ord.end(), 0);
                std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key[a] < key[b]; });
            }
            for (int p = 1; p < N; ++p) split[p] = key[ord[static_cast<size_t>(m.nv) * p / N]];
        }
        owner[k].resize(m.nv);
        for (int v = 0; v < m.nv; ++v) {
            int p = 0;
            while (p + 1 < N && split[p + 1] <= key[v]) ++p;
            owner[k][v] = p;
        }
        if (m.ord) {
            DG_TRY(download(m.ord, m.nv, &order[k]));
        } else {
            order[k].resize(m.nv);
            std::iota(order[k].begin(), order[k].end(), 0);
        }
    }
    // the replicated levels (>= ka) run on the shared hierarchy in its internal
    // numbering (common.cuh Level::ord): global ids of level ka map through inv
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
    // owned lists (Morton order of the level) and halo sets for every rank
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
            std::sort(H.begin(), H.end());
        }
    }
    // per local rank: local numbering, operators, exchange plans
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
            // L rows
            std::vector<int> lrow(d.nown);
            std::iota(lrow.begin(), lrow.end(), 0);
            const int lm = maxlen(Lh[k]);
            d.Lw = lm <= 7 ? 7 : 8;
            if (lm > 8) return Status::Err(DECMG_RUNTIME, "dist: vertex valence above 7 is not supported");
            DG_TRY(build_local_ell(D, Lh[k], own[k][p], lrow, g2l[k], d.Lw, true, &d.Lci, &d.Lv, &d.Lrow));
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
            // R rows: owned level-(k+1) vertices
            const bool next_dist = k + 1 < ka;
            std::vector<int> rrow;
            for (int u : own[k + 1][p]) rrow.push_back(next_dist ? -2 : inv_ka[u]);  // filled below when distributed
            d.nR = static_cast<int>(own[k + 1][p].size());
            if (next_dist)
                for (int q = 0; q < d.nR; ++q) rrow[q] = q;  // owned rows come first in the local numbering
            const int rm = maxlen(Rh[k]);
            d.Rw = rm <= 7 ? 7 : 8;
            if (rm > 8) return Status::Err(DECMG_RUNTIME, "dist: restriction row longer than 8");
            DG_TRY(build_local_ell(D, Rh[k], own[k + 1][p], rrow, g2l[k], d.Rw, false, &d.Rci, &d.Rv, &d.Rrow));
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
            DG_TRY(build_local_ell(D, Ph[k], own[k][p], lrow, pmap, 2, false, &d.Pci, &d.Pv, nullptr));
            // halo exchange plan of level k
            for (int q = 0; q < N; ++q) {
                if (q == p) continue;
                XPeer x;
                x.rank = q;
                std::vector<int> s, r;
                for (int v : halo[k][q])
                    if (owner[k][v] == p) s.push_back(g2l[k][v]);
                for (int v : halo[k][p])
                    if (owner[k][v] == q) r.push_back(g2l[k][v]);
                if (s.empty() && r.empty()) continue;
                x.nsend = static_cast<int>(s.size());
                x.nrecv = static_cast<int>(r.size());
                DG_TRY(upload(D, &x.d_send, s));
                DG_TRY(upload(D, &x.d_recv, r));
                DG_TRY(dmalloc(D, &x.sbuf, static_cast<size_t>(x.nsend) * D->max_nrhs));
                DG_TRY(dmalloc(D, &x.rbuf, static_cast<size_t>(x.nrecv) * D->max_nrhs));
                d.peers.push_back(x);
            }
            const size_t nv = static_cast<size_t>(d.nloc) * D->max_nrhs;
            DG_TRY(dmalloc(D, &d.x[0], nv));
            DG_TRY(dmalloc(D, &d.x[1], nv));
            DG_TRY(dmalloc(D, &d.b, nv));
            DG_TRY(dmalloc(D, &d.r, nv));
        }
        // all-gather plans: level ka (restricted RHS) and level 0 (solution),
        // global-id slots, owned entries to every other rank
        // (slots: internal rows at level ka, reference ids at level 0)
        auto allgather_plan = [&](int k, std::vector<XPeer>* peers) -> Status {
            auto slots = [&](int r) {
                std::vector<int> v = own[k][r];
                if (k == ka)
                    for (int& u : v) u = inv_ka[u];
                return v;
            };
            for (int q = 0; q < N; ++q) {
                if (q == p) continue;
                XPeer x;
                x.rank = q;
                x.nsend = static_cast<int>(own[k][p].size());
                x.nrecv = static_cast<int>(own[k][q].size());
                DG_TRY(upload(D, &x.d_send, slots(p)));
                DG_TRY(upload(D, &x.d_recv, slots(q)));
                DG_TRY(dmalloc(D, &x.sbuf, static_cast<size_t>(x.nsend) * D->max_nrhs));
                DG_TRY(dmalloc(D, &x.rbuf, static_cast<size_t>(x.nrecv) * D->max_nrhs));
                peers->push_back(x);
            }
            return Status::Ok();
        };
        DG_TRY(allgather_plan(ka, &R.bpeers));
        DG_TRY(allgather_plan(0, &R.xpeers));
        DG_TRY(dmalloc(D, &R.red, g->red_cap + static_cast<size_t>(N) * 32));
        DG_TRY(dmalloc(D, &R.dsum, 64));
    }
    DG_CUDA(cudaMallocHost(&D->hsum, sizeof(double) * 32 * std::max(N, 1) + 64));
    return Status::Ok();
}

// --------------------------------------------------------------- driver ----
struct DistDriver {
    decmg_gpu_dist* D;
    int nrhs;
    std::vector<Driver> drv;  // one single-GPU driver per local rank (replicated levels + launches)

    decmg_gpu_ctx* g() const { return D->g.get(); }
    cudaStream_t stream() const { return g()->stream; }
    unsigned grid(int64_t t) const { return grid_for(t, 256); }

    // Exchange halo (or all-gather) values of one vector on every local rank.
    template <class Sel>
    Status exchange(Sel peers_of, std::function<double*(DRank&)> vec_of) {
        // pack
        for (DRank& R : D->ranks)
            for (XPeer& x : *peers_of(R))
                if (x.nsend) {
                    double* v = vec_of(R);
                    DG_TRY(launch(g(), 6, 0.0, [&] {
                        k_pack<<<grid(static_cast<int64_t>(x.nsend) * nrhs), 256, 0, stream()>>>(x.nsend, nrhs,
                                                                                                  x.d_send, v, x.sbuf);
                    }));
                }
        if (D->emulate) {
            for (DRank& R : D->ranks)
                for (XPeer& x : *peers_of(R)) {
                    if (!x.nrecv) continue;
                    DRank& Q = D->ranks[x.rank];
                    XPeer* src = nullptr;
                    for (XPeer& y : *peers_of(Q))
                        if (y.rank == R.rank) src = &y;
                    if (!src || src->nsend != x.nrecv) return Status::Err(DECMG_RUNTIME, "dist: inconsistent plan");
                    DG_CUDA(cudaMemcpyAsync(x.rbuf, src->sbuf, sizeof(double) * x.nrecv * nrhs,
                                            cudaMemcpyDeviceToDevice, stream()));
                }
        } else {
            DG_NCCL(ncclGroupStart());
            for (DRank& R : D->ranks)
                for (XPeer& x : *peers_of(R)) {
                    if (x.nsend) DG_NCCL(ncclSend(x.sbuf, static_cast<size_t>(x.nsend) * nrhs, ncclDouble, x.rank,
                                                  D->comm, stream()));
                    if (x.nrecv) DG_NCCL(ncclRecv(x.rbuf, static_cast<size_t>(x.nrecv) * nrhs, ncclDouble, x.rank,
                                                  D->comm, stream()));
                }
            DG_NCCL(ncclGroupEnd());
        }
        for (DRank& R : D->ranks)
            for (XPeer& x : *peers_of(R))
                if (x.nrecv) {
                    double* v = vec_of(R);
                    DG_TRY(launch(g(), 6, 0.0, [&] {
                        k_unpack<<<grid(static_cast<int64_t>(x.nrecv) * nrhs), 256, 0, stream()>>>(x.nrecv, nrhs,
                                                                                                    x.d_recv, x.rbuf, v);
                    }));
                }
        return Status::Ok();
    }

    Status halo_x(int k) {
        return exchange([k](DRank& R) { return &R.lv[k].peers; },
                        [k](DRank& R) { return R.lv[k].x[R.lv[k].cur]; });
    }
    Status halo_r(int k) {
        return exchange([k](DRank& R) { return &R.lv[k].peers; }, [k](DRank& R) { return R.lv[k].r; });
    }

    Status ensure_x(DRank& R, int k) {
        DLevel& d = R.lv[k];
        if (d.x_zero) {
            DG_CUDA(cudaMemsetAsync(d.x[d.cur], 0, sizeof(double) * d.nloc * nrhs, stream()));
            d.x_zero = false;
        }
        return Status::Ok();
    }

    Status smooth(int k, int iters, const Plan& plan) {
        if (iters <= 0) return Status::Ok();
        if (k >= D->ka) {
            DG_TRY(drv[0].smooth(k, iters, plan));  // replicated: one full copy per process
            return Status::Ok();
        }
        for (DRank& R : D->ranks)
            if (R.lv[k].zero_diag_row >= 0)
                return Status::Err(DECMG_RUNTIME,
                                   "jacobi: zero diagonal at row " + std::to_string(R.lv[k].zero_diag_row));
        for (int it = 0; it < iters; ++it) {
            const bool zero = D->ranks[0].lv[k].x_zero;
            if (!zero) DG_TRY(halo_x(k));
            for (size_t i = 0; i < D->ranks.size(); ++i) {
                DRank& R = D->ranks[i];
                DLevel& d = R.lv[k];
                double* xo = d.x[d.cur ^ 1];
                if (zero) {
                    const double bytes = 8.0 * d.nown + 16.0 * d.nown * nrhs;
                    Driver& dr = drv[i];
                    DG_TRY(launch(g(), 7, bytes, [&] {
                        DISPATCH_BP(dr.key, k_sweep_zero<BP, RPT><<<dr.rows_grid(d.nown), 256, 0, stream()>>>(
                                                d.nown, nrhs, d.diag, d.b, xo, plan.omega));
                    }));
                } else {
                    const double bytes = 12.0 * (7.0 * d.nown) + 4.0 * d.nown + 24.0 * d.nown * nrhs;
                    DG_TRY(drv[i].pipe_w<OP_SWEEP>(d.Lw, k == 0 ? 0 : 4, bytes, d.nown, d.Lci, d.Lv, d.Lrow,
                                         d.x[d.cur], d.b, xo, nullptr, nullptr, plan.omega, nullptr));
                }
                d.cur ^= 1;
                d.x_zero = false;
            }
        }
        return Status::Ok();
    }

    // r = b - A x on level k (owned rows), then b_{k+1} = R r on the owned coarse rows
    Status residual_restrict(int k) {
        if (k >= D->ka) {
            DG_TRY(drv[0].residual_restrict(k));
            return Status::Ok();
        }
        for (DRank& R : D->ranks) DG_TRY(ensure_x(R, k));
        DG_TRY(halo_x(k));
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DLevel& d = D->ranks[i].lv[k];
            DG_TRY(drv[i].pipe_w<OP_RES_STORE>(d.Lw, k == 0 ? 1 : 4, 0.0, d.nown, d.Lci, d.Lv, d.Lrow, d.x[d.cur],
                                 d.b, d.r, nullptr, nullptr, 0.0, nullptr));
        }
        DG_TRY(halo_r(k));
        const bool next_dist = k + 1 < D->ka;
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DRank& R = D->ranks[i];
            DLevel& d = R.lv[k];
            double* out = next_dist ? R.lv[k + 1].b : g()->lv[k + 1].b;
            const int* zr = nullptr;
            if (g()->dirichlet) zr = next_dist ? R.lv[k + 1].bd : g()->lv[k + 1].bd_i;
            DG_TRY(drv[i].pipe_w<OP_SPMV>(d.Rw, k == 0 ? 2 : 4, 0.0, d.nR, d.Rci, d.Rv, d.Rrow, d.r, nullptr, out,
                                 nullptr, zr, 0.0, nullptr));
        }
        if (!next_dist) {  // all-gather the owned entries of b_ka
            DG_TRY(exchange([](DRank& R) { return &R.bpeers; }, [this](DRank&) { return g()->lv[D->ka].b; }));
        }
        return Status::Ok();
    }

    // x_k += P_k x_{k+1} on the owned fine rows
    Status prolong(int k) {
        if (k >= D->ka) {
            DG_TRY(drv[0].prolong(k));
            return Status::Ok();
        }
        const bool next_dist = k + 1 < D->ka;
        if (next_dist) {
            for (DRank& R : D->ranks) DG_TRY(ensure_x(R, k + 1));
            DG_TRY(halo_x(k + 1));
        } else {
            DG_TRY(drv[0].ensure_x(k + 1));
        }
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DRank& R = D->ranks[i];
            DG_TRY(ensure_x(R, k));
            DLevel& d = R.lv[k];
            const double* xc = next_dist ? R.lv[k + 1].x[R.lv[k + 1].cur] : g()->lv[k + 1].x[g()->lv[k + 1].cur];
            DG_TRY((drv[i].pipe<OP_PROLONG, 2>(k == 0 ? 3 : 4, 0.0, d.nown, d.Pci, d.Pv, d.Lrow, xc, nullptr,
                                               d.x[d.cur], nullptr, nullptr, 0.0, nullptr)));
        }
        return Status::Ok();
    }

    Status cycle_once(const Plan& plan) {
        const int nw = static_cast<int>(plan.walk.size());
        const int L = D->L;
        int level = 0;
        for (int w = 0; w < nw; ++w) {
            if (plan.walk[w] == 'd') {
                DG_TRY(smooth(level, plan.pre[level], plan));
                DG_TRY(residual_restrict(level));
                ++level;
                if (level < D->ka) {
                    for (DRank& R : D->ranks) R.lv[level].x_zero = true;
                } else {
                    g()->lv[level].x_zero = true;
                }
                if (level == L - 1) {
                    DG_TRY(drv[0].coarse_solve(level));  // replicated (one shared hierarchy per process)
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

    // hist[lane] = ||b - A x|| / denom over all ranks' owned level-0 rows
    Status resnorm(double* h_out, const double* denom_host) {
        const int N = D->world;
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DRank& R = D->ranks[i];
            DG_TRY(ensure_x(R, 0));
        }
        DG_TRY(halo_x(0));
        for (size_t i = 0; i < D->ranks.size(); ++i) {
            DRank& R = D->ranks[i];
            DLevel& d = R.lv[0];
            int gsz = 0;
            double* save = g()->red;
            g()->red = R.red;  // Driver::reduce_partials folds in ctx->red
            Status s = drv[i].pipe_w<OP_RES_NORM>(d.Lw, 1, 0.0, d.nown, d.Lci, d.Lv, d.Lrow, d.x[d.cur], d.b,
                                     nullptr, R.red, nullptr, 0.0, &gsz);
            if (s.ok()) s = drv[i].reduce_partials(gsz, R.dsum, 0, nullptr);
            g()->red = save;
            DG_TRY(s);
        }
        // gather every rank's per-lane sums, add them in rank order
        std::vector<double> sums(static_cast<size_t>(N) * nrhs, 0.0);
        if (D->emulate) {
            for (DRank& R : D->ranks)
                DG_CUDA(cudaMemcpyAsync(D->hsum + static_cast<size_t>(R.rank) * nrhs, R.dsum, sizeof(double) * nrhs,
                                        cudaMemcpyDeviceToHost, stream()));
            DG_CUDA(cudaStreamSynchronize(stream()));
        } else {
            DRank& R = D->ranks[0];
            double* all = R.red;  // scratch [N][nrhs]
            DG_NCCL(ncclAllGather(R.dsum, all, nrhs, ncclDouble, D->comm, stream()));
            DG_CUDA(cudaMemcpyAsync(D->hsum, all, sizeof(double) * N * nrhs, cudaMemcpyDeviceToHost, stream()));
            DG_CUDA(cudaStreamSynchronize(stream()));
        }
        for (int l = 0; l < nrhs; ++l) {
            double t = 0.0;
            for (int p = 0; p < N; ++p) t += D->hsum[static_cast<size_t>(p) * nrhs + l];
            h_out[l] = std::sqrt(t) / denom_host[l];
        }
        return Status::Ok();
    }
};

}  // namespace

// Distributed run: b (full, projected or not) replicated on every rank.
Status dist_run(decmg_gpu_dist* D, const Plan& plan, int nrhs, const double* h_b, const double* h_x0, int ncycles,
                bool solve, double tol, double* h_x, double* h_hist, int* cycles_done, double* h_final) {
    decmg_gpu_ctx* g = D->g.get();
    if (nrhs < 1 || nrhs > D->max_nrhs) return Status::Err(DECMG_INVALID_ARGUMENT, "nrhs must be in [1, max_nrhs]");
    const int n0 = g->lv[0].nv;
    const size_t nb = sizeof(double) * n0 * nrhs;
    DistDriver dd{D, nrhs, {}};
    for (size_t i = 0; i < D->ranks.size(); ++i) {
        Driver dr{g, nrhs, bp_of(nrhs), g->io_b};
        dr.init();
        dd.drv.push_back(dr);
    }
    cudaStream_t st = g->stream;
    // full right-hand side on this process (replicated), projected like gmg_solve
    DG_CUDA(cudaMemcpyAsync(g->io_b, h_b, nb, cudaMemcpyHostToDevice, st));
    if (solve && !g->dirichlet) DG_TRY(project_compatible(g, nrhs, g->io_b));
    // denominator ||b|| (replicated computation on the full vector)
    Driver& d0 = dd.drv[0];
    DG_TRY(d0.make_denom(g->dsmall));
    std::vector<double> denom(nrhs);
    DG_CUDA(cudaMemcpyAsync(denom.data(), g->dsmall, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, st));
    if (h_x0) DG_CUDA(cudaMemcpyAsync(g->io_x0, h_x0, nb, cudaMemcpyHostToDevice, st));
    for (DRank& R : D->ranks) {
        DLevel& d = R.lv[0];
        DG_TRY(launch(g, 6, 0.0, [&] {
            k_gather_rows<<<grid_for(static_cast<int64_t>(d.nown) * nrhs, 256), 256, 0, st>>>(d.nown, nrhs, d.d_own,
                                                                                              g->io_b, d.b);
        }));
        d.cur = 0;
        if (h_x0) {
            DG_TRY(launch(g, 6, 0.0, [&] {
                k_gather_rows<<<grid_for(static_cast<int64_t>(d.nown) * nrhs, 256), 256, 0, st>>>(
                    d.nown, nrhs, d.d_own, g->io_x0, d.x[0]);
            }));
            d.x_zero = false;
        } else {
            d.x_zero = true;
        }
    }
    DG_CUDA(cudaStreamSynchronize(st));
    const int maxc = ncycles;
    std::vector<double> hist(nrhs);
    std::vector<int> done(nrhs, 0);
    std::vector<double> fin(nrhs, 0.0);
    unsigned active = nrhs == 32 ? 0xffffffffu : ((1u << nrhs) - 1u);
    int cyc = 0;
    // snapshot of converged lanes: gather owned rows of lanes in `mask` into g->xsol (full numbering)
    auto snapshot = [&](unsigned mask) -> Status {
        for (DRank& R : D->ranks) {
            DLevel& d = R.lv[0];
            DG_TRY(dd.ensure_x(R, 0));
            // scatter owned rows into a full-size buffer, then copy the selected lanes
            DG_TRY(launch(g, 6, 0.0, [&] {
                k_scatter_rows<<<grid_for(static_cast<int64_t>(d.nown) * nrhs, 256), 256, 0, st>>>(
                    d.nown, nrhs, d.d_own, d.x[d.cur], g->io_x);
            }));
        }
        if (!D->emulate)
            DG_TRY(dd.exchange([](DRank& R) { return &R.xpeers; }, [g](DRank&) { return g->io_x; }));
        const int64_t total = static_cast<int64_t>(n0) * nrhs;
        DG_TRY(launch(g, 6, 0.0, [&] {
            k_copy_lanes<<<grid_for(total, 256), 256, 0, st>>>(total, nrhs, mask, g->io_x, g->xsol);
        }));
        return Status::Ok();
    };
    if (!D->ev[0]) {
        DG_CUDA(cudaEventCreate(&D->ev[0]));
        DG_CUDA(cudaEventCreate(&D->ev[1]));
    }
    DG_CUDA(cudaEventRecord(D->ev[0], st));
    while (cyc < maxc && active) {
        DG_TRY(dd.cycle_once(plan));
        ++cyc;
        DG_TRY(dd.resnorm(hist.data(), denom.data()));
        unsigned finm = 0;
        for (int l = 0; l < nrhs; ++l) {
            if (!(active & (1u << l))) continue;
            if (h_hist) h_hist[static_cast<int64_t>(cyc - 1) * nrhs + l] = hist[l];
            fin[l] = hist[l];
            done[l] = cyc;
            if (solve && (hist[l] <= tol || cyc == maxc)) finm |= 1u << l;
        }
        if (finm) {
            DG_TRY(snapshot(finm));
            active &= ~finm;
        }
    }
    DG_CUDA(cudaEventRecord(D->ev[1], st));
    DG_CUDA(cudaEventSynchronize(D->ev[1]));
    DG_CUDA(cudaEventElapsedTime(&D->last_cycle_ms, D->ev[0], D->ev[1]));
    if (active) DG_TRY(snapshot(active));
    DG_CUDA(cudaMemcpyAsync(h_x, g->xsol, nb, cudaMemcpyDeviceToHost, st));
    DG_CUDA(cudaStreamSynchronize(st));
    for (int l = 0; l < nrhs; ++l) {
        if (cycles_done) cycles_done[l] = done[l];
        if (h_final) h_final[l] = fin[l];
    }
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

int decmg_gpu_dist_create(const double* positions, int nv, const int* corner_triples, int nt, int nsub,
                          unsigned flags, const decmg_gpu_config* cfg, int world_size, int rank,
                          const void* nccl_id, int agglomerate_below, decmg_gpu_dist** out) {
    if (!out || world_size < 1 || rank < -1 || rank >= world_size) return DECMG_INVALID_ARGUMENT;
    *out = nullptr;
    auto* D = new decmg_gpu_dist();
    D->world = world_size;
    D->emulate = nccl_id == nullptr;
    if (D->emulate) {
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
    if (s.ok() && !D->emulate) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof id);
        cudaSetDevice(cfg ? cfg->device : 0);
        if (ncclCommInitRank(&D->comm, world_size, id, rank) != ncclSuccess)
            s = Status::Err(DECMG_NCCL, "ncclCommInitRank failed");
    }
    for (DRank& R : D->ranks) R.g = D->g.get();
    if (!s.ok()) {
        decmg_gpu_dist_destroy(D);
        g_dist_create_error = s.msg;
        return s.code;
    }
    *out = D;
    return DECMG_OK;
}

void decmg_gpu_dist_destroy(decmg_gpu_dist* D) {
    if (!D) return;
    if (D->g) cudaStreamSynchronize(D->g->stream);
    if (D->comm) ncclCommDestroy(D->comm);
    for (cudaEvent_t e : D->ev)
        if (e) cudaEventDestroy(e);
    for (void* p : D->allocs) cudaFree(p);
    if (D->hsum) cudaFreeHost(D->hsum);
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
    if (s.ok()) s = dist_run(D, p, nrhs, b, x0, max_cycles, solve != 0, tol, x_out, hist_out, cycles_done, final_out);
    if (!s.ok()) {
        D->err = s.msg;
        return s.code;
    }
    return DECMG_OK;
}

}  // extern "C"
