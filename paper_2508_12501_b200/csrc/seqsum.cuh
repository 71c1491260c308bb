// Exact parallel evaluation of a sequential fp64 sum.
//
// project_compatible (proj/src/multigrid.cpp:240-250) computes
//     mean = 0.0; for i ascending: mean += w[i] * b[i];
// A constant offset in b is invisible to the V-cycle, so the last bit of this
// mean shows up as a permanent residual floor: the device must reproduce the
// chain s_{i+1} = fl(s_i + p_i) bit for bit. Run literally it
// is a 10.5 M-long dependent DADD chain per right-hand side (~75 ms at config 4,
// the largest item of a host-to-host gmg_solve). This file evaluates the same
// chain exactly, in parallel.
//
// Idea. While the running sum s stays in one binade [2^e, 2^(e+1)) with one
// sign, every double there is an integer multiple m of u = 2^(e-52), with m in
// [2^52, 2^53). Adding p then rounds on that fixed grid:
//     fl(s + p) = sgn * u * RNE(m + x),   x = sgn * p / u   (exact: a shift),
// provided the result stays inside the binade. RNE(m + x) = m + q where q is
// x rounded to an integer, except when x is exactly halfway (ties to even):
// then q depends on the parity of m. So each element acts on m as a
// translation by d[m & 1], and a segment of elements composes into the same
// form (total offsets d[par], plus the minimum and maximum intermediate offsets
// mn[par], mx[par] to check that no intermediate result leaves the binade).
// Composition is associative, so a segment's function is a parallel reduction.
//
// Algorithm over rows [r0, r1), records of kRecRows = 32 rows:
//   1. k_seq_prod:  p = w * b (the reference's __dmul_rn), stored; approximate
//                   record sums (any order) -- only used to guess binades.
//   2. k_seq_guess: exclusive scan of the approximate sums from the exact
//                   running state -> a guessed start value per record, whose
//                   binade (e, sign) is the speculation.
//   3. k_seq_fn:    each record's function in its guessed binade.
//   4. k_seq_walk:  one warp per right-hand side walks the records with the
//                   EXACT running sum: if s lies in the guessed binade and
//                   m + mn >= 2^52 + 1, m + mx <= 2^53 - 1 for its parity, a
//                   record (or a composed run of up to 32 records sharing a
//                   binade) is applied in O(1) -- the result is exactly what
//                   the element-by-element chain gives; otherwise (zero
//                   crossing, binade change, wrong guess, inf/nan, huge terms)
//                   it runs the literal __dadd_rn chain over that record.
// The guesses only decide which records take the fast path; the result is
// the sequential chain's in every case. tools/seqsum_proto.c is the host
// model of the same decomposition (checked against the plain loop on random,
// tie-heavy, wide-range and signed-zero inputs); tests/test_gpu_parity.py checks
// the device result against the oracle's sequential projection.
#pragma once

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "ptx.cuh"

namespace decmg_gpu {

constexpr int kRecRows = 32;                           // rows per record (one binade guess each)
constexpr int kGrpRecs = 32;                           // records per group (one tree of 63 nodes)
constexpr int kGrpRows = kRecRows * kGrpRecs;          // 1024
constexpr int kGrpNodes = 63;
constexpr int kTileRows = 256;                         // rows per block of k_seq_prod
constexpr int kTileRecs = kTileRows / kRecRows;        // 8
constexpr int kSeqPassRows = 1 << 20;                  // rows per pass (bounds the scratch)
constexpr int kSeqPassRecs = kSeqPassRows / kRecRows;  // 32768
constexpr int kSeqPassGrps = kSeqPassRows / kGrpRows;  // 1024
constexpr long long kSeqLo = (1ll << 52) + 1, kSeqHi = (1ll << 53) - 1;
constexpr long long kSeqBig = 1ll << 62;
constexpr long long kTagNone = -1, kTagAny = -2;  // no fast path / padding (identity)

// record function m -> m + d[m & 1]; mn/mx: extreme intermediate offsets
struct SegFn {
    long long d0, d1, mn0, mn1, mx0, mx1;
};
// A tree node in the walk's form: for the parity of the running sum's last
// mantissa bit, the fast path holds iff lo <= s <= hi, and then
// fl(s + p_first) ... = s + D exactly (one exact DADD). Never: lo = +inf;
// padding: lo = -inf, hi = +inf, D = -0.0 (s + -0.0 == s for every s).
struct SeqNode {
    double lo0, hi0, d0, lo1, hi1, d1;
};
static_assert(sizeof(SeqNode) * kGrpNodes % 16 == 0, "node blocks must be bulk-copyable");

__device__ __forceinline__ SegFn seg_ident() { return SegFn{0, 0, kSeqBig, kSeqBig, -kSeqBig, -kSeqBig}; }

// f then one element with offsets (e0 for even m, e1 for odd m)
__device__ __forceinline__ void seg_push(SegFn& f, long long e0, long long e1) {
    const long long a = (f.d0 & 1) ? e1 : e0;  // parity after f, start even
    const long long b = ((1 + f.d1) & 1) ? e1 : e0;
    f.d0 += a;
    f.d1 += b;
    f.mn0 = min(f.mn0, f.d0);
    f.mx0 = max(f.mx0, f.d0);
    f.mn1 = min(f.mn1, f.d1);
    f.mx1 = max(f.mx1, f.d1);
}

// f then g
__device__ __forceinline__ SegFn seg_compose(const SegFn& f, const SegFn& g) {
    SegFn h;
    const bool o0 = (f.d0 & 1) != 0, o1 = ((1 + f.d1) & 1) != 0;
    h.d0 = f.d0 + (o0 ? g.d1 : g.d0);
    h.mn0 = min(f.mn0, f.d0 + (o0 ? g.mn1 : g.mn0));
    h.mx0 = max(f.mx0, f.d0 + (o0 ? g.mx1 : g.mx0));
    h.d1 = f.d1 + (o1 ? g.d1 : g.d0);
    h.mn1 = min(f.mn1, f.d1 + (o1 ? g.mn1 : g.mn0));
    h.mx1 = max(f.mx1, f.d1 + (o1 ? g.mx1 : g.mx0));
    return h;
}

__device__ __forceinline__ long long tag_join(long long a, long long b) {
    if (a == kTagAny) return b;
    if (b == kTagAny) return a;
    return a == b ? a : kTagNone;
}

__device__ __forceinline__ SegFn seg_shfl_down(const SegFn& f, int o) {
    SegFn g;
    g.d0 = __shfl_down_sync(0xffffffffu, f.d0, o);
    g.d1 = __shfl_down_sync(0xffffffffu, f.d1, o);
    g.mn0 = __shfl_down_sync(0xffffffffu, f.mn0, o);
    g.mn1 = __shfl_down_sync(0xffffffffu, f.mn1, o);
    g.mx0 = __shfl_down_sync(0xffffffffu, f.mx0, o);
    g.mx1 = __shfl_down_sync(0xffffffffu, f.mx1, o);
    return g;
}

// Offsets of one element p on the grid of binade e (unbiased) with the sum's
// sign neg. Returns false when the element cannot take the fast path.
__device__ __forceinline__ bool seg_elem(double p, int e, bool neg, long long& e0, long long& e1) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(p));
    const int E = static_cast<int>((bits >> 52) & 0x7ff);
    unsigned long long M = bits & ((1ull << 52) - 1);
    if (E == 0x7ff) return false;
    e0 = e1 = 0;
    if (E == 0 && M == 0) return true;  // +-0.0: s + 0 = s (s != 0)
    int ex;
    if (E == 0) {
        ex = -1074;
    } else {
        M |= 1ull << 52;
        ex = E - 1075;
    }
    const bool xneg = ((bits >> 63) != 0) != neg;  // sign of x = sgn(s) * p / u
    const int k = ex - (e - 52);                   // |x| = M * 2^k
    if (k >= 0) {
        if (k >= 11 || (M << k) >= (1ull << 52)) return false;
        const long long q = static_cast<long long>(M << k);
        e0 = e1 = xneg ? -q : q;
        return true;
    }
    const int sh = -k;
    if (sh >= 54) return true;  // |x| < 1/2, never a tie
    const unsigned long long ip = M >> sh, rem = M & ((1ull << sh) - 1), half = 1ull << (sh - 1);
    if (rem == half) {  // tie: the result is whichever of m+a, m+a+1 is even
        const long long a = xneg ? -static_cast<long long>(ip) - 1 : static_cast<long long>(ip);
        e0 = a + (a & 1);
        e1 = a + ((1 + a) & 1);
    } else {
        const long long q = static_cast<long long>(ip) + (rem > half ? 1 : 0);
        e0 = e1 = xneg ? -q : q;
    }
    return true;
}

// 1. products p = w * b (kept for steps 3-4, lane-major: prodT[l * stride +
// row - r0]) and approximate record sums. grid = 256-row tiles of the pass,
// block = 256, dynamic smem = kTileRows*(nrhs+1) doubles.
__global__ void __launch_bounds__(256) k_seq_prod(int r0, int r1, int nrhs, int stride, const double* __restrict__ w,
                                                  const double* __restrict__ b, double* __restrict__ prodT,
                                                  double* __restrict__ approx) {
    extern __shared__ double tile[];  // [kTileRows][nrhs + 1]
    const int j = blockIdx.x;
    const int row0 = r0 + j * kTileRows;
    const int rows = min(kTileRows, r1 - row0);
    const int64_t base = static_cast<int64_t>(row0) * nrhs;
    const int cnt = rows * nrhs;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        const int row = q / nrhs, l = q - row * nrhs;
        tile[row * (nrhs + 1) + l] = __dmul_rn(__ldcs(w + row0 + row), __ldcs(b + base + q));
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    for (int l = warp; l < nrhs; l += blockDim.x >> 5) {
        double* dst = prodT + static_cast<int64_t>(l) * stride + (row0 - r0);
        for (int row = t; row < rows; row += 32) __stcs(dst + row, tile[row * (nrhs + 1) + l]);
        double s = 0.0;
        for (int i = 0; i < 8; ++i) {
            const int row = t * 8 + i;
            if (row < rows) s += tile[row * (nrhs + 1) + l];
        }
        s += __shfl_down_sync(0xffffffffu, s, 1);
        s += __shfl_down_sync(0xffffffffu, s, 2);
        const int rec = j * kTileRecs + (t >> 2);
        if ((t & 3) == 0 && t * 8 < rows) approx[static_cast<int64_t>(l) * kSeqPassRecs + rec] = s;
    }
}

// 2. guessed start of every record: exact state + exclusive scan of the
// approximate sums. grid = nrhs blocks of 1024 threads, 32 records per thread.
__global__ void __launch_bounds__(1024) k_seq_guess(int nrec, const double* __restrict__ approx,
                                                    const double* __restrict__ state, double* __restrict__ guess) {
    using Scan = cub::BlockScan<double, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    constexpr int kPer = kSeqPassRecs / 1024;
    static_assert(kPer * 1024 == kSeqPassRecs, "pass records");
    const int l = blockIdx.x, t = threadIdx.x;
    const double* a = approx + static_cast<int64_t>(l) * kSeqPassRecs + t * kPer;
    double* g = guess + static_cast<int64_t>(l) * kSeqPassRecs + t * kPer;
    double acc = 0.0;
    for (int i = 0; i < kPer; ++i)
        if (t * kPer + i < nrec) acc += a[i];
    double pre;
    Scan(tmp).ExclusiveSum(acc, pre);
    double v = state[l] + pre;
    for (int i = 0; i < kPer; ++i) {
        if (t * kPer + i >= nrec) break;
        g[i] = v;
        v += a[i];
    }
}

// A composed function with its binade tag in the walk's node form.
__device__ __forceinline__ SeqNode node_make(const SegFn& f, long long tag) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    if (tag == kTagAny) return SeqNode{-inf, inf, -0.0, -inf, inf, -0.0};
    const SeqNode never{inf, -inf, 0.0, inf, -inf, 0.0};
    if (tag < 0) return never;
    const int E = static_cast<int>(tag & 2047);  // biased exponent of the binade
    if (E < 124) return never;                   // keep u = 2^(e-52) and m*u normal
    const bool neg = (tag & 2048) != 0;
    const double u = __longlong_as_double(static_cast<long long>(E - 52) << 52);
    SeqNode n;
    const long long mn[2] = {f.mn0, f.mn1}, mx[2] = {f.mx0, f.mx1}, d[2] = {f.d0, f.d1};
    double lo[2], hi[2], dd[2];
    for (int p = 0; p < 2; ++p) {
        const long long mlo = max(1ll << 52, kSeqLo - mn[p]), mhi = min(kSeqHi, kSeqHi - mx[p]);
        if (mlo > mhi) {
            lo[p] = inf;
            hi[p] = -inf;
            dd[p] = 0.0;
        } else {  // m in [mlo, mhi]: |d| < 2^53, every product below is exact
            const double a = __dmul_rn(static_cast<double>(mlo), u), b = __dmul_rn(static_cast<double>(mhi), u);
            const double dv = __dmul_rn(static_cast<double>(d[p]), u);
            lo[p] = neg ? -b : a;
            hi[p] = neg ? -a : b;
            dd[p] = neg ? -dv : dv;
        }
    }
    n.lo0 = lo[0];
    n.hi0 = hi[0];
    n.d0 = dd[0];
    n.lo1 = lo[1];
    n.hi1 = hi[1];
    n.d1 = dd[1];
    return n;
}

// Streaming (evict-first) store of a node: the projection runs beside another
// batch's V-cycle (solve_batches), whose L2-resident data it must not displace.
__device__ __forceinline__ void st_node(SeqNode* p, const SeqNode& n) {
    __stcs(&p->lo0, n.lo0);
    __stcs(&p->hi0, n.hi0);
    __stcs(&p->d0, n.d0);
    __stcs(&p->lo1, n.lo1);
    __stcs(&p->hi1, n.hi1);
    __stcs(&p->d1, n.d1);
}

// 3. record functions in their guessed binades and each group's tree of
// compositions (nodes of 1, 2, 4, ..., 32 records; a node is usable when its
// records share one binade). grid = (groups of the pass, ceil(nrhs/4)),
// block = 128: warp w = lane blockIdx.y*4 + w; thread t = record t of the group.
__global__ void __launch_bounds__(128) k_seq_tree(int r0, int r1, int nrhs, int stride,
                                                  const double* __restrict__ prodT, const double* __restrict__ guess,
                                                  SeqNode* __restrict__ nodes) {
    __shared__ double tile[4][kGrpRecs * (kRecRows + 1)];
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    const int l = blockIdx.y * 4 + warp;
    if (l >= nrhs) return;
    const int g = blockIdx.x;
    const int row0 = g * kGrpRows;  // relative to r0
    const int rows = min(kGrpRows, r1 - r0 - row0);
    const double* src = prodT + static_cast<int64_t>(l) * stride + row0;
    double* tl = tile[warp];
    for (int i = t; i < rows; i += 32) tl[(i >> 5) * (kRecRows + 1) + (i & 31)] = __ldcs(src + i);
    __syncwarp();
    const int rec = g * kGrpRecs + t;
    const int rrows = min(kRecRows, rows - t * kRecRows);  // <= 0: padding record
    SegFn f = seg_ident();
    long long tag = kTagAny;
    if (rrows > 0) {
        const double gs = guess[static_cast<int64_t>(l) * kSeqPassRecs + rec];
        const unsigned long long gb = static_cast<unsigned long long>(__double_as_longlong(gs));
        const int gE = static_cast<int>((gb >> 52) & 0x7ff);
        const bool gneg = (gb >> 63) != 0;
        bool ok = gE != 0 && gE != 0x7ff;  // a normal, nonzero guess
        if (ok) {
            const int e = gE - 1023;
            for (int i = 0; i < rrows; ++i) {
                long long e0 = 0, e1 = 0;
                ok &= seg_elem(tl[t * (kRecRows + 1) + i], e, gneg, e0, e1);
                seg_push(f, e0, e1);
            }
        }
        constexpr long long kLim = 1ll << 53;  // a valid record moves m by less than 2^53
        ok &= f.mn0 > -kLim && f.mn1 > -kLim && f.mx0 < kLim && f.mx1 < kLim;
        tag = ok ? static_cast<long long>(gE | (gneg ? 2048 : 0)) : kTagNone;
        if (!ok) f = seg_ident();
    }
    SeqNode* out = nodes + (static_cast<int64_t>(l) * kSeqPassGrps + g) * kGrpNodes;
    st_node(out + t, node_make(f, tag));
    for (int lev = 1; lev <= 5; ++lev) {
        const int o = 1 << (lev - 1);
        const SegFn h = seg_shfl_down(f, o);
        const long long th = __shfl_down_sync(0xffffffffu, tag, o);
        if ((t & (2 * o - 1)) == 0) {
            tag = tag_join(tag, th);
            if (tag != kTagNone) f = seg_compose(f, h);
            st_node(out + (64 - (64 >> lev)) + (t >> lev), node_make(f, tag));
        }
    }
}

#ifdef SEQ_PROFILE  // tools/bench_seqwalk.cu: walk cycles (wait, tries, literal, #tries)
__device__ unsigned long long g_seq_prof[6];
#endif

// The fast path of node n on the exact running sum s: one exact add.
__device__ __forceinline__ bool node_apply(double& s, const SeqNode& n) {
    const bool odd = __double_as_longlong(s) & 1;
    const double lo = odd ? n.lo1 : n.lo0, hi = odd ? n.hi1 : n.hi0;
    if (!(s >= lo && s <= hi)) return false;
    s = __dadd_rn(s, odd ? n.d1 : n.d0);
    return true;
}

// 4. the exact walk: block l (one warp) = right-hand side l. Every thread
// carries the same running sum, so control flow is warp-uniform. Groups are
// walked in batches of 32 whose root nodes (the composition of the whole
// group) the warp loads one batch ahead; most groups are applied by their root
// in one step. A group whose root cannot apply -- predicted when the root is
// empty for both parities (its records straddle a binade or zero), or found
// when the exact sum misses its interval -- needs its 63-node tree and its
// 1024 products: predicted groups are prefetched with cp.async into
// kWalkSlots shared-memory slots as soon as their batch starts, others are
// fetched on demand into one more slot. Such a group is walked down its tree:
// from each aligned position the largest node is tried, halved on failure,
// and a single record whose fast path fails is chained literally (__dadd_rn in
// row order); after a success the walk climbs back to the largest aligned
// node, so only the records where the sum crosses a binade (or zero) run
// element by element.
constexpr int kWalkSlots = 3;
constexpr int kWalkNodeBytes = static_cast<int>(sizeof(SeqNode)) * kGrpNodes;  // 3024
constexpr int kWalkStageBytes = kWalkNodeBytes + 16 + kGrpRows * 8;           // nodes | pad | products
constexpr int kWalkSmem = (kWalkSlots + 1) * kWalkStageBytes + 32 * static_cast<int>(sizeof(SeqNode));

// mbarrier arrival when all of this thread's earlier cp.async copies have landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(32) k_seq_walk(int r0, int r1, int stride, const double* __restrict__ prodT,
                                                 const SeqNode* __restrict__ nodes, double* __restrict__ state,
                                                 double total, double* __restrict__ mean_out,
                                                 int* __restrict__ fallbacks) {
    extern __shared__ __align__(128) unsigned char walk_smem[];
    __shared__ __align__(8) uint64_t bar[kWalkSlots + 1];
    SeqNode* roots = reinterpret_cast<SeqNode*>(walk_smem + (kWalkSlots + 1) * kWalkStageBytes);
    const int l = blockIdx.x, t = threadIdx.x;
    const int nrows = r1 - r0;
    const int ngrp = (nrows + kGrpRows - 1) / kGrpRows;
    const SeqNode* lnode = nodes + static_cast<int64_t>(l) * kSeqPassGrps * kGrpNodes;
    const unsigned char* ln = reinterpret_cast<const unsigned char*>(lnode);
    const unsigned char* lp = reinterpret_cast<const unsigned char*>(prodT + static_cast<int64_t>(l) * stride);
    if (t == 0) {
        for (int i = 0; i <= kWalkSlots; ++i) mbar_init(&bar[i], 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned par = 0;  // phase parity per slot (bit i)
    // every thread copies its share of group g's nodes and products into slot
    // sl; the slot's barrier completes when all 32 threads' copies have landed
    auto fetch = [&](int g, int sl) {
        unsigned char* base = walk_smem + sl * kWalkStageBytes;
        const unsigned char* ns = ln + static_cast<int64_t>(g) * kWalkNodeBytes;
        for (int i = t; i < kWalkNodeBytes / 16; i += 32) cp_async16(base + 16 * i, ns + 16 * i);
        const int rows = min(kGrpRows, nrows - g * kGrpRows);
        const int nchunk = (rows + 1) >> 1;  // stride is even: 16-byte chunks stay inside the lane
        const unsigned char* ps = lp + static_cast<int64_t>(g) * kGrpRows * 8;
        unsigned char* pd = base + kWalkNodeBytes + 16;
        for (int i = t; i < nchunk; i += 32) cp_async16(pd + 16 * i, ps + 16 * i);
        cp_async_mbar_arrive(&bar[sl]);
    };
    auto wait_slot = [&](int sl) {
        mbar_wait(&bar[sl], (par >> sl) & 1u);
        par ^= 1u << sl;
        __syncwarp();
    };
    auto load_root = [&](int g, SeqNode& r) {
        if (g < ngrp) r = lnode[static_cast<int64_t>(g) * kGrpNodes + (kGrpNodes - 1)];
    };
    SeqNode rnext;
    load_root(t, rnext);
    double s = state[l];
    int nfb = 0;
#ifdef SEQ_PROFILE
    const long long c_start = clock64();
    long long pw = 0, pt = 0, pl = 0, ntry = 0, pi = 0;
#endif
    int slot_grp[kWalkSlots];
#pragma unroll
    for (int i = 0; i < kWalkSlots; ++i) slot_grp[i] = -1;
    for (int g0 = 0; g0 < ngrp; g0 += 32) {
        __syncwarp();
        roots[t] = rnext;
        __syncwarp();
        load_root(g0 + 32 + t, rnext);  // next batch, in flight during this one
        const double inf = __longlong_as_double(0x7ff0000000000000ll);
        const bool pred = g0 + t < ngrp && roots[t].lo0 == inf && roots[t].lo1 == inf;
        unsigned pend = __ballot_sync(0xffffffffu, pred);  // predicted crossings not yet prefetched
#pragma unroll
        for (int i = 0; i < kWalkSlots; ++i)
            if (pend) {
                const int g = g0 + __ffs(pend) - 1;
                pend &= pend - 1;
                fetch(g, i);
                slot_grp[i] = g;
            }
        const int jb = min(32, ngrp - g0);
        for (int k = 0; k < jb; ++k) {
            const int g = g0 + k;
#ifdef SEQ_PROFILE
            ++ntry;
#endif
            if (node_apply(s, roots[k])) continue;
            int sl = kWalkSlots;  // the demand slot unless prefetched
#pragma unroll
            for (int i = 0; i < kWalkSlots; ++i)
                if (slot_grp[i] == g) sl = i;
#ifdef SEQ_PROFILE
            const long long c0 = clock64();
#endif
            if (sl == kWalkSlots) fetch(g, sl);
            wait_slot(sl);
#ifdef SEQ_PROFILE
            pw += clock64() - c0;
#endif
            const SeqNode* nd = reinterpret_cast<const SeqNode*>(walk_smem + sl * kWalkStageBytes);
            const double* pr = reinterpret_cast<const double*>(walk_smem + sl * kWalkStageBytes + kWalkNodeBytes + 16);
            const int rows = min(kGrpRows, nrows - g * kGrpRows);
            const int jn = (rows + kRecRows - 1) / kRecRows;
            int pos = 0;
            while (pos < jn) {
                int lev = pos ? min(4, __ffs(pos) - 1) : 4;  // the root (level 5) already failed
                for (;;) {
#ifdef SEQ_PROFILE
                    ++ntry;
#endif
                    if (node_apply(s, nd[(64 - (64 >> lev)) + (pos >> lev)])) {
                        pos += 1 << lev;
                        break;
                    }
                    if (lev > 0) {
                        --lev;
                        continue;
                    }
                    ++nfb;  // the literal chain over record pos
#ifdef SEQ_PROFILE
                    const long long c3 = clock64();
#endif
                    const int rr = min(kRecRows, rows - pos * kRecRows);
                    const double* p = pr + pos * kRecRows;
                    if (rr == kRecRows) {  // full record: operands in registers first, then the add chain
                        double q[kRecRows];
#pragma unroll
                        for (int i = 0; i < kRecRows; ++i) q[i] = p[i];
#pragma unroll
                        for (int i = 0; i < kRecRows; ++i) s = __dadd_rn(s, q[i]);
                    } else {
                        for (int i = 0; i < rr; ++i) s = __dadd_rn(s, p[i]);
                    }
#ifdef SEQ_PROFILE
                    pl += clock64() - c3;
#endif
                    pos += 1;
                    break;
                }
            }
            __syncwarp();
            if (sl < kWalkSlots) {  // slot free: prefetch the batch's next predicted crossing
                slot_grp[sl] = -1;
                if (pend) {
                    const int g2 = g0 + __ffs(pend) - 1;
                    pend &= pend - 1;
                    fetch(g2, sl);
                    slot_grp[sl] = g2;
                }
            }
        }
        // prefetched groups whose root applied after all: retire their copies
#pragma unroll
        for (int i = 0; i < kWalkSlots; ++i)
            if (slot_grp[i] >= 0) {
                wait_slot(i);
                slot_grp[i] = -1;
            }
    }
    if (t == 0) {
        state[l] = s;
        if (mean_out) mean_out[l] = __ddiv_rn(s, total);
        if (fallbacks) atomicAdd(fallbacks, nfb);
#ifdef SEQ_PROFILE
        atomicAdd(&g_seq_prof[0], static_cast<unsigned long long>(pw));
        atomicAdd(&g_seq_prof[1], static_cast<unsigned long long>(pt));
        atomicAdd(&g_seq_prof[2], static_cast<unsigned long long>(pl));
        atomicAdd(&g_seq_prof[3], static_cast<unsigned long long>(ntry));
        atomicAdd(&g_seq_prof[4], static_cast<unsigned long long>(clock64() - c_start));
        atomicAdd(&g_seq_prof[5], static_cast<unsigned long long>(pi));
#endif
    }
}

}  // namespace decmg_gpu
