// Hierarchy construction on the device.
//
// Replaces, for binary subdivision towers, the reference's host setup path:
//   subdivide_nary(n=2)        proj/src/subdivision.cpp:12-110
//   from_triangles + finalize  proj/src/mesh.cpp:72-157
//   build_dual                 proj/src/dual.cpp:7-63, circumcenter geometry.cpp:5-16
//   hodge stars + laplacian_0  proj/src/operators.cpp:68-122 (via sparse.cpp:117-180)
//   matrix_of^T / restriction  proj/src/multigrid.cpp:215-216, geometric_map.cpp:162-223
// The reference scatters (+=) in triangle order; here every accumulation is a
// per-output gather over a sorted incidence list, which adds the same terms in
// the same order -- deterministic and bit-identical, no atomics on values.
// Integer structure (edge numbering, triangle edge triples, CSR) is built with
// counting sorts: counts (atomics, order-free) -> exclusive scan -> fill ->
// per-segment insertion sort, so the result never depends on thread timing.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

#include <cstdlib>
#include <cstring>

namespace decmg_gpu {
namespace {

constexpr int kBlock = 256;

// ---------------------------------------------------------------- Vec3 -----
// proj/include/decmg/geometry.hpp:12-43, component formulas verbatim.
struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 ld3(const double* p, int64_t i) {
    return {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
}
__device__ __forceinline__ void st3(double* p, int64_t i, V3 v) {
    p[3 * i] = v.x;
    p[3 * i + 1] = v.y;
    p[3 * i + 2] = v.z;
}
__device__ __forceinline__ V3 add(V3 a, V3 b) {
    return {__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z)};
}
__device__ __forceinline__ V3 sub(V3 a, V3 b) {
    return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)};
}
__device__ __forceinline__ V3 mul(V3 a, double s) {
    return {__dmul_rn(a.x, s), __dmul_rn(a.y, s), __dmul_rn(a.z, s)};
}
__device__ __forceinline__ V3 dvd(V3 a, double s) {
    return {__ddiv_rn(a.x, s), __ddiv_rn(a.y, s), __ddiv_rn(a.z, s)};
}
__device__ __forceinline__ double dot(V3 a, V3 b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ V3 cross(V3 a, V3 o) {
    return {__dsub_rn(__dmul_rn(a.y, o.z), __dmul_rn(a.z, o.y)),
            __dsub_rn(__dmul_rn(a.z, o.x), __dmul_rn(a.x, o.z)),
            __dsub_rn(__dmul_rn(a.x, o.y), __dmul_rn(a.y, o.x))};
}
__device__ __forceinline__ double norm(V3 a) { return __dsqrt_rn(dot(a, a)); }
__device__ __forceinline__ V3 midpt(V3 a, V3 b) { return mul(add(a, b), 0.5); }

__device__ __forceinline__ int64_t gtid() {
    return static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
}

// --------------------------------------------------------- subdivision -----
// subdivide_nary n = 2 (proj/src/subdivision.cpp:27-42): copies, then one
// midpoint per coarse edge at p_s*(1-1/2) + p_t*(1/2). project: extension x2.
__global__ void k_sub_pos(int nvc, int nec, const double* __restrict__ posc,
                          const int* __restrict__ edges_c, double* __restrict__ posf,
                          int project) {
    const int64_t j = gtid();
    if (j >= static_cast<int64_t>(nvc) + nec) return;
    if (j < nvc) {
        st3(posf, j, ld3(posc, j));
        return;
    }
    const int e = static_cast<int>(j - nvc);
    const V3 ps = ld3(posc, edges_c[2 * e]), pt = ld3(posc, edges_c[2 * e + 1]);
    const double tk = 1.0 / 2;
    V3 p = add(mul(ps, __dsub_rn(1.0, tk)), mul(pt, tk));
    if (project) {
        const double inv = __ddiv_rn(1.0, norm(p));
        p = mul(p, inv);
    }
    st3(posf, j, p);
}

// Four children per parent, in the lattice loop order of
// proj/src/subdivision.cpp:89-103: [v0,m01,m02],[m01,m12,m02],[m02,m12,v2],[m01,v1,m12],
// with m_ab = nv + e(a,b) (lattice_vertex, 63-87).
__global__ void k_sub_tris(int ntc, int nvc, const int* __restrict__ corners_c,
                           const int* __restrict__ tris_c, int* __restrict__ corners_f) {
    const int64_t t = gtid();
    if (t >= ntc) return;
    const int v0 = corners_c[3 * t], v1 = corners_c[3 * t + 1], v2 = corners_c[3 * t + 2];
    const int m12 = nvc + tris_c[3 * t], m02 = nvc + tris_c[3 * t + 1],
              m01 = nvc + tris_c[3 * t + 2];
    int* o = corners_f + 12 * t;
    o[0] = v0;  o[1] = m01;  o[2] = m02;
    o[3] = m01; o[4] = m12;  o[5] = m02;
    o[6] = m02; o[7] = m12;  o[8] = v2;
    o[9] = m01; o[10] = v1;  o[11] = m12;
}

// subdivide_nary n = 3, "cubic" (proj/src/subdivision.cpp:12-110,116-120):
// copies; points k = 1, 2 of coarse edge e at p_s*(1-t_k) + p_t*t_k, t_k = k/3
// (ids nvc + 2e + k - 1); the interior point of triangle t at
// (p0*b0 + p1*b1) + p2*b2, b1 = b2 = 1/3, b0 = (1 - b1) - b2 (id nvc + 2nec + t).
// project: every new point scaled by 1.0/|p| (extension x2).
__global__ void k_sub_pos3(int nvc, int nec, int ntc, const double* __restrict__ posc,
                           const int* __restrict__ edges_c, const int* __restrict__ corners_c,
                           double* __restrict__ posf, int project) {
    const int64_t j = gtid();
    const int64_t ne2 = 2 * static_cast<int64_t>(nec);
    if (j >= nvc + ne2 + ntc) return;
    if (j < nvc) {
        st3(posf, j, ld3(posc, j));
        return;
    }
    V3 p;
    if (j < nvc + ne2) {
        const int e = static_cast<int>((j - nvc) / 2), k = static_cast<int>((j - nvc) % 2) + 1;
        const V3 ps = ld3(posc, edges_c[2 * e]), pt = ld3(posc, edges_c[2 * e + 1]);
        const double tk = __ddiv_rn(static_cast<double>(k), 3.0);
        p = add(mul(ps, __dsub_rn(1.0, tk)), mul(pt, tk));
    } else {
        const int t = static_cast<int>(j - nvc - ne2);
        const double b1 = __ddiv_rn(1.0, 3.0), b2 = b1, b0 = __dsub_rn(__dsub_rn(1.0, b1), b2);
        p = add(add(mul(ld3(posc, corners_c[3 * t]), b0), mul(ld3(posc, corners_c[3 * t + 1]), b1)),
                mul(ld3(posc, corners_c[3 * t + 2]), b2));
    }
    if (project) {
        const double inv = __ddiv_rn(1.0, norm(p));
        p = mul(p, inv);
    }
    st3(posf, j, p);
}

// lattice_vertex (subdivision.cpp:63-87) for n = 3; the parent triangle
// stores e(v1,v2), e(v0,v2), e(v0,v1) (mesh.cpp:149-154)
__device__ int lattice3(int nvc, int nec, int t, int v0, int v1, int v2, const int* tris_c, const int* edges_c, int i,
                        int j) {
    const int k0 = 3 - i - j;
    if (i == 0 && j == 0) return v0;
    if (k0 == 0 && j == 0) return v1;
    if (k0 == 0 && i == 0) return v2;
    int a, e, k;
    if (j == 0) { a = v0; e = tris_c[3 * t + 2]; k = i; }
    else if (i == 0) { a = v0; e = tris_c[3 * t + 1]; k = j; }
    else if (k0 == 0) { a = v1; e = tris_c[3 * t]; k = j; }
    else return nvc + 2 * nec + t;
    const int step = edges_c[2 * e] == a ? k : 3 - k;
    return nvc + e * 2 + (step - 1);
}

// nine children per parent in the lattice loop order (subdivision.cpp:89-103)
__global__ void k_sub_tris3(int ntc, int nvc, int nec, const int* __restrict__ corners_c,
                            const int* __restrict__ tris_c, const int* __restrict__ edges_c,
                            int* __restrict__ corners_f) {
    const int64_t t = gtid();
    if (t >= ntc) return;
    const int v0 = corners_c[3 * t], v1 = corners_c[3 * t + 1], v2 = corners_c[3 * t + 2];
    int* o = corners_f + 27 * t;
    int q = 0;
    auto L = [&](int i, int j) { return lattice3(nvc, nec, static_cast<int>(t), v0, v1, v2, tris_c, edges_c, i, j); };
    for (int i = 0; i < 3; ++i)
        for (int j = 0; i + j < 3; ++j) {
            o[q++] = L(i, j);
            o[q++] = L(i + 1, j);
            o[q++] = L(i, j + 1);
            if (i + j < 2) {
                o[q++] = L(i + 1, j);
                o[q++] = L(i + 1, j + 1);
                o[q++] = L(i, j + 1);
            }
        }
}

// Map-column weights of the cubic points after GeometricMap::make
// (geometric_map.cpp:18-42): renormalised by the column's sequential sum when
// |sum - 1| <= 1e-9 (the sums here are 1.0, so the weights keep their bits).
__device__ void cubic_edge_w(int k, double* ws, double* wt) {
    const double tk = __ddiv_rn(static_cast<double>(k), 3.0);
    double a = __dsub_rn(1.0, tk), b = tk;
    const double sum = __dadd_rn(__dadd_rn(0.0, a), b);
    if (fabs(__dsub_rn(sum, 1.0)) <= 1e-9 && sum != 0.0) {
        a = __ddiv_rn(a, sum);
        b = __ddiv_rn(b, sum);
    }
    *ws = a;
    *wt = b;
}
__device__ void cubic_face_w(double* w) {
    const double b1 = __ddiv_rn(1.0, 3.0), b2 = b1, b0 = __dsub_rn(__dsub_rn(1.0, b1), b2);
    w[0] = b0; w[1] = b1; w[2] = b2;
    const double sum = __dadd_rn(__dadd_rn(__dadd_rn(0.0, b0), b1), b2);
    if (fabs(__dsub_rn(sum, 1.0)) <= 1e-9 && sum != 0.0)
        for (int a = 0; a < 3; ++a) w[a] = __ddiv_rn(w[a], sum);
}

// P = M(f)^T for the cubic map: rows sorted by coarse column (and weight)
__global__ void k_P_fill3(int nvf, int nvc, int nec, const int* __restrict__ edges_c,
                          const int* __restrict__ corners_c, int* __restrict__ rp, int* __restrict__ ci,
                          double* __restrict__ v) {
    const int64_t j = gtid();
    if (j > nvf) return;
    const int64_t ne2 = 2 * static_cast<int64_t>(nec);
    const int64_t r = j < nvc ? j : (j < nvc + ne2 ? nvc + 2 * (j - nvc) : nvc + 2 * ne2 + 3 * (j - nvc - ne2));
    rp[j] = static_cast<int>(r);
    if (j == nvf) return;
    if (j < nvc) {
        ci[r] = static_cast<int>(j);
        v[r] = 1.0;
    } else if (j < nvc + ne2) {
        const int e = static_cast<int>((j - nvc) / 2), k = static_cast<int>((j - nvc) % 2) + 1;
        double ws, wt;
        cubic_edge_w(k, &ws, &wt);
        ci[r] = edges_c[2 * e];  // src < tgt
        v[r] = ws;
        ci[r + 1] = edges_c[2 * e + 1];
        v[r + 1] = wt;
    } else {
        const int t = static_cast<int>(j - nvc - ne2);
        double w[3];
        cubic_face_w(w);
        int vv[3] = {corners_c[3 * t], corners_c[3 * t + 1], corners_c[3 * t + 2]};
        for (int a = 1; a < 3; ++a)  // sort (vertex, weight) pairs
            for (int b = a; b > 0 && (vv[b] < vv[b - 1] || (vv[b] == vv[b - 1] && w[b] < w[b - 1])); --b) {
                const int tv = vv[b]; vv[b] = vv[b - 1]; vv[b - 1] = tv;
                const double tw = w[b]; w[b] = w[b - 1]; w[b - 1] = tw;
            }
        for (int a = 0; a < 3; ++a) {
            ci[r + a] = vv[a];
            v[r + a] = w[a];
        }
    }
}

// R = rownormalize(M(f)) for the cubic map (geometric_map.cpp:205-223): row i
// = its copy, the two points of each incident edge (ascending edge), the
// interior point of each incident triangle (ascending triangle) -- ascending
// fine id -- with the row sum accumulated in that order.
__global__ void k_R_fill3(int nvc, int nec, const int* __restrict__ ve_ptr, const int* __restrict__ ve,
                          const int* __restrict__ vt_ptr, const int* __restrict__ vt,
                          const int* __restrict__ edges_c, int* __restrict__ rp, int* __restrict__ ci,
                          double* __restrict__ v) {
    const int64_t i = gtid();
    if (i > nvc) return;
    const int r0 = static_cast<int>(i) + 2 * ve_ptr[i] + vt_ptr[i];
    rp[i] = r0;
    if (i == nvc) return;
    double fw[3];
    cubic_face_w(fw);
    double rs = __dadd_rn(0.0, 1.0);
    for (int q = ve_ptr[i]; q < ve_ptr[i + 1]; ++q) {
        const int e = ve[q];
        for (int k = 1; k <= 2; ++k) {
            double ws, wt;
            cubic_edge_w(k, &ws, &wt);
            rs = __dadd_rn(rs, edges_c[2 * e] == i ? ws : wt);
        }
    }
    for (int q = vt_ptr[i]; q < vt_ptr[i + 1]; ++q) rs = __dadd_rn(rs, fw[vt[q] % 3]);
    const double inv = __ddiv_rn(1.0, rs);
    int k = r0;
    ci[k] = static_cast<int>(i);
    v[k++] = __dmul_rn(1.0, inv);
    for (int q = ve_ptr[i]; q < ve_ptr[i + 1]; ++q) {
        const int e = ve[q];
        for (int kk = 1; kk <= 2; ++kk) {
            double ws, wt;
            cubic_edge_w(kk, &ws, &wt);
            ci[k] = nvc + 2 * e + (kk - 1);
            v[k++] = __dmul_rn(edges_c[2 * e] == i ? ws : wt, inv);
        }
    }
    for (int q = vt_ptr[i]; q < vt_ptr[i + 1]; ++q) {
        ci[k] = nvc + 2 * nec + vt[q] / 3;
        v[k++] = __dmul_rn(fw[vt[q] % 3], inv);
    }
}

// ------------------------------------------------------ from_triangles -----// ------------------------------------------------------ from_triangles -----
__global__ void k_check_triples(int nt, int nv, const int* __restrict__ c, int* bad) {
    const int64_t t = gtid();
    if (t >= nt) return;
    for (int i = 0; i < 3; ++i) {
        const int a = c[3 * t + i], b = c[3 * t + (i + 1) % 3];
        if (a < 0 || a >= nv || b < 0 || b >= nv || a == b) atomicMin(bad, static_cast<int>(t));
    }
}

__global__ void k_pair_count(int nt, const int* __restrict__ c, int* cnt) {
    const int64_t q = gtid();
    if (q >= 3 * static_cast<int64_t>(nt)) return;
    const int64_t t = q / 3;
    const int i = static_cast<int>(q % 3);
    const int a = c[3 * t + i], b = c[3 * t + (i + 1) % 3];
    atomicAdd(&cnt[min(a, b)], 1);
}

__global__ void k_pair_fill(int nt, const int* __restrict__ c, const int* __restrict__ off,
                            int* fill, int* __restrict__ bucket) {
    const int64_t q = gtid();
    if (q >= 3 * static_cast<int64_t>(nt)) return;
    const int64_t t = q / 3;
    const int i = static_cast<int>(q % 3);
    const int a = c[3 * t + i], b = c[3 * t + (i + 1) % 3];
    const int s = min(a, b);
    bucket[off[s] + atomicAdd(&fill[s], 1)] = max(a, b);
}

// Sorts each segment ascending (insertion sort; segments are vertex or edge
// stars, a handful of entries).
__device__ void sort_range(int* v, int lo, int hi) {
    for (int i = lo + 1; i < hi; ++i) {
        const int key = v[i];
        int j = i - 1;
        while (j >= lo && v[j] > key) {
            v[j + 1] = v[j];
            --j;
        }
        v[j + 1] = key;
    }
}

__global__ void k_bucket_unique(int nv, const int* __restrict__ off, int* bucket, int* ucnt) {
    const int64_t v = gtid();
    if (v >= nv) return;
    const int lo = off[v], hi = off[v + 1];
    sort_range(bucket, lo, hi);
    int u = 0;
    for (int i = lo; i < hi; ++i)
        if (i == lo || bucket[i] != bucket[i - 1]) bucket[lo + u++] = bucket[i];
    ucnt[v] = u;
}

__global__ void k_write_edges(int nv, const int* __restrict__ off, const int* __restrict__ bucket,
                              const int* __restrict__ eptr, int* __restrict__ edges) {
    const int64_t v = gtid();
    if (v >= nv) return;
    for (int e = eptr[v]; e < eptr[v + 1]; ++e) {
        edges[2 * static_cast<int64_t>(e)] = static_cast<int>(v);
        edges[2 * static_cast<int64_t>(e) + 1] = bucket[off[v] + (e - eptr[v])];
    }
}

__device__ int find_edge(const int* __restrict__ eptr, const int* __restrict__ edges, int a, int b) {
    const int s = min(a, b), t = max(a, b);
    int lo = eptr[s], hi = eptr[s + 1] - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int v = edges[2 * static_cast<int64_t>(mid) + 1];
        if (v == t) return mid;
        if (v < t) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

// triangle = {e(v1,v2), e(v0,v2), e(v0,v1)} (proj/src/mesh.cpp:149-154)
__global__ void k_tri_edges(int nt, const int* __restrict__ c, const int* __restrict__ eptr,
                            const int* __restrict__ edges, int* __restrict__ tris) {
    const int64_t t = gtid();
    if (t >= nt) return;
    const int v0 = c[3 * t], v1 = c[3 * t + 1], v2 = c[3 * t + 2];
    tris[3 * t] = find_edge(eptr, edges, v1, v2);
    tris[3 * t + 1] = find_edge(eptr, edges, v0, v2);
    tris[3 * t + 2] = find_edge(eptr, edges, v0, v1);
}

__global__ void k_deg_count(int ne, const int* __restrict__ edges, int* deg) {
    const int64_t e = gtid();
    if (e >= ne) return;
    atomicAdd(&deg[edges[2 * e]], 1);
    atomicAdd(&deg[edges[2 * e + 1]], 1);
}

__global__ void k_ve_fill_tgt(int ne, const int* __restrict__ edges, const int* __restrict__ ve_ptr,
                              int* fill, int* __restrict__ ve) {
    const int64_t e = gtid();
    if (e >= ne) return;
    const int t = edges[2 * e + 1];
    ve[ve_ptr[t] + atomicAdd(&fill[t], 1)] = static_cast<int>(e);
}

// vertex -> incident edges ascending (proj/src/mesh.cpp:99-104): edges where
// v is the target all precede (lexicographically) the ones where it is the
// source, which are already contiguous and ascending.
__global__ void k_ve_finish(int nv, const int* __restrict__ eptr, const int* __restrict__ ve_ptr,
                            const int* __restrict__ fill, int* __restrict__ ve) {
    const int64_t v = gtid();
    if (v >= nv) return;
    const int base = ve_ptr[v], nt_ = fill[v];
    sort_range(ve, base, base + nt_);
    for (int e = eptr[v]; e < eptr[v + 1]; ++e) ve[base + nt_ + (e - eptr[v])] = e;
}

// edge -> triangles and vertex -> (triangle, corner) incidences
__global__ void k_inc_count(int nt, const int* __restrict__ idx, int* cnt) {
    const int64_t q = gtid();
    if (q >= 3 * static_cast<int64_t>(nt)) return;
    atomicAdd(&cnt[idx[q]], 1);
}
__global__ void k_inc_fill(int nt, const int* __restrict__ idx, const int* __restrict__ ptr,
                           int* fill, int* __restrict__ out) {
    const int64_t q = gtid();
    if (q >= 3 * static_cast<int64_t>(nt)) return;
    const int s = idx[q];
    // store triangle*3 + slot: sorting it orders by triangle, then slot
    out[ptr[s] + atomicAdd(&fill[s], 1)] = static_cast<int>(q);
}
__global__ void k_sort_segments(int nseg, const int* __restrict__ ptr, int* vals) {
    const int64_t s = gtid();
    if (s >= nseg) return;
    sort_range(vals, ptr[s], ptr[s + 1]);
}

// -------------------------------------------------------------- dual -------
// proj/src/dual.cpp:15-23
__global__ void k_edge_geom(int ne, const double* __restrict__ pos, const int* __restrict__ edges,
                            double* __restrict__ mid, double* __restrict__ plen, int* bad) {
    const int64_t e = gtid();
    if (e >= ne) return;
    const V3 a = ld3(pos, edges[2 * e]), b = ld3(pos, edges[2 * e + 1]);
    st3(mid, e, midpt(a, b));
    const double l = norm(sub(b, a));
    plen[e] = l;
    if (l <= 0.0) atomicMin(bad, static_cast<int>(e));
}

// proj/src/dual.cpp:25-60 per triangle; circumcenter per geometry.cpp:5-16.
// Writes the three |cc - mid_e| terms (slot order of triangles[t]) and the six
// signed wedges in loop order (w_i(0), w_j(0), w_i(1), w_j(1), w_i(2), w_j(2)).
__global__ void k_tri_geom(int nt, const double* __restrict__ pos, const int* __restrict__ corners,
                           const int* __restrict__ tris, const double* __restrict__ mid,
                           double* __restrict__ dist, double* __restrict__ wedge, int* bad) {
    const int64_t t = gtid();
    if (t >= nt) return;
    const int vid[3] = {corners[3 * t], corners[3 * t + 1], corners[3 * t + 2]};
    const V3 p[3] = {ld3(pos, vid[0]), ld3(pos, vid[1]), ld3(pos, vid[2])};
    const V3 a = sub(p[1], p[0]), b = sub(p[2], p[0]);
    const V3 n = cross(a, b);
    const double n2 = dot(n, n);
    if (n2 <= __dmul_rn(__dmul_rn(1e-28, dot(a, a)), dot(b, b))) {
        atomicMin(bad, static_cast<int>(t));
        return;
    }
    const V3 num = add(mul(cross(b, n), dot(a, a)), mul(cross(n, a), dot(b, b)));
    const V3 cc = add(p[0], dvd(num, __dmul_rn(2.0, n2)));
    const double area2 = norm(n);
    const V3 nhat = dvd(n, area2);
    for (int j = 0; j < 3; ++j) {
        const int e = tris[3 * t + j];
        dist[3 * t + j] = norm(sub(cc, ld3(mid, e)));
    }
    for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3;
        const V3 m = midpt(p[i], p[j]);
        wedge[6 * t + 2 * i] = __dmul_rn(0.5, dot(cross(sub(m, p[i]), sub(cc, p[i])), nhat));
        wedge[6 * t + 2 * i + 1] = __dmul_rn(0.5, dot(cross(sub(p[j], m), sub(cc, m)), nhat));
    }
}

// |*e| = sum over incident triangles ascending (dual.cpp:44-46) and
// star1 = |*e| / |e| (operators.cpp:76).
__global__ void k_edge_w(int ne, const int* __restrict__ et_ptr, const int* __restrict__ et,
                         const double* __restrict__ dist, const double* __restrict__ plen,
                         double* __restrict__ w) {
    const int64_t e = gtid();
    if (e >= ne) return;
    double s = 0.0;
    for (int q = et_ptr[e]; q < et_ptr[e + 1]; ++q) s = __dadd_rn(s, dist[et[q]]);
    w[e] = __ddiv_rn(s, plen[e]);
}

// dual cell area: the two wedges of every incident triangle, triangles
// ascending, in the order the reference loop adds them (dual.cpp:56-59).
__global__ void k_vertex_area(int nv, const int* __restrict__ vt_ptr, const int* __restrict__ vt,
                              const double* __restrict__ wedge, double* __restrict__ area) {
    const int64_t v = gtid();
    if (v >= nv) return;
    double A = 0.0;
    for (int q = vt_ptr[v]; q < vt_ptr[v + 1]; ++q) {
        const int64_t code = vt[q];
        const int64_t t = code / 3;
        const int c = static_cast<int>(code % 3);
        const double* w = wedge + 6 * t;
        const double first = c == 0 ? w[0] : (c == 1 ? w[1] : w[3]);
        const double second = c == 0 ? w[5] : (c == 1 ? w[2] : w[4]);
        A = __dadd_rn(A, first);
        A = __dadd_rn(A, second);
    }
    area[v] = A;
}

// extension x1: endpoints of edges with exactly one incident triangle
__global__ void k_boundary(int ne, const int* __restrict__ et_ptr, const int* __restrict__ edges,
                           int* bd) {
    const int64_t e = gtid();
    if (e >= ne) return;
    if (et_ptr[e + 1] - et_ptr[e] == 1) {
        bd[edges[2 * e]] = 1;
        bd[edges[2 * e + 1]] = 1;
    }
}

__global__ void k_lap_count(int nv, const int* __restrict__ ve_ptr, int* cnt) {
    const int64_t i = gtid();
    if (i >= nv) return;
    cnt[i] = 1 + ve_ptr[i + 1] - ve_ptr[i];
}

// laplacian_0 = scale_rows(star0_inv, (-1) * d0^T (star1 d0)) (operators.cpp:102-122):
//   L_ij = ((0.0 + (-w_e)) * -1.0) * (1.0/A_i)
//   L_ii = ((((0.0 + w_e1) + w_e2) + ...) * -1.0) * (1.0/A_i)
// columns ascending, structural zeros kept. Extension x1 replaces boundary
// rows by identity rows with the same sparsity.
__global__ void k_lap_fill(int nv, const int* __restrict__ edges, const int* __restrict__ ve_ptr,
                           const int* __restrict__ ve, const double* __restrict__ w,
                           const double* __restrict__ area, const int* __restrict__ bd,
                           int dirichlet, const int* __restrict__ L_rp, int* __restrict__ L_ci,
                           double* __restrict__ L_v, double* __restrict__ diag, int* bad_area,
                           int* zero_diag) {
    const int64_t i64 = gtid();
    if (i64 >= nv) return;
    const int i = static_cast<int>(i64);
    const double A = area[i];
    if (A <= 0.0) atomicMin(bad_area, i);
    const double inv = __ddiv_rn(1.0, A);
    double sum = 0.0;
    for (int q = ve_ptr[i]; q < ve_ptr[i + 1]; ++q) sum = __dadd_rn(sum, w[ve[q]]);
    const bool ident = dirichlet && bd[i];
    const double dval = ident ? 1.0 : __dmul_rn(__dmul_rn(sum, -1.0), inv);
    int k = L_rp[i];
    bool placed = false;
    for (int q = ve_ptr[i]; q < ve_ptr[i + 1]; ++q) {
        const int e = ve[q];
        const int s = edges[2 * static_cast<int64_t>(e)], t = edges[2 * static_cast<int64_t>(e) + 1];
        const int j = s == i ? t : s;
        if (!placed && j > i) {
            L_ci[k] = i;
            L_v[k] = dval;
            ++k;
            placed = true;
        }
        const double a = __dadd_rn(0.0, -w[e]);
        L_ci[k] = j;
        L_v[k] = ident ? 0.0 : __dmul_rn(__dmul_rn(a, -1.0), inv);
        ++k;
    }
    if (!placed) {
        L_ci[k] = i;
        L_v[k] = dval;
    }
    diag[i] = dval;
    if (dval == 0.0) atomicMin(zero_diag, i);
}

// P = M(f)^T: copy rows {(j,1.0)}, midpoint rows {(s,0.5),(t,0.5)}
// (subdivision.cpp:27-42, geometric_map.cpp:18-42, multigrid.cpp:215)
__global__ void k_P_fill(int nvf, int nvc, const int* __restrict__ edges_c, int* __restrict__ rp,
                         int* __restrict__ ci, double* __restrict__ v) {
    const int64_t j = gtid();
    if (j > nvf) return;
    const int64_t r = j < nvc ? j : nvc + 2 * (j - nvc);
    rp[j] = static_cast<int>(r);
    if (j == nvf) return;
    if (j < nvc) {
        ci[r] = static_cast<int>(j);
        v[r] = 1.0;
    } else {
        const int64_t e = j - nvc;
        ci[r] = edges_c[2 * e];
        v[r] = 0.5;
        ci[r + 1] = edges_c[2 * e + 1];
        v[r + 1] = 0.5;
    }
}

// R = scale_rows(M, 1/rowsum) (geometric_map.cpp:205-223): row i = coarse
// vertex i, columns {i} U {nvc + e : e incident to i} ascending; rowsum added
// in CSC (= fine column) order: 1.0 then 0.5 per incident edge.
__global__ void k_R_fill(int nvc, const int* __restrict__ ve_ptr, const int* __restrict__ ve,
                         int* __restrict__ rp, int* __restrict__ ci, double* __restrict__ v) {
    const int64_t i = gtid();
    if (i > nvc) return;
    const int r0 = static_cast<int>(i) + ve_ptr[i];
    rp[i] = r0;
    if (i == nvc) return;
    double rs = 0.0;
    rs = __dadd_rn(rs, 1.0);
    for (int q = ve_ptr[i]; q < ve_ptr[i + 1]; ++q) rs = __dadd_rn(rs, 0.5);
    const double inv = __ddiv_rn(1.0, rs);
    ci[r0] = static_cast<int>(i);
    v[r0] = __dmul_rn(1.0, inv);
    int k = r0 + 1;
    for (int q = ve_ptr[i]; q < ve_ptr[i + 1]; ++q, ++k) {
        ci[k] = nvc + ve[q];
        v[k] = __dmul_rn(0.5, inv);
    }
}

// ------------------------------------------------------------ row order ----
// Processing order for the hot kernels: vertices sorted by the Morton code of
// their position (21 bits per axis inside the mesh bounding box), ties by id.
// Spatial neighbours then sit in nearby rows, so the gathers of x[col] of the
// rows in flight hit L2 instead of HBM. The order only changes which thread
// computes which row, never the arithmetic of a row.
__device__ __forceinline__ unsigned long long okey(double d) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}

__global__ void k_bbox(int n, const double* __restrict__ pos, unsigned long long* mm) {
    __shared__ unsigned long long lo[3][kBlock], hi[3][kBlock];
    const int64_t i = gtid();
    for (int c = 0; c < 3; ++c) {
        const unsigned long long k = i < n ? okey(pos[3 * i + c]) : 0;
        lo[c][threadIdx.x] = i < n ? k : ~0ULL;
        hi[c][threadIdx.x] = i < n ? k : 0ULL;
    }
    __syncthreads();
    for (int s = kBlock / 2; s >= 1; s >>= 1) {
        if (threadIdx.x < s)
            for (int c = 0; c < 3; ++c) {
                lo[c][threadIdx.x] = min(lo[c][threadIdx.x], lo[c][threadIdx.x + s]);
                hi[c][threadIdx.x] = max(hi[c][threadIdx.x], hi[c][threadIdx.x + s]);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 3; ++c) {
            atomicMin(&mm[c], lo[c][0]);
            atomicMax(&mm[3 + c], hi[c][0]);
        }
}

__device__ __forceinline__ unsigned long long spread3(unsigned long long x) {
    x &= 0x1fffffULL;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

__global__ void k_morton(int n, const double* __restrict__ pos, double lx, double ly, double lz, double sx,
                         double sy, double sz, unsigned long long* __restrict__ key, int* __restrict__ id) {
    const int64_t i = gtid();
    if (i >= n) return;
    const double lo[3] = {lx, ly, lz}, sc[3] = {sx, sy, sz};
    unsigned long long q[3];
    for (int c = 0; c < 3; ++c) {
        double f = (pos[3 * i + c] - lo[c]) * sc[c];
        f = f < 0.0 ? 0.0 : (f > 2097151.0 ? 2097151.0 : f);
        q[c] = static_cast<unsigned long long>(f);
    }
    key[i] = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
    id[i] = static_cast<int>(i);
}

// Renumbering of a CSR operator: row r of the output is row ord[r] of the
// input (ord == nullptr: identity) with its entries in the input order and
// every column c replaced by cinv[c] (cinv == nullptr: unchanged).
__global__ void k_perm_count(int n, const int* __restrict__ ord, const int* __restrict__ rp, int* cnt) {
    const int64_t r = gtid();
    if (r >= n) return;
    const int o = ord ? ord[r] : static_cast<int>(r);
    cnt[r] = rp[o + 1] - rp[o];
}

__global__ void k_perm_fill(int n, const int* __restrict__ ord, const int* __restrict__ cinv,
                            const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                            const int* __restrict__ orp, int* __restrict__ oci, double* __restrict__ ov) {
    const int64_t r = gtid();
    if (r >= n) return;
    const int o = ord ? ord[r] : static_cast<int>(r);
    const int src = rp[o], len = rp[o + 1] - src, dst = orp[r];
    for (int k = 0; k < len; ++k) {
        oci[dst + k] = cinv ? cinv[ci[src + k]] : ci[src + k];
        ov[dst + k] = v[src + k];
    }
}

// Level schedule of gauss_seidel_sweep (multigrid.cpp:13-34) in the reference
// numbering: ph[i] = 1 + max ph[j] over neighbours j < i (j > i for the
// reverse sweep), 0 without such neighbours. Jacobi-style relaxation from 0
// reaches the fixpoint after depth + 1 steps.
__global__ void k_gs_phase_step(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                const int* __restrict__ ph_in, int* __restrict__ ph_out, int reverse,
                                int* changed) {
    const int64_t i = gtid();
    if (i >= n) return;
    int p = 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = ci[k];
        if (reverse ? j > i : j < i) p = max(p, ph_in[j] + 1);
    }
    ph_out[i] = p;
    if (p != ph_in[i]) *changed = 1;
}

__global__ void k_gs_keys(int n, const int* __restrict__ ord, const int* __restrict__ ph, int* __restrict__ key,
                          int* __restrict__ q) {
    const int64_t r = gtid();
    if (r >= n) return;
    key[r] = ph[ord ? ord[r] : static_cast<int>(r)];
    q[r] = static_cast<int>(r);
}

__global__ void k_invert(int n, const int* __restrict__ ord, int* __restrict__ inv) {
    const int64_t q = gtid();
    if (q < n) inv[ord[q]] = static_cast<int>(q);
}

template <class T>
__global__ void k_take(int n, const int* __restrict__ ord, const T* __restrict__ in, T* __restrict__ out) {
    const int64_t q = gtid();
    if (q < n) out[q] = in[ord[q]];
}

__global__ void k_row_maxlen(int n, const int* __restrict__ rp, int* mx) {
    const int64_t q = gtid();
    if (q >= n) return;
    atomicMax(mx, rp[q + 1] - rp[q]);
}

// rows >= n are padding (column -1, row id -1) up to npad
// Padded ELL copy of a CSR operator in row order ord. Padding entries hold a
// real column with value 0.0 -- the row itself for L (diag), the row's first
// column otherwise -- so the row kernels need no validity test: s + 0.0 * x
// equals s bit for bit for finite x (s starts at +0.0 and is never -0.0).
// erow[q] = original row id | (slot of the diagonal entry << kRowBits)
// (common.cuh), -1 for padding rows past n.
__global__ void k_ell_fill(int n, int npad, int W, const int* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, const int* __restrict__ ord, bool diag,
                           int* __restrict__ eci, double* __restrict__ ev, int* __restrict__ erow) {
    const int64_t q = gtid();
    if (q >= npad) return;
    const int k0 = q < n ? rp[q] : 0, len = q < n ? rp[q + 1] - k0 : 0;
    const int row = q < n ? (ord ? ord[q] : static_cast<int>(q)) : -1;
    const int padc = q >= n ? -1 : (diag ? row : (len > 0 ? ci[k0] : 0));
    int slot = 0;
    for (int j = 0; j < W; ++j) {
        const int c = j < len ? ci[k0 + j] : padc;
        eci[q * W + j] = c;
        ev[q * W + j] = j < len ? v[k0 + j] : 0.0;
        if (diag && j < len && c == row) slot = j;
    }
    if (erow) erow[q] = q < n ? (row | (slot << kRowBits)) : -1;
}

// ------------------------------------------------------------ helpers ------
struct TmpPool {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit TmpPool(cudaStream_t st) : s(st) {}
    template <class T>
    Status get(T** p, size_t n) {
        void* q = nullptr;
        DG_CUDA(cudaMallocAsync(&q, (n ? n : 1) * sizeof(T), s));
        ptrs.push_back(q);
        *p = static_cast<T*>(q);
        return Status::Ok();
    }
    ~TmpPool() {
        for (void* q : ptrs) cudaFreeAsync(q, s);
    }
};

Status read_int(decmg_gpu_ctx* c, const int* d, int* h) {
    DG_CUDA(cudaMemcpyAsync(h, d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    DG_CUDA(cudaStreamSynchronize(c->stream));
    return Status::Ok();
}

Status check_flag(decmg_gpu_ctx* c, const int* d_flag, const char* msg, const char* what = nullptr) {
    int v = 0;
    DG_TRY(read_int(c, d_flag, &v));
    if (v != 0x7fffffff) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s %d%s", msg, v, what ? what : "");
        return Status::Err(DECMG_RUNTIME, buf);
    }
    return Status::Ok();
}

Status new_flag(decmg_gpu_ctx* c, TmpPool& tp, int** f) {
    DG_TRY(tp.get(f, 1));
    const int big = 0x7fffffff;
    DG_CUDA(cudaMemcpyAsync(*f, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    return Status::Ok();
}

#define LAUNCH(cls, n, kernel, ...)                                                             \
    DG_TRY(launch(c, cls, 0.0, [&] {                                                            \
        if ((n) > 0) kernel<<<grid_for((n), kBlock), kBlock, 0, c->stream>>>(__VA_ARGS__);       \
    }))

// Counting-sort an incidence list: for q in [0, 3 nt), key idx[q] -> segment.
Status incidence(decmg_gpu_ctx* c, TmpPool& tp, int nt, const int* idx, int nseg, int** ptr,
                 int** vals) {
    int *cnt, *fill;
    DG_TRY(tp.get(&cnt, nseg + 1));
    DG_TRY(tp.get(&fill, nseg));
    DG_TRY(tp.get(ptr, nseg + 1));
    DG_TRY(tp.get(vals, 3 * static_cast<size_t>(nt)));
    DG_CUDA(cudaMemsetAsync(cnt, 0, (nseg + 1) * sizeof(int), c->stream));
    DG_CUDA(cudaMemsetAsync(fill, 0, nseg * sizeof(int), c->stream));
    LAUNCH(4, 3 * static_cast<int64_t>(nt), k_inc_count, nt, idx, cnt);
    DG_TRY(exclusive_scan(c, cnt, *ptr, nseg));
    LAUNCH(4, 3 * static_cast<int64_t>(nt), k_inc_fill, nt, idx, *ptr, fill, *vals);
    LAUNCH(4, nseg, k_sort_segments, nseg, *ptr, *vals);
    return Status::Ok();
}

// EmbeddedComplex2D::from_triangles (proj/src/mesh.cpp:122-157) on the device.
// pos [nv][3] and corners [nt][3] must already be context allocations.
Status mesh_from_triangles(decmg_gpu_ctx* c, Level& m, double* pos, int nv, int* corners, int nt) {
    TmpPool tp(c->stream);
    m.nv = nv;
    m.nt = nt;
    m.pos = pos;
    m.corners = corners;
    int* bad;
    DG_TRY(new_flag(c, tp, &bad));
    LAUNCH(4, nt, k_check_triples, nt, nv, corners, bad);
    {
        int v = 0;
        DG_TRY(read_int(c, bad, &v));
        if (v != 0x7fffffff) return Status::Err(DECMG_RUNTIME, "from_triangles: bad corner triple");
    }
    int *cnt, *off, *fill, *bucket, *ucnt;
    DG_TRY(tp.get(&cnt, nv + 1));
    DG_TRY(tp.get(&off, nv + 1));
    DG_TRY(tp.get(&fill, nv));
    DG_TRY(tp.get(&bucket, 3 * static_cast<size_t>(nt)));
    DG_TRY(tp.get(&ucnt, nv + 1));
    DG_CUDA(cudaMemsetAsync(cnt, 0, (nv + 1) * sizeof(int), c->stream));
    DG_CUDA(cudaMemsetAsync(fill, 0, nv * sizeof(int), c->stream));
    DG_CUDA(cudaMemsetAsync(ucnt, 0, (nv + 1) * sizeof(int), c->stream));
    LAUNCH(4, 3 * static_cast<int64_t>(nt), k_pair_count, nt, corners, cnt);
    DG_TRY(exclusive_scan(c, cnt, off, nv));
    LAUNCH(4, 3 * static_cast<int64_t>(nt), k_pair_fill, nt, corners, off, fill, bucket);
    LAUNCH(4, nv, k_bucket_unique, nv, off, bucket, ucnt);
    DG_TRY(dalloc(c, &m.eptr, nv + 1));
    DG_TRY(exclusive_scan(c, ucnt, m.eptr, nv));
    DG_TRY(read_int(c, m.eptr + nv, &m.ne));
    DG_TRY(dalloc(c, &m.edges, 2 * static_cast<size_t>(m.ne)));
    LAUNCH(4, nv, k_write_edges, nv, off, bucket, m.eptr, m.edges);
    DG_TRY(dalloc(c, &m.tris, 3 * static_cast<size_t>(nt)));
    LAUNCH(4, nt, k_tri_edges, nt, corners, m.eptr, m.edges, m.tris);
    // vertex -> edges (finalize, mesh.cpp:99-104)
    int *deg, *vfill;
    DG_TRY(tp.get(&deg, nv + 1));
    DG_TRY(tp.get(&vfill, nv));
    DG_CUDA(cudaMemsetAsync(deg, 0, (nv + 1) * sizeof(int), c->stream));
    DG_CUDA(cudaMemsetAsync(vfill, 0, nv * sizeof(int), c->stream));
    LAUNCH(4, m.ne, k_deg_count, m.ne, m.edges, deg);
    DG_TRY(dalloc(c, &m.ve_ptr, nv + 1));
    DG_TRY(exclusive_scan(c, deg, m.ve_ptr, nv));
    DG_TRY(dalloc(c, &m.ve, 2 * static_cast<size_t>(m.ne)));
    LAUNCH(4, m.ne, k_ve_fill_tgt, m.ne, m.edges, m.ve_ptr, vfill, m.ve);
    LAUNCH(4, nv, k_ve_finish, nv, m.eptr, m.ve_ptr, vfill, m.ve);
    DG_CUDA(cudaStreamSynchronize(c->stream));
    return Status::Ok();
}

// build_dual + laplacian_0 + boundary for one level.
__global__ void k_clamp_area(int nv, double floor_area, double* __restrict__ area) {
    const int64_t i = gtid();
    if (i < nv && area[i] <= 0.0) area[i] = floor_area;
}
// dual_areas = 1 / star0_inv (operators.cpp:109-114, clamped assembly)
__global__ void k_area_from_inv(int nv, double* __restrict__ area) {
    const int64_t i = gtid();
    if (i < nv) area[i] = __ddiv_rn(1.0, __ddiv_rn(1.0, area[i]));
}

Status assemble(decmg_gpu_ctx* c, Level& m, bool dirichlet, bool clamp) {
    TmpPool tp(c->stream);
    const int nv = m.nv, ne = m.ne, nt = m.nt;
    int *bad_edge, *bad_tri, *bad_area, *zero_diag;
    DG_TRY(new_flag(c, tp, &bad_edge));
    DG_TRY(new_flag(c, tp, &bad_tri));
    DG_TRY(new_flag(c, tp, &bad_area));
    DG_TRY(new_flag(c, tp, &zero_diag));
    double *mid, *plen, *dist, *wedge, *w;
    DG_TRY(tp.get(&mid, 3 * static_cast<size_t>(ne)));
    DG_TRY(tp.get(&plen, ne));
    DG_TRY(tp.get(&dist, 3 * static_cast<size_t>(nt)));
    DG_TRY(tp.get(&wedge, 6 * static_cast<size_t>(nt)));
    DG_TRY(tp.get(&w, ne));
    LAUNCH(4, ne, k_edge_geom, ne, m.pos, m.edges, mid, plen, bad_edge);
    DG_TRY(check_flag(c, bad_edge, "build_dual: zero-length edge"));
    LAUNCH(4, nt, k_tri_geom, nt, m.pos, m.corners, m.tris, mid, dist, wedge, bad_tri);
    {
        int v = 0;
        DG_TRY(read_int(c, bad_tri, &v));
        if (v != 0x7fffffff) return Status::Err(DECMG_RUNTIME, "circumcenter: degenerate triangle");
    }
    int *et_ptr, *et, *vt_ptr, *vt;
    DG_TRY(incidence(c, tp, nt, m.tris, ne, &et_ptr, &et));
    DG_TRY(incidence(c, tp, nt, m.corners, nv, &vt_ptr, &vt));
    LAUNCH(4, ne, k_edge_w, ne, et_ptr, et, dist, plen, w);
    DG_TRY(dalloc(c, &m.area, nv));
    LAUNCH(4, nv, k_vertex_area, nv, vt_ptr, vt, wedge, m.area);
    if (clamp) {
        // HodgeOptions::clamp_dual_areas (operators.cpp:80-98): nonpositive areas
        // become 1e-14 * mean, the mean summed in vertex order
        std::vector<double> a(nv);
        DG_CUDA(cudaMemcpyAsync(a.data(), m.area, sizeof(double) * nv, cudaMemcpyDeviceToHost, c->stream));
        DG_CUDA(cudaStreamSynchronize(c->stream));
        double mean = 0.0;
        for (double x : a) mean += x;
        mean /= std::max(nv, 1);
        LAUNCH(4, nv, k_clamp_area, nv, 1e-14 * mean, m.area);
    }
    DG_TRY(dalloc(c, &m.bd, nv));
    DG_CUDA(cudaMemsetAsync(m.bd, 0, nv * sizeof(int), c->stream));
    LAUNCH(4, ne, k_boundary, ne, et_ptr, m.edges, m.bd);
    int* cnt;
    DG_TRY(tp.get(&cnt, nv + 1));
    DG_CUDA(cudaMemsetAsync(cnt, 0, (nv + 1) * sizeof(int), c->stream));
    LAUNCH(4, nv, k_lap_count, nv, m.ve_ptr, cnt);
    DG_TRY(dalloc(c, &m.L_rp, nv + 1));
    DG_TRY(exclusive_scan(c, cnt, m.L_rp, nv));
    m.nnzL = static_cast<int64_t>(nv) + 2 * static_cast<int64_t>(ne);
    DG_TRY(dalloc(c, &m.L_ci, m.nnzL));
    DG_TRY(dalloc(c, &m.L_v, m.nnzL));
    DG_TRY(dalloc(c, &m.diag, nv));
    LAUNCH(4, nv, k_lap_fill, nv, m.edges, m.ve_ptr, m.ve, w, m.area, m.bd, dirichlet ? 1 : 0,
           m.L_rp, m.L_ci, m.L_v, m.diag, bad_area, zero_diag);
    DG_TRY(check_flag(c, bad_area, "hodge_star_0_inv: non-well-centered dual cell at vertex"));
    if (clamp) LAUNCH(4, nv, k_area_from_inv, nv, m.area);
    int zd = 0;
    DG_TRY(read_int(c, zero_diag, &zd));
    m.zero_diag_row = zd == 0x7fffffff ? -1 : zd;
    DG_CUDA(cudaStreamSynchronize(c->stream));
    return Status::Ok();
}

}  // namespace

// Bounding box of a level's positions and the 21-bit quantization scale.
Status level_bbox(decmg_gpu_ctx* c, const Level& m, double lo[3], double sc[3]) {
    TmpPool tp(c->stream);
    unsigned long long* mm;
    DG_TRY(tp.get(&mm, 6));
    const unsigned long long init[6] = {~0ULL, ~0ULL, ~0ULL, 0ULL, 0ULL, 0ULL};
    DG_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
    LAUNCH(4, m.nv, k_bbox, m.nv, m.pos, mm);
    unsigned long long h[6];
    DG_CUDA(cudaMemcpyAsync(h, mm, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    DG_CUDA(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < 3; ++k) {
        auto dec = [](unsigned long long u) {
            u = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
            double d;
            std::memcpy(&d, &u, sizeof d);
            return d;
        };
        lo[k] = dec(h[k]);
        const double ext = dec(h[3 + k]) - lo[k];
        sc[k] = ext > 0.0 ? 2097151.0 / ext : 0.0;
    }
    return Status::Ok();
}

// Morton keys of a level's positions in a given box (ids written to d_id if non-null).
Status morton_keys(decmg_gpu_ctx* c, const Level& m, const double lo[3], const double sc[3],
                   unsigned long long* d_keys, int* d_id) {
    TmpPool tp(c->stream);
    int* id = d_id;
    if (!id) DG_TRY(tp.get(&id, m.nv));
    LAUNCH(4, m.nv, k_morton, m.nv, m.pos, lo[0], lo[1], lo[2], sc[0], sc[1], sc[2], d_keys, id);
    DG_CUDA(cudaStreamSynchronize(c->stream));
    return Status::Ok();
}

namespace {

Status morton_order(decmg_gpu_ctx* c, Level& m) {
    TmpPool tp(c->stream);
    double lo[3], sc[3];
    DG_TRY(level_bbox(c, m, lo, sc));
    unsigned long long *kin, *kout;
    int *iin;
    DG_TRY(tp.get(&kin, m.nv));
    DG_TRY(tp.get(&kout, m.nv));
    DG_TRY(tp.get(&iin, m.nv));
    DG_TRY(dalloc(c, &m.ord, m.nv));
    DG_TRY(morton_keys(c, m, lo, sc, kin, iin));
    size_t bytes = 0;
    DG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, iin, m.ord, m.nv, 0, 64, c->stream));
    void* tmp;
    DG_TRY(tp.get(reinterpret_cast<char**>(&tmp), bytes));
    DG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, iin, m.ord, m.nv, 0, 64, c->stream));
    DG_TRY(dalloc(c, &m.inv, m.nv));
    LAUNCH(4, m.nv, k_invert, m.nv, m.ord, m.inv);
    return Status::Ok();
}

Status permute_rows(decmg_gpu_ctx* c, int nrows, const int* ord, const int* cinv, const int* rp, const int* ci,
                    const double* v, int64_t nnz, int** orp, int** oci, double** ov) {
    if (!ord && !cinv) {  // identity on both sides: share the reference arrays
        *orp = const_cast<int*>(rp);
        *oci = const_cast<int*>(ci);
        *ov = const_cast<double*>(v);
        return Status::Ok();
    }
    TmpPool tp(c->stream);
    int* cnt;
    DG_TRY(tp.get(&cnt, nrows + 1));
    DG_CUDA(cudaMemsetAsync(cnt, 0, (nrows + 1) * sizeof(int), c->stream));
    DG_TRY(dalloc(c, orp, nrows + 1));
    DG_TRY(dalloc(c, oci, nnz));
    DG_TRY(dalloc(c, ov, nnz));
    LAUNCH(4, nrows, k_perm_count, nrows, ord, rp, cnt);
    DG_TRY(exclusive_scan(c, cnt, *orp, nrows));
    LAUNCH(4, nrows, k_perm_fill, nrows, ord, cinv, rp, ci, v, *orp, *oci, *ov);
    return Status::Ok();
}

// Padded ELL copy of a row-ordered CSR when every row has <= W entries;
// rows padded to a multiple of 224 (the largest pipelined tile, cycle.cu).
// W < 0: pick the narrowest of |W|-1 and |W| that fits (7 or 8); *wout = width used.
Status build_ell(decmg_gpu_ctx* c, int nrows, const int* rp, const int* ci, const double* v, const int* ord, int W,
                 bool diag, int** eci, double** ev, int** erow, int* wout = nullptr) {
    if (nrows >= (1 << kRowBits)) return Status::Err(DECMG_INVALID_ARGUMENT, "level too large for the ELL row ids");
    TmpPool tp(c->stream);
    int* mx;
    DG_TRY(tp.get(&mx, 1));
    DG_CUDA(cudaMemsetAsync(mx, 0, sizeof(int), c->stream));
    LAUNCH(4, nrows, k_row_maxlen, nrows, rp, mx);
    int h = 0;
    DG_TRY(read_int(c, mx, &h));
    if (W < 0) W = h <= -W - 1 ? -W - 1 : -W;
    if (wout) *wout = h > W ? 0 : W;
    if (h > W) {
        *eci = nullptr;
        *ev = nullptr;
        return Status::Ok();
    }
    const int npad = (nrows + 223) / 224 * 224;
    DG_TRY(dalloc(c, eci, static_cast<size_t>(npad) * W));
    DG_TRY(dalloc(c, ev, static_cast<size_t>(npad) * W));
    if (erow) DG_TRY(dalloc(c, erow, npad));
    LAUNCH(4, npad, k_ell_fill, nrows, npad, W, rp, ci, v, ord, diag, *eci, *ev, erow ? *erow : nullptr);
    return Status::Ok();
}

// Phases of the exact Gauss-Seidel sweeps (both directions) and their
// internal row lists, ascending within a phase (stable radix sort by phase).
}  // namespace

Status build_gs_schedule(decmg_gpu_ctx* c, Level& m) {
    TmpPool tp(c->stream);
    const int n = m.nv;
    int *pa, *pb, *changed, *key, *keys, *qin;
    DG_TRY(tp.get(&pa, n));
    DG_TRY(tp.get(&pb, n));
    DG_TRY(tp.get(&changed, 1));
    DG_TRY(tp.get(&key, n));
    DG_TRY(tp.get(&keys, n));
    DG_TRY(tp.get(&qin, n));
    for (int reverse = 0; reverse < 2; ++reverse) {
        DG_CUDA(cudaMemsetAsync(pa, 0, sizeof(int) * n, c->stream));
        int steps = 0;  // phases never exceed the number of relaxation steps
        for (;; ++steps) {
            if (steps > n) return Status::Err(DECMG_RUNTIME, "gauss_seidel: schedule did not converge");
            DG_CUDA(cudaMemsetAsync(changed, 0, sizeof(int), c->stream));
            LAUNCH(4, n, k_gs_phase_step, n, m.L_rp, m.L_ci, pa, pb, reverse, changed);
            std::swap(pa, pb);
            int h = 0;
            DG_TRY(read_int(c, changed, &h));
            if (!h) break;
        }
        LAUNCH(4, n, k_gs_keys, n, m.ord, pa, key, qin);
        int* rows = nullptr;
        DG_TRY(dalloc(c, &rows, n));
        int bits = 1;
        while ((1 << bits) <= steps) ++bits;
        size_t bytes = 0;
        DG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, keys, qin, rows, n, 0, bits, c->stream));
        char* tmp;
        DG_TRY(tp.get(&tmp, bytes));
        DG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, key, keys, qin, rows, n, 0, bits, c->stream));
        std::vector<int> hk(n);
        DG_CUDA(cudaMemcpyAsync(hk.data(), keys, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
        DG_CUDA(cudaStreamSynchronize(c->stream));
        const int nph = n ? hk[n - 1] + 1 : 0;
        std::vector<int> ptr(nph + 1, 0);
        for (int v : hk) ++ptr[v + 1];
        for (int p = 0; p < nph; ++p) ptr[p + 1] += ptr[p];
        (reverse ? m.gsr_rows : m.gsf_rows) = rows;
        (reverse ? m.gsr_ptr : m.gsf_ptr) = std::move(ptr);
    }
    return Status::Ok();
}

namespace {

// Internal numbering for every level except the coarsest (its CG runs
// sequentially in the reference order): Morton order, the renumbered L, P, R
// (common.cuh Level), their ELL copies, diag and boundary flags by internal row.
Status build_orders(decmg_gpu_ctx* c) {
    const int L = static_cast<int>(c->lv.size());
    {  // project_compatible's `total += w[i]` chain (multigrid.cpp:244-247), once
        const Level& m = c->lv[0];
        std::vector<double> a(m.nv);
        DG_CUDA(cudaMemcpy(a.data(), m.area, sizeof(double) * m.nv, cudaMemcpyDeviceToHost));
        double t = 0.0;
        for (double x : a) t += x;
        c->wtot0 = t;
    }
    for (int k = 0; k + 1 < L; ++k)
        if (c->lv[k].pos) DG_TRY(morton_order(c, c->lv[k]));
    for (int k = 0; k < L; ++k) {
        Level& m = c->lv[k];
        DG_TRY(permute_rows(c, m.nv, m.ord, m.inv, m.L_rp, m.L_ci, m.L_v, m.nnzL, &m.Lo_rp, &m.Lo_ci, &m.Lo_v));
        if (m.ord) {
            DG_TRY(dalloc(c, &m.diag_i, m.nv));
            LAUNCH(4, m.nv, k_take<double>, m.nv, m.ord, m.diag, m.diag_i);
            DG_TRY(dalloc(c, &m.area_i, m.nv));
            LAUNCH(4, m.nv, k_take<double>, m.nv, m.ord, m.area, m.area_i);
            if (m.bd) {
                DG_TRY(dalloc(c, &m.bd_i, m.nv));
                LAUNCH(4, m.nv, k_take<int>, m.nv, m.ord, m.bd, m.bd_i);
            }
        } else {
            m.diag_i = m.diag;
            m.area_i = m.area;
            m.bd_i = m.bd;
        }
        if (k + 1 < L) {
            const Level& cm = c->lv[k + 1];
            DG_TRY(permute_rows(c, m.nv, m.ord, cm.inv, m.P_rp, m.P_ci, m.P_v, m.nnzP, &m.Po_rp, &m.Po_ci, &m.Po_v));
            DG_TRY(permute_rows(c, cm.nv, cm.ord, m.inv, m.R_rp, m.R_ci, m.R_v, m.nnzR, &m.Ro_rp, &m.Ro_ci, &m.Ro_v));
        }
    }
    for (int k = 0; k + 1 < L; ++k) {  // the coarsest level only runs the sequential CG
        Level& m = c->lv[k];
        const Level& cm = c->lv[k + 1];
        DG_TRY(build_ell(c, m.nv, m.Lo_rp, m.Lo_ci, m.Lo_v, nullptr, -8, true, &m.Le_ci, &m.Le_v, &m.Le_row, &m.Le_w));
        DG_TRY(build_ell(c, m.nv, m.Po_rp, m.Po_ci, m.Po_v, nullptr, 2, false, &m.Pe_ci, &m.Pe_v, nullptr));
        DG_TRY(build_ell(c, cm.nv, m.Ro_rp, m.Ro_ci, m.Ro_v, nullptr, -8, false, &m.Re_ci, &m.Re_v, &m.Re_row,
                         &m.Re_w));
        DG_TRY(build_gs_schedule(c, m));
        if (m.Pe_ci && !m.Le_row) {  // P rows share L's row ids
            m.Pe_ci = nullptr;
            m.Pe_v = nullptr;
        }
    }
    DG_CUDA(cudaStreamSynchronize(c->stream));
    return Status::Ok();
}

}  // namespace

Status exclusive_scan(decmg_gpu_ctx* c, const int* in, int* out, int n) {
    // in has n+1 entries with in[n] == 0, so out[n] is the total.
    size_t bytes = 0;
    DG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n + 1, c->stream));
    void* tmp = nullptr;
    DG_CUDA(cudaMallocAsync(&tmp, bytes ? bytes : 1, c->stream));
    DG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n + 1, c->stream));
    DG_CUDA(cudaFreeAsync(tmp, c->stream));
    return Status::Ok();
}

Status build_from_base(decmg_gpu_ctx* c, const double* hpos, int nv, const int* hcorners, int nt,
                       int nsub, unsigned flags, int use_levels) {
    if (nv < 3 || nt < 1 || nsub < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "create_from_base: bad sizes");
    if (use_levels < 0) return Status::Err(DECMG_INVALID_ARGUMENT, "create_from_base: use_levels >= 0");
    int L = nsub + 1;
    const bool cubic = (flags & DECMG_CUBIC) != 0;
    // size guard: every count must stay inside int32 (reference uses int)
    {
        int64_t v = nv, t = nt, e = 3 * static_cast<int64_t>(nt);
        for (int k = 0; k < nsub; ++k) {
            if (cubic) {
                v = v + 2 * e + t;
                e = 3 * e + 9 * t;
                t = 9 * t;
            } else {
                v = v + e;
                e = 2 * e + 3 * t;
                t = 4 * t;
            }
        }
        if (v + 2 * e > INT32_MAX || 3 * t > INT32_MAX)
            return Status::Err(DECMG_INVALID_ARGUMENT, "create_from_base: mesh exceeds int32 indexing");
    }
    c->lv.assign(L, Level{});
    c->dirichlet = (flags & DECMG_DIRICHLET) != 0;
    const int project = (flags & DECMG_PROJECT_SPHERE) ? 1 : 0;
    double* pos;
    int* cor;
    DG_TRY(dalloc(c, &pos, 3 * static_cast<size_t>(nv)));
    DG_TRY(dalloc(c, &cor, 3 * static_cast<size_t>(nt)));
    DG_CUDA(cudaMemcpyAsync(pos, hpos, 3 * sizeof(double) * nv, cudaMemcpyHostToDevice, c->stream));
    DG_CUDA(cudaMemcpyAsync(cor, hcorners, 3 * sizeof(int) * nt, cudaMemcpyHostToDevice, c->stream));
    DG_TRY(mesh_from_triangles(c, c->lv[L - 1], pos, nv, cor, nt));
    for (int k = L - 2; k >= 0; --k) {
        const Level& cm = c->lv[k + 1];
        const int fnv = cubic ? cm.nv + 2 * cm.ne + cm.nt : cm.nv + cm.ne, fnt = (cubic ? 9 : 4) * cm.nt;
        double* fpos;
        int* fcor;
        DG_TRY(dalloc(c, &fpos, 3 * static_cast<size_t>(fnv)));
        DG_TRY(dalloc(c, &fcor, 3 * static_cast<size_t>(fnt)));
        if (cubic) {
            LAUNCH(4, fnv, k_sub_pos3, cm.nv, cm.ne, cm.nt, cm.pos, cm.edges, cm.corners, fpos, project);
            LAUNCH(4, cm.nt, k_sub_tris3, cm.nt, cm.nv, cm.ne, cm.corners, cm.tris, cm.edges, fcor);
        } else {
            LAUNCH(4, fnv, k_sub_pos, cm.nv, cm.ne, cm.pos, cm.edges, fpos, project);
            LAUNCH(4, cm.nt, k_sub_tris, cm.nt, cm.nv, cm.corners, cm.tris, fcor);
        }
        DG_TRY(mesh_from_triangles(c, c->lv[k], fpos, fnv, fcor, fnt));
    }
    // build_hierarchy's use_levels (multigrid.cpp:333-337): keep the finest
    // use_levels meshes; the coarse solve then runs on a finer mesh
    if (use_levels > 0 && use_levels < L) {
        L = use_levels;
        c->lv.resize(L);
    }
    for (int k = 0; k < L; ++k) DG_TRY(assemble(c, c->lv[k], c->dirichlet, (flags & DECMG_CLAMP_DUAL_AREAS) != 0));
    for (int k = 0; k + 1 < L; ++k) {
        Level& f = c->lv[k];
        const Level& cm = c->lv[k + 1];
        f.nnzP = cubic ? static_cast<int64_t>(cm.nv) + 4 * static_cast<int64_t>(cm.ne) + 3 * static_cast<int64_t>(cm.nt)
                       : static_cast<int64_t>(cm.nv) + 2 * static_cast<int64_t>(cm.ne);
        f.nnzR = f.nnzP;
        DG_TRY(dalloc(c, &f.P_rp, f.nv + 1));
        DG_TRY(dalloc(c, &f.P_ci, f.nnzP));
        DG_TRY(dalloc(c, &f.P_v, f.nnzP));
        DG_TRY(dalloc(c, &f.R_rp, cm.nv + 1));
        DG_TRY(dalloc(c, &f.R_ci, f.nnzR));
        DG_TRY(dalloc(c, &f.R_v, f.nnzR));
        if (cubic) {
            TmpPool tp(c->stream);
            int *vt_ptr, *vt;
            DG_TRY(incidence(c, tp, cm.nt, cm.corners, cm.nv, &vt_ptr, &vt));
            LAUNCH(4, static_cast<int64_t>(f.nv) + 1, k_P_fill3, f.nv, cm.nv, cm.ne, cm.edges, cm.corners, f.P_rp,
                   f.P_ci, f.P_v);
            LAUNCH(4, static_cast<int64_t>(cm.nv) + 1, k_R_fill3, cm.nv, cm.ne, cm.ve_ptr, cm.ve, vt_ptr, vt,
                   cm.edges, f.R_rp, f.R_ci, f.R_v);
            DG_CUDA(cudaStreamSynchronize(c->stream));
        } else {
            LAUNCH(4, static_cast<int64_t>(f.nv) + 1, k_P_fill, f.nv, cm.nv, cm.edges, f.P_rp, f.P_ci, f.P_v);
            LAUNCH(4, static_cast<int64_t>(cm.nv) + 1, k_R_fill, cm.nv, cm.ve_ptr, cm.ve, f.R_rp, f.R_ci, f.R_v);
        }
    }
    // coarsest-level weight total, sequential as PinnedDirectSolver's ctor
    // (proj/src/direct.cpp:44-45)
    {
        Level& cl = c->lv[L - 1];
        std::vector<double> a(cl.nv);
        DG_CUDA(cudaMemcpyAsync(a.data(), cl.area, sizeof(double) * cl.nv, cudaMemcpyDeviceToHost, c->stream));
        DG_CUDA(cudaStreamSynchronize(c->stream));
        double wt = 0.0;
        for (double x : a) wt += x;
        cl.wtot = wt;
    }
    DG_TRY(build_orders(c));
    DG_TRY(alloc_work(c));
    DG_CUDA(cudaStreamSynchronize(c->stream));
    return Status::Ok();
}

Status build_from_levels(decmg_gpu_ctx* c, const decmg_gpu_level_desc* d, int L, unsigned flags) {
    if (!d || L < 1) return Status::Err(DECMG_INVALID_ARGUMENT, "hierarchy: no meshes");
    c->lv.assign(L, Level{});
    c->dirichlet = (flags & DECMG_DIRICHLET) != 0;
    for (int k = 0; k < L; ++k) {
        Level& m = c->lv[k];
        const decmg_gpu_level_desc& s = d[k];
        if (s.nv < 1 || !s.L_row_ptr || !s.L_col_idx || !s.L_values || !s.dual_areas)
            return Status::Err(DECMG_INVALID_ARGUMENT, "hierarchy: incomplete level description");
        m.nv = s.nv;
        m.nnzL = s.L_nnz;
        DG_TRY(dalloc(c, &m.L_rp, m.nv + 1));
        DG_TRY(dalloc(c, &m.L_ci, m.nnzL));
        DG_TRY(dalloc(c, &m.L_v, m.nnzL));
        DG_TRY(dalloc(c, &m.area, m.nv));
        DG_TRY(dalloc(c, &m.bd, m.nv));
        DG_TRY(dalloc(c, &m.diag, m.nv));
        DG_CUDA(cudaMemcpy(m.L_rp, s.L_row_ptr, sizeof(int) * (m.nv + 1), cudaMemcpyHostToDevice));
        DG_CUDA(cudaMemcpy(m.L_ci, s.L_col_idx, sizeof(int) * m.nnzL, cudaMemcpyHostToDevice));
        DG_CUDA(cudaMemcpy(m.L_v, s.L_values, sizeof(double) * m.nnzL, cudaMemcpyHostToDevice));
        DG_CUDA(cudaMemcpy(m.area, s.dual_areas, sizeof(double) * m.nv, cudaMemcpyHostToDevice));
        std::vector<int> bd(m.nv, 0);
        if (s.boundary) bd.assign(s.boundary, s.boundary + m.nv);
        DG_CUDA(cudaMemcpy(m.bd, bd.data(), sizeof(int) * m.nv, cudaMemcpyHostToDevice));
        // diagonal_vector (sparse.cpp:188-197) and the zero-diagonal check
        std::vector<double> dg(m.nv, 0.0);
        for (int i = 0; i < m.nv; ++i)
            for (int q = s.L_row_ptr[i]; q < s.L_row_ptr[i + 1]; ++q)
                if (s.L_col_idx[q] == i) dg[i] = s.L_values[q];
        m.zero_diag_row = -1;
        for (int i = 0; i < m.nv; ++i)
            if (dg[i] == 0.0) { m.zero_diag_row = i; break; }
        DG_CUDA(cudaMemcpy(m.diag, dg.data(), sizeof(double) * m.nv, cudaMemcpyHostToDevice));
        double wt = 0.0;
        for (int i = 0; i < m.nv; ++i) wt += s.dual_areas[i];
        m.wtot = wt;
        if (k + 1 < L) {
            const int nvc = d[k + 1].nv;
            if (!s.P_row_ptr || !s.R_row_ptr)
                return Status::Err(DECMG_INVALID_ARGUMENT, "hierarchy: need one map per mesh pair");
            m.nnzP = s.P_nnz;
            m.nnzR = s.R_nnz;
            DG_TRY(dalloc(c, &m.P_rp, m.nv + 1));
            DG_TRY(dalloc(c, &m.P_ci, m.nnzP));
            DG_TRY(dalloc(c, &m.P_v, m.nnzP));
            DG_TRY(dalloc(c, &m.R_rp, nvc + 1));
            DG_TRY(dalloc(c, &m.R_ci, m.nnzR));
            DG_TRY(dalloc(c, &m.R_v, m.nnzR));
            DG_CUDA(cudaMemcpy(m.P_rp, s.P_row_ptr, sizeof(int) * (m.nv + 1), cudaMemcpyHostToDevice));
            DG_CUDA(cudaMemcpy(m.P_ci, s.P_col_idx, sizeof(int) * m.nnzP, cudaMemcpyHostToDevice));
            DG_CUDA(cudaMemcpy(m.P_v, s.P_values, sizeof(double) * m.nnzP, cudaMemcpyHostToDevice));
            DG_CUDA(cudaMemcpy(m.R_rp, s.R_row_ptr, sizeof(int) * (nvc + 1), cudaMemcpyHostToDevice));
            DG_CUDA(cudaMemcpy(m.R_ci, s.R_col_idx, sizeof(int) * m.nnzR, cudaMemcpyHostToDevice));
            DG_CUDA(cudaMemcpy(m.R_v, s.R_values, sizeof(double) * m.nnzR, cudaMemcpyHostToDevice));
        }
    }
    DG_TRY(build_orders(c));
    DG_TRY(alloc_work(c));
    return Status::Ok();
}

Status alloc_work(decmg_gpu_ctx* c) {
    const int B = c->max_nrhs;
    for (Level& m : c->lv) {
        const size_t n = static_cast<size_t>(m.nv) * B;
        DG_TRY(dalloc(c, &m.x[0], n));
        DG_TRY(dalloc(c, &m.x[1], n));
        DG_TRY(dalloc(c, &m.b, n));
    }
    const size_t n0 = static_cast<size_t>(c->lv[0].nv) * B;
    DG_TRY(dalloc(c, &c->r, n0));
    DG_TRY(dalloc(c, &c->bproj, n0));
    DG_TRY(dalloc(c, &c->xsol, n0));
    DG_TRY(dalloc(c, &c->io_b, n0));
    DG_TRY(dalloc(c, &c->io_x0, n0));
    DG_TRY(dalloc(c, &c->io_x, n0));
    int bp = 1;
    while (bp < B) bp *= 2;
    c->red_cap = 2 * ((static_cast<size_t>(c->lv[0].nv) * bp / 256 + 2) * bp + 64);
    DG_TRY(dalloc(c, &c->red, c->red_cap));
    DG_TRY(dalloc(c, &c->dsmall, 1024));
    DG_CUDA(cudaMallocHost(&c->hsmall, 1024 * sizeof(double)));
    const Level& cl = c->lv.back();
    DG_TRY(dalloc(c, &c->coarse_scratch, 4 * static_cast<size_t>(cl.nv) * B));
    return Status::Ok();
}

}  // namespace decmg_gpu
