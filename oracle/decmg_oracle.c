/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle (checker) for the DEC geometric
 * multigrid V-cycle; see decmg_oracle.h. Never linked into the product.
 *
 * Plain-C restatement of the reference `decmg` library (/root/reference/proj).
 * Every routine cites the reference lines it follows. Floating-point
 * expressions are written in the reference's evaluation order; the file is
 * compiled with -ffp-contract=off (oracle/Makefile), matching the reference
 * build, so results are bit-identical to the reference where the reference
 * is deterministic (everything except the Eigen coarse solve, replaced by the
 * documented projected weighted CG -- see oracle/ref_standin_direct.cpp).
 *
 * Data structures are flat arrays; mesh construction uses bucketed sorts
 * instead of the reference's std::set/std::map so configs up to 10.5 M
 * vertices fit in seconds, but the resulting numbering is identical
 * (pinned by tests/test_oracle_pins.py against the reference's hashes).
 */
#include "decmg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static char g_err[512];
static void set_err(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
const char* orc_last_error(void) { return g_err; }

#define NEW(T, n) ((T*)calloc((size_t)((n) > 0 ? (n) : 1), sizeof(T)))

/* ---------------------------------------------------------------- Vec3 ----
 * proj/include/decmg/geometry.hpp:12-43 (component formulas verbatim). */
typedef struct { double x, y, z; } v3;
static v3 v3_add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 v3_sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 v3_mul(v3 a, double s) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static v3 v3_div(v3 a, double s) { v3 r = {a.x / s, a.y / s, a.z / s}; return r; }
static double v3_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 v3_cross(v3 a, v3 o) {
    v3 r = {a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x};
    return r;
}
static double v3_norm2(v3 a) { return v3_dot(a, a); }
static double v3_norm(v3 a) { return sqrt(v3_norm2(a)); }
static v3 v3_mid(v3 a, v3 b) { return v3_mul(v3_add(a, b), 0.5); } /* geometry.hpp:31 */
static v3 v3_at(const double* p, int i) { v3 r = {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; return r; }

/* proj/src/geometry.cpp:5-16 */
static int circumcenter(v3 p0, v3 p1, v3 p2, v3* out) {
    const v3 a = v3_sub(p1, p0);
    const v3 b = v3_sub(p2, p0);
    const v3 n = v3_cross(a, b);
    const double n2 = v3_norm2(n);
    if (n2 <= 1e-28 * v3_norm2(a) * v3_norm2(b)) return -1;
    const v3 num = v3_add(v3_mul(v3_cross(b, n), v3_norm2(a)), v3_mul(v3_cross(n, a), v3_norm2(b)));
    *out = v3_add(p0, v3_div(num, 2.0 * n2));
    return 0;
}

/* ---------------------------------------------------------------- FNV ---- */
/* proj/src/mesh.cpp:11-19 */
static uint64_t fnv1a(const void* data, size_t n, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}
uint64_t orc_fnv(const void* data, int64_t nbytes) {
    return fnv1a(data, (size_t)nbytes, 1469598103934665603ULL);
}

/* ---------------------------------------------------------------- mesh --- */
typedef struct {
    int nv, ne, nt;
    double* pos;   /* [nv][3] */
    int* edges;    /* [ne][2] src < tgt, lexicographic */
    int* tris;     /* [nt][3] edge triple (e0,e1,e2), e_i opposite corner i */
    int* corners;  /* [nt][3] (v0,v1,v2) */
    int* ve_ptr;   /* vertex -> incident edges, ascending (mesh.cpp:99-104) */
    int* ve;
    int* et_ptr;   /* edge -> incident triangles, ascending (mesh.cpp:105-110) */
    int* et;
    int* eptr;     /* edges with src == v are eptr[v] .. eptr[v+1]-1 */
    uint64_t hash;
} mesh_t;

static void mesh_free(mesh_t* m) {
    free(m->pos); free(m->edges); free(m->tris); free(m->corners);
    free(m->ve_ptr); free(m->ve); free(m->et_ptr); free(m->et); free(m->eptr);
    memset(m, 0, sizeof *m);
}

/* edge id of unordered pair (a, b); -1 if absent (EmbeddedComplex2D::find_edge,
 * mesh.cpp:60-63). Binary search inside the src bucket. */
static int find_edge(const mesh_t* m, int a, int b) {
    int s = a < b ? a : b, t = a < b ? b : a;
    int lo = m->eptr[s], hi = m->eptr[s + 1] - 1;
    while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        int v = m->edges[2 * mid + 1];
        if (v == t) return mid;
        if (v < t) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* EmbeddedComplex2D::from_triangles (proj/src/mesh.cpp:122-157) + finalize
 * (72-120). Edges = unique (min,max) pairs in lexicographic order; triangle
 * t stores {e(v1,v2), e(v0,v2), e(v0,v1)}. Takes ownership of pos. */
static int mesh_from_triangles(mesh_t* m, double* pos, int nv, const int* corner, int nt) {
    memset(m, 0, sizeof *m);
    m->nv = nv; m->nt = nt; m->pos = pos;
    for (int t = 0; t < nt; ++t)
        for (int i = 0; i < 3; ++i) {
            int a = corner[3 * t + i], b = corner[3 * t + (i + 1) % 3];
            if (a < 0 || a >= nv || b < 0 || b >= nv || a == b) {
                set_err("from_triangles: bad corner triple");
                return -1;
            }
        }
    /* bucket every corner pair by its min vertex */
    int* cnt = NEW(int, nv + 1);
    for (int t = 0; t < nt; ++t)
        for (int i = 0; i < 3; ++i) {
            int a = corner[3 * t + i], b = corner[3 * t + (i + 1) % 3];
            cnt[(a < b ? a : b) + 1]++;
        }
    for (int v = 0; v < nv; ++v) cnt[v + 1] += cnt[v];
    int* fill = NEW(int, nv);
    int* bucket = NEW(int, 3 * (size_t)nt);
    for (int t = 0; t < nt; ++t)
        for (int i = 0; i < 3; ++i) {
            int a = corner[3 * t + i], b = corner[3 * t + (i + 1) % 3];
            int s = a < b ? a : b, u = a < b ? b : a;
            bucket[cnt[s] + fill[s]++] = u;
        }
    /* sort + unique each bucket */
    m->eptr = NEW(int, nv + 1);
    for (int v = 0; v < nv; ++v) {
        int lo = cnt[v], hi = cnt[v + 1];
        for (int i = lo + 1; i < hi; ++i) {
            int key = bucket[i], j = i - 1;
            while (j >= lo && bucket[j] > key) { bucket[j + 1] = bucket[j]; --j; }
            bucket[j + 1] = key;
        }
        int u = 0;
        for (int i = lo; i < hi; ++i)
            if (i == lo || bucket[i] != bucket[i - 1]) bucket[lo + u++] = bucket[i];
        m->eptr[v + 1] = m->eptr[v] + u;
    }
    m->ne = m->eptr[nv];
    m->edges = NEW(int, 2 * (size_t)m->ne);
    for (int v = 0; v < nv; ++v)
        for (int e = m->eptr[v]; e < m->eptr[v + 1]; ++e) {
            m->edges[2 * e] = v;
            m->edges[2 * e + 1] = bucket[cnt[v] + (e - m->eptr[v])];
        }
    free(cnt); free(fill); free(bucket);
    m->tris = NEW(int, 3 * (size_t)nt);
    m->corners = NEW(int, 3 * (size_t)nt);
    for (int t = 0; t < nt; ++t) {
        const int v0 = corner[3 * t], v1 = corner[3 * t + 1], v2 = corner[3 * t + 2];
        m->tris[3 * t] = find_edge(m, v1, v2);
        m->tris[3 * t + 1] = find_edge(m, v0, v2);
        m->tris[3 * t + 2] = find_edge(m, v0, v1);
        m->corners[3 * t] = v0; m->corners[3 * t + 1] = v1; m->corners[3 * t + 2] = v2;
    }
    /* finalize: vertex -> edges, edge -> triangles (mesh.cpp:99-110) */
    m->ve_ptr = NEW(int, nv + 1);
    for (int e = 0; e < m->ne; ++e) { m->ve_ptr[m->edges[2 * e] + 1]++; m->ve_ptr[m->edges[2 * e + 1] + 1]++; }
    for (int v = 0; v < nv; ++v) m->ve_ptr[v + 1] += m->ve_ptr[v];
    m->ve = NEW(int, 2 * (size_t)m->ne);
    int* f2 = NEW(int, nv);
    for (int e = 0; e < m->ne; ++e)
        for (int j = 0; j < 2; ++j) {
            int v = m->edges[2 * e + j];
            m->ve[m->ve_ptr[v] + f2[v]++] = e;
        }
    free(f2);
    m->et_ptr = NEW(int, m->ne + 1);
    for (int t = 0; t < nt; ++t)
        for (int j = 0; j < 3; ++j) m->et_ptr[m->tris[3 * t + j] + 1]++;
    for (int e = 0; e < m->ne; ++e) m->et_ptr[e + 1] += m->et_ptr[e];
    m->et = NEW(int, 3 * (size_t)nt);
    int* f3 = NEW(int, m->ne);
    for (int t = 0; t < nt; ++t)
        for (int j = 0; j < 3; ++j) {
            int e = m->tris[3 * t + j];
            m->et[m->et_ptr[e] + f3[e]++] = t;
        }
    free(f3);
    /* content hash (mesh.cpp:112-119) */
    uint64_t h = 1469598103934665603ULL;
    const int counts[3] = {nv, m->ne, nt};
    h = fnv1a(counts, sizeof counts, h);
    if (nv) h = fnv1a(m->pos, (size_t)nv * 3 * sizeof(double), h);
    if (m->ne) h = fnv1a(m->edges, (size_t)m->ne * 2 * sizeof(int), h);
    if (nt) h = fnv1a(m->tris, (size_t)nt * 3 * sizeof(int), h);
    m->hash = h;
    return 0;
}

/* make_triangulated_grid (proj/src/mesh.cpp:232-257) */
static int base_grid(mesh_t* m, int nx, int ny, double lx, double ly) {
    if (nx < 1 || ny < 1 || lx <= 0 || ly <= 0) { set_err("make_triangulated_grid: bad args"); return -1; }
    const int nv = (nx + 1) * (ny + 1);
    double* pos = NEW(double, 3 * (size_t)nv);
    const double dx = lx / nx, dy = ly / ny;
    int k = 0;
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
            pos[3 * k] = i * dx; pos[3 * k + 1] = j * dy; pos[3 * k + 2] = 0.0; ++k;
        }
    int* tri = NEW(int, 6 * (size_t)nx * ny);
    int t = 0;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const int bl = j * (nx + 1) + i, br = j * (nx + 1) + i + 1;
            const int tr = (j + 1) * (nx + 1) + i + 1, tl = (j + 1) * (nx + 1) + i;
            tri[3 * t] = bl; tri[3 * t + 1] = br; tri[3 * t + 2] = tr; ++t;
            tri[3 * t] = bl; tri[3 * t + 1] = tr; tri[3 * t + 2] = tl; ++t;
        }
    int rc = mesh_from_triangles(m, pos, nv, tri, t);
    free(tri);
    return rc;
}

/* make_equilateral_grid (proj/src/mesh.cpp:259-291) */
static int base_equi(mesh_t* m, int rows, int cols, double side) {
    if (rows < 1 || cols < 1 || side <= 0 || (cols % 2 != 0 && rows > 1)) {
        set_err("make_equilateral_grid: bad args");
        return -1;
    }
    const int nup = (cols + 1) / 2, ndown = cols / 2, row_verts = nup + 1;
    const double hy = side * sqrt(3.0) / 2.0;
    double* pos = NEW(double, 3 * (size_t)(rows + 1) * row_verts);
    int nv = 0;
    for (int j = 0; j <= rows; ++j) {
        const int count = (j == rows && ndown < nup) ? ndown + 1 : row_verts;
        for (int i = 0; i < count; ++i) {
            pos[3 * nv] = i * side + j * side / 2.0; pos[3 * nv + 1] = j * hy; pos[3 * nv + 2] = 0.0; ++nv;
        }
    }
    int* tri = NEW(int, 3 * (size_t)rows * cols);
    int t = 0;
#define VID(i, j) ((j) * row_verts + (i))
    for (int j = 0; j < rows; ++j) {
        for (int i = 0; i < nup; ++i) {
            tri[3 * t] = VID(i, j); tri[3 * t + 1] = VID(i + 1, j); tri[3 * t + 2] = VID(i, j + 1); ++t;
        }
        for (int i = 0; i < ndown; ++i) {
            tri[3 * t] = VID(i + 1, j); tri[3 * t + 1] = VID(i + 1, j + 1); tri[3 * t + 2] = VID(i, j + 1); ++t;
        }
    }
#undef VID
    int rc = mesh_from_triangles(m, pos, nv, tri, t);
    free(tri);
    return rc;
}

/* Extension x2: canonical icosahedron, vertices (0,+-1,+-phi)
 * cyclic, each scaled by 1.0/|p|; 20 outward counter-clockwise faces. */
static const int kIcoFaces[20][3] = {
    {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11}, {1, 5, 9},  {5, 11, 4},
    {11, 10, 2}, {10, 7, 6}, {7, 1, 8},  {3, 9, 4},  {3, 4, 2},   {3, 2, 6},  {3, 6, 8},
    {3, 8, 9},  {4, 9, 5},  {2, 4, 11}, {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
static int base_ico(mesh_t* m) {
    const double phi = (1.0 + sqrt(5.0)) / 2.0;
    const double raw[12][3] = {{-1, phi, 0}, {1, phi, 0},  {-1, -phi, 0}, {1, -phi, 0},
                               {0, -1, phi}, {0, 1, phi},  {0, -1, -phi}, {0, 1, -phi},
                               {phi, 0, -1}, {phi, 0, 1},  {-phi, 0, -1}, {-phi, 0, 1}};
    double* pos = NEW(double, 36);
    for (int i = 0; i < 12; ++i) {
        v3 p = {raw[i][0], raw[i][1], raw[i][2]};
        const double s = 1.0 / v3_norm(p);
        p = v3_mul(p, s);
        pos[3 * i] = p.x; pos[3 * i + 1] = p.y; pos[3 * i + 2] = p.z;
    }
    return mesh_from_triangles(m, pos, 12, &kIcoFaces[0][0], 20);
}

/* subdivide_nary with n = 2 (proj/src/subdivision.cpp:12-110): copies first,
 * then one midpoint per coarse edge p_s*0.5 + p_t*0.5 (36-37), four children
 * per parent [v0,m01,m02],[m01,m12,m02],[m02,m12,v2],[m01,v1,m12] (89-103).
 * project != 0: extension x2, midpoints scaled by 1.0/|p|. */
static int binary_subdivide(const mesh_t* c, mesh_t* f, int project) {
    const int nv = c->nv, ne = c->ne, nt = c->nt;
    const int fnv = nv + ne;
    double* pos = NEW(double, 3 * (size_t)fnv);
    memcpy(pos, c->pos, (size_t)nv * 3 * sizeof(double));
    for (int e = 0; e < ne; ++e) {
        const v3 ps = v3_at(c->pos, c->edges[2 * e]), pt = v3_at(c->pos, c->edges[2 * e + 1]);
        const double tk = 1.0 / 2;
        v3 p = v3_add(v3_mul(ps, 1.0 - tk), v3_mul(pt, tk));
        if (project) {
            const double inv = 1.0 / v3_norm(p);
            p = v3_mul(p, inv);
        }
        pos[3 * (nv + e)] = p.x; pos[3 * (nv + e) + 1] = p.y; pos[3 * (nv + e) + 2] = p.z;
    }
    int* tri = NEW(int, 12 * (size_t)nt);
    for (int t = 0; t < nt; ++t) {
        const int v0 = c->corners[3 * t], v1 = c->corners[3 * t + 1], v2 = c->corners[3 * t + 2];
        const int m12 = nv + c->tris[3 * t], m02 = nv + c->tris[3 * t + 1], m01 = nv + c->tris[3 * t + 2];
        const int ch[4][3] = {{v0, m01, m02}, {m01, m12, m02}, {m02, m12, v2}, {m01, v1, m12}};
        memcpy(tri + 12 * (size_t)t, ch, sizeof ch);
    }
    int rc = mesh_from_triangles(f, pos, fnv, tri, 4 * nt);
    free(tri);
    return rc;
}

/* subdivide_nary with n = 3, "cubic" (proj/src/subdivision.cpp:12-110,
 * 116-120): copies; two points per coarse edge at p_s*(1-t_k) + p_t*t_k,
 * t_k = k/3 (k = 1, 2; ids nv + 2e + k - 1); one point per triangle at
 * (p0*b0 + p1*b1) + p2*b2 with b1 = b2 = 1/3, b0 = 1 - b1 - b2 (id
 * nv + 2ne + t); nine children per parent over the barycentric lattice
 * (lattice_vertex, 63-87; loop 89-103). project != 0: every new point scaled
 * by 1.0/|p| (extension x2 for the icosphere). Also returns the map columns
 * (fine vertex -> up to 3 (coarse vertex, weight) pairs, unsorted) for
 * build_transfers_nary. */
typedef struct { int n; int v[3]; double w[3]; } mcol_t;

static int cubic_lattice(const mesh_t* c, int t, int i, int j) {
    const int n = 3, nv = c->nv;
    const int v0 = c->corners[3 * t], v1 = c->corners[3 * t + 1], v2 = c->corners[3 * t + 2];
    const int k0 = n - i - j;
    if (i == 0 && j == 0) return v0;
    if (k0 == 0 && j == 0) return v1;
    if (k0 == 0 && i == 0) return v2;
    int a, b, k;
    if (j == 0) { a = v0; b = v1; k = i; }
    else if (i == 0) { a = v0; b = v2; k = j; }
    else if (k0 == 0) { a = v1; b = v2; k = j; }
    else return nv + 2 * c->ne + t;  /* the single interior point of n = 3 */
    const int e = find_edge(c, a, b);
    const int step = c->edges[2 * e] == a ? k : n - k;
    return nv + e * 2 + (step - 1);
}

static int cubic_subdivide(const mesh_t* c, mesh_t* f, int project, mcol_t** cols_out) {
    const int nv = c->nv, ne = c->ne, nt = c->nt;
    const int fnv = nv + 2 * ne + nt;
    double* pos = NEW(double, 3 * (size_t)fnv);
    mcol_t* cols = NEW(mcol_t, fnv);
    memcpy(pos, c->pos, (size_t)nv * 3 * sizeof(double));
    for (int v = 0; v < nv; ++v) { cols[v].n = 1; cols[v].v[0] = v; cols[v].w[0] = 1.0; }
    for (int e = 0; e < ne; ++e) {
        const int s = c->edges[2 * e], t = c->edges[2 * e + 1];
        const v3 ps = v3_at(c->pos, s), pt = v3_at(c->pos, t);
        for (int k = 1; k <= 2; ++k) {
            const double tk = (double)k / 3;
            v3 p = v3_add(v3_mul(ps, 1.0 - tk), v3_mul(pt, tk));
            if (project) p = v3_mul(p, 1.0 / v3_norm(p));
            const int j = nv + 2 * e + (k - 1);
            pos[3 * j] = p.x; pos[3 * j + 1] = p.y; pos[3 * j + 2] = p.z;
            cols[j].n = 2; cols[j].v[0] = s; cols[j].w[0] = 1.0 - tk; cols[j].v[1] = t; cols[j].w[1] = tk;
        }
    }
    for (int t = 0; t < nt; ++t) {
        const int v0 = c->corners[3 * t], v1 = c->corners[3 * t + 1], v2 = c->corners[3 * t + 2];
        const double b1 = 1.0 / 3, b2 = 1.0 / 3, b0 = 1.0 - b1 - b2;
        v3 p = v3_add(v3_add(v3_mul(v3_at(c->pos, v0), b0), v3_mul(v3_at(c->pos, v1), b1)),
                      v3_mul(v3_at(c->pos, v2), b2));
        if (project) p = v3_mul(p, 1.0 / v3_norm(p));
        const int j = nv + 2 * ne + t;
        pos[3 * j] = p.x; pos[3 * j + 1] = p.y; pos[3 * j + 2] = p.z;
        cols[j].n = 3;
        cols[j].v[0] = v0; cols[j].w[0] = b0;
        cols[j].v[1] = v1; cols[j].w[1] = b1;
        cols[j].v[2] = v2; cols[j].w[2] = b2;
    }
    int* tri = NEW(int, 27 * (size_t)nt);
    int q = 0;
    for (int t = 0; t < nt; ++t)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; i + j < 3; ++j) {
                tri[q++] = cubic_lattice(c, t, i, j);
                tri[q++] = cubic_lattice(c, t, i + 1, j);
                tri[q++] = cubic_lattice(c, t, i, j + 1);
                if (i + j < 2) {
                    tri[q++] = cubic_lattice(c, t, i + 1, j);
                    tri[q++] = cubic_lattice(c, t, i + 1, j + 1);
                    tri[q++] = cubic_lattice(c, t, i, j + 1);
                }
            }
    int rc = mesh_from_triangles(f, pos, fnv, tri, 9 * nt);
    free(tri);
    if (rc) { free(cols); return rc; }
    *cols_out = cols;
    return 0;
}

/* ---------------------------------------------------------------- level -- */
typedef struct {
    mesh_t m;
    double* area;          /* dual cell areas = diag(star0) */
    int* bd;               /* boundary flag (extension x1) */
    int* L_rp; int* L_ci; double* L_v; int64_t nnzL;
    double* diag;
    int* P_rp; int* P_ci; double* P_v; int64_t nnzP;   /* to next coarser level */
    int* R_rp; int* R_ci; double* R_v; int64_t nnzR;
} level_t;

struct orc_hier {
    int L;
    int dirichlet;
    level_t* lv;
    double wtot_coarse;
};

/* build_dual (proj/src/dual.cpp:7-63) + hodge_star_1 (operators.cpp:68-79) +
 * hodge_star_0_inv (81-100) + laplacian_0 (102-122) via multiply/scaled/
 * scale_rows (sparse.cpp:117-180). Resulting entries, derived in DESIGN.md:
 *   L_ij = ((0.0 + (-w_e)) * -1.0) * (1.0/A_i)
 *   L_ii = ((((0.0 + w_e1) + w_e2) + ...) * -1.0) * (1.0/A_i), edges ascending. */
static int assemble_level(level_t* lv, int dirichlet) {
    mesh_t* m = &lv->m;
    const int nv = m->nv, ne = m->ne, nt = m->nt;
    v3* mid = NEW(v3, ne);
    double* plen = NEW(double, ne);
    for (int e = 0; e < ne; ++e) {
        const v3 a = v3_at(m->pos, m->edges[2 * e]), b = v3_at(m->pos, m->edges[2 * e + 1]);
        mid[e] = v3_mid(a, b);
        plen[e] = v3_norm(v3_sub(b, a));
        if (plen[e] <= 0.0) { set_err("build_dual: zero-length edge %d", e); return -1; }
    }
    double* dlen = NEW(double, ne);
    lv->area = NEW(double, nv);
    for (int t = 0; t < nt; ++t) {
        const int v0 = m->corners[3 * t], v1 = m->corners[3 * t + 1], v2 = m->corners[3 * t + 2];
        const v3 p0 = v3_at(m->pos, v0), p1 = v3_at(m->pos, v1), p2 = v3_at(m->pos, v2);
        v3 cc;
        if (circumcenter(p0, p1, p2, &cc)) { set_err("circumcenter: degenerate triangle"); return -1; }
        const v3 n = v3_cross(v3_sub(p1, p0), v3_sub(p2, p0));
        const double area2 = v3_norm(n);
        const v3 nhat = v3_div(n, area2);
        for (int j = 0; j < 3; ++j) {
            const int e = m->tris[3 * t + j];
            dlen[e] += v3_norm(v3_sub(cc, mid[e]));
        }
        const v3 p[3] = {p0, p1, p2};
        const int vid[3] = {v0, v1, v2};
        for (int i = 0; i < 3; ++i) {
            const int j = (i + 1) % 3;
            const v3 mm = v3_mid(p[i], p[j]);
            const double wi = 0.5 * v3_dot(v3_cross(v3_sub(mm, p[i]), v3_sub(cc, p[i])), nhat);
            const double wj = 0.5 * v3_dot(v3_cross(v3_sub(p[j], mm), v3_sub(cc, mm)), nhat);
            lv->area[vid[i]] += wi;
            lv->area[vid[j]] += wj;
        }
    }
    double* w = NEW(double, ne);
    for (int e = 0; e < ne; ++e) w[e] = dlen[e] / plen[e];
    double* inv = NEW(double, nv);
    for (int v = 0; v < nv; ++v) {
        if (lv->area[v] <= 0.0) {
            set_err("hodge_star_0_inv: non-well-centered dual cell at vertex %d", v);
            return -1;
        }
        inv[v] = 1.0 / lv->area[v];
    }
    /* boundary: endpoints of edges with exactly one triangle (x1) */
    lv->bd = NEW(int, nv);
    for (int e = 0; e < ne; ++e)
        if (m->et_ptr[e + 1] - m->et_ptr[e] == 1) {
            lv->bd[m->edges[2 * e]] = 1;
            lv->bd[m->edges[2 * e + 1]] = 1;
        }
    /* CSR: row i = {i} U neighbours ascending; neighbour order == incident
     * edge id order (edges are lexicographic). */
    lv->nnzL = (int64_t)nv + 2 * (int64_t)ne;
    lv->L_rp = NEW(int, nv + 1);
    lv->L_ci = NEW(int, lv->nnzL);
    lv->L_v = NEW(double, lv->nnzL);
    lv->diag = NEW(double, nv);
    int64_t k = 0;
    for (int i = 0; i < nv; ++i) {
        lv->L_rp[i] = (int)k;
        double sum = 0.0;
        for (int q = m->ve_ptr[i]; q < m->ve_ptr[i + 1]; ++q) sum += w[m->ve[q]];
        const double dval = (sum * -1.0) * inv[i];
        int placed = 0;
        for (int q = m->ve_ptr[i]; q < m->ve_ptr[i + 1]; ++q) {
            const int e = m->ve[q];
            const int j = m->edges[2 * e] == i ? m->edges[2 * e + 1] : m->edges[2 * e];
            if (!placed && j > i) {
                lv->L_ci[k] = i; lv->L_v[k] = dval; ++k; placed = 1;
            }
            const double a = 0.0 + (-w[e]);
            lv->L_ci[k] = j;
            lv->L_v[k] = (a * -1.0) * inv[i];
            ++k;
        }
        if (!placed) { lv->L_ci[k] = i; lv->L_v[k] = dval; ++k; }
    }
    lv->L_rp[nv] = (int)k;
    if (dirichlet) {
        for (int i = 0; i < nv; ++i)
            if (lv->bd[i])
                for (int q = lv->L_rp[i]; q < lv->L_rp[i + 1]; ++q) lv->L_v[q] = lv->L_ci[q] == i ? 1.0 : 0.0;
    }
    for (int i = 0; i < nv; ++i)
        for (int q = lv->L_rp[i]; q < lv->L_rp[i + 1]; ++q)
            if (lv->L_ci[q] == i) lv->diag[i] = lv->L_v[q];
    free(mid); free(plen); free(dlen); free(w); free(inv);
    return 0;
}

/* P = M(f)^T (multigrid.cpp:215) and R = rownormalize(M(f))
 * (geometric_map.cpp:205-223) for a binary subdivision fine -> coarse. */
static void build_transfers(level_t* fine, const level_t* coarse) {
    const mesh_t* c = &coarse->m;
    const int nvc = c->nv, nvf = fine->m.nv;
    fine->nnzP = (int64_t)nvc + 2 * (int64_t)c->ne;
    fine->P_rp = NEW(int, nvf + 1);
    fine->P_ci = NEW(int, fine->nnzP);
    fine->P_v = NEW(double, fine->nnzP);
    int64_t k = 0;
    for (int j = 0; j < nvf; ++j) {
        fine->P_rp[j] = (int)k;
        if (j < nvc) {
            fine->P_ci[k] = j; fine->P_v[k] = 1.0; ++k;
        } else {
            const int e = j - nvc;
            fine->P_ci[k] = c->edges[2 * e]; fine->P_v[k] = 0.5; ++k;
            fine->P_ci[k] = c->edges[2 * e + 1]; fine->P_v[k] = 0.5; ++k;
        }
    }
    fine->P_rp[nvf] = (int)k;
    fine->nnzR = fine->nnzP;
    fine->R_rp = NEW(int, nvc + 1);
    fine->R_ci = NEW(int, fine->nnzR);
    fine->R_v = NEW(double, fine->nnzR);
    k = 0;
    for (int i = 0; i < nvc; ++i) {
        fine->R_rp[i] = (int)k;
        double rs = 0.0;
        rs += 1.0;
        for (int q = c->ve_ptr[i]; q < c->ve_ptr[i + 1]; ++q) rs += 0.5;
        const double inv = 1.0 / rs;
        fine->R_ci[k] = i; fine->R_v[k] = 1.0 * inv; ++k;
        for (int q = c->ve_ptr[i]; q < c->ve_ptr[i + 1]; ++q) {
            fine->R_ci[k] = nvc + c->ve[q]; fine->R_v[k] = 0.5 * inv; ++k;
        }
    }
    fine->R_rp[nvc] = (int)k;
}

/* P = M(f)^T and R = rownormalize(M(f)) from general map columns
 * (GeometricMap::make, geometric_map.cpp:18-42: drop |w| <= 1e-12, renormalise
 * by the column's sequential sum when |sum - 1| <= 1e-9, sort by vertex;
 * matrix / transposed, sparse.cpp:90-115; restriction_matrix 205-223: row sums
 * accumulated over fine columns in ascending order, inv = 1.0/sum,
 * R_ij = M_ij * inv). */
static void build_transfers_nary(level_t* fine, const level_t* coarse, mcol_t* cols) {
    const int nvc = coarse->m.nv, nvf = fine->m.nv;
    int64_t nnz = 0;
    for (int j = 0; j < nvf; ++j) {
        mcol_t* c = &cols[j];
        mcol_t k;
        k.n = 0;
        double sum = 0.0;
        for (int a = 0; a < c->n; ++a) {
            if (fabs(c->w[a]) <= 1e-12) continue;
            k.v[k.n] = c->v[a]; k.w[k.n] = c->w[a]; ++k.n;
            sum += c->w[a];
        }
        if (fabs(sum - 1.0) <= 1e-9 && sum != 0.0)
            for (int a = 0; a < k.n; ++a) k.w[a] /= sum;
        for (int a = 1; a < k.n; ++a)  /* sort by (vertex, weight) */
            for (int b = a; b > 0 && (k.v[b] < k.v[b - 1] || (k.v[b] == k.v[b - 1] && k.w[b] < k.w[b - 1])); --b) {
                int tv = k.v[b]; k.v[b] = k.v[b - 1]; k.v[b - 1] = tv;
                double tw = k.w[b]; k.w[b] = k.w[b - 1]; k.w[b - 1] = tw;
            }
        *c = k;
        nnz += k.n;
    }
    fine->nnzP = fine->nnzR = nnz;
    fine->P_rp = NEW(int, nvf + 1);
    fine->P_ci = NEW(int, nnz);
    fine->P_v = NEW(double, nnz);
    int64_t q = 0;
    for (int j = 0; j < nvf; ++j) {
        fine->P_rp[j] = (int)q;
        for (int a = 0; a < cols[j].n; ++a) { fine->P_ci[q] = cols[j].v[a]; fine->P_v[q] = cols[j].w[a]; ++q; }
    }
    fine->P_rp[nvf] = (int)q;
    /* R: rows = coarse vertices, columns (fine j) ascending */
    fine->R_rp = NEW(int, nvc + 1);
    fine->R_ci = NEW(int, nnz);
    fine->R_v = NEW(double, nnz);
    int* cnt = NEW(int, nvc + 1);
    memset(cnt, 0, sizeof(int) * (nvc + 1));
    for (int64_t e = 0; e < nnz; ++e) ++cnt[fine->P_ci[e] + 1];
    for (int i = 0; i < nvc; ++i) cnt[i + 1] += cnt[i];
    memcpy(fine->R_rp, cnt, sizeof(int) * (nvc + 1));
    double* rs = NEW(double, nvc);
    for (int i = 0; i < nvc; ++i) rs[i] = 0.0;
    for (int j = 0; j < nvf; ++j)
        for (int a = fine->P_rp[j]; a < fine->P_rp[j + 1]; ++a) {
            const int i = fine->P_ci[a];
            fine->R_ci[cnt[i]] = j;
            fine->R_v[cnt[i]] = fine->P_v[a];
            ++cnt[i];
            rs[i] += fine->P_v[a];
        }
    for (int i = 0; i < nvc; ++i) {
        const double inv = 1.0 / rs[i];
        for (int a = fine->R_rp[i]; a < fine->R_rp[i + 1]; ++a) fine->R_v[a] = fine->R_v[a] * inv;
    }
    free(cnt); free(rs);
}

static void level_free(level_t* lv) {
    mesh_free(&lv->m);
    free(lv->area); free(lv->bd); free(lv->L_rp); free(lv->L_ci); free(lv->L_v); free(lv->diag);
    free(lv->P_rp); free(lv->P_ci); free(lv->P_v); free(lv->R_rp); free(lv->R_ci); free(lv->R_v);
}

void orc_free(orc_hier* h) {
    if (!h) return;
    for (int k = 0; k < h->L; ++k) level_free(&h->lv[k]);
    free(h->lv);
    free(h);
}

/* subdivision_tower + build_hierarchy (subdivision.cpp:127-139,
 * multigrid.cpp:196-238,325-341): levels finest first, level L-1 = base. */
orc_hier* orc_build(const char* base, int nsub, int dirichlet) {
    if (nsub < 0) { set_err("nsub >= 0"); return NULL; }
    orc_hier* h = (orc_hier*)calloc(1, sizeof *h);
    h->L = nsub + 1;
    h->dirichlet = dirichlet;
    h->lv = (level_t*)calloc((size_t)h->L, sizeof(level_t));
    int project = 0, rc, cubic = 0;
    char spec[256];
    snprintf(spec, sizeof spec, "%s", base);
    const size_t sl = strlen(spec);
    if (sl > 6 && strcmp(spec + sl - 6, "+cubic") == 0) {  /* SubdivisionScheme::Cubic */
        cubic = 1;
        spec[sl - 6] = 0;
    }
    base = spec;
    mesh_t* b = &h->lv[h->L - 1].m;
    if (strcmp(base, "square") == 0) {
        rc = base_grid(b, 1, 1, 1.0, 1.0);
    } else if (strcmp(base, "ico") == 0) {
        rc = base_ico(b);
        project = 1;
    } else if (strncmp(base, "grid:", 5) == 0) {
        int nx, ny; double lx, ly;
        if (sscanf(base, "grid:%d:%d:%lf:%lf", &nx, &ny, &lx, &ly) != 4) { set_err("bad grid spec"); orc_free(h); return NULL; }
        rc = base_grid(b, nx, ny, lx, ly);
    } else if (strncmp(base, "equi:", 5) == 0) {
        int r, c; double s;
        if (sscanf(base, "equi:%d:%d:%lf", &r, &c, &s) != 3) { set_err("bad equi spec"); orc_free(h); return NULL; }
        rc = base_equi(b, r, c, s);
    } else {
        set_err("unknown base %s", base);
        orc_free(h);
        return NULL;
    }
    if (rc) { orc_free(h); return NULL; }
    mcol_t** cols = cubic ? (mcol_t**)calloc((size_t)h->L, sizeof(mcol_t*)) : NULL;
    for (int k = h->L - 2; k >= 0; --k) {
        rc = cubic ? cubic_subdivide(&h->lv[k + 1].m, &h->lv[k].m, project, &cols[k])
                   : binary_subdivide(&h->lv[k + 1].m, &h->lv[k].m, project);
        if (rc) break;
    }
    for (int k = 0; !rc && k < h->L; ++k) rc = assemble_level(&h->lv[k], dirichlet);
    for (int k = 0; !rc && k + 1 < h->L; ++k) {
        if (cubic) build_transfers_nary(&h->lv[k], &h->lv[k + 1], cols[k]);
        else build_transfers(&h->lv[k], &h->lv[k + 1]);
    }
    if (cols) {
        for (int k = 0; k < h->L; ++k) free(cols[k]);
        free(cols);
    }
    if (rc) { orc_free(h); return NULL; }
    const level_t* cl = &h->lv[h->L - 1];
    h->wtot_coarse = 0.0;
    for (int i = 0; i < cl->m.nv; ++i) h->wtot_coarse += cl->area[i];
    return h;
}

int orc_levels(const orc_hier* h) { return h->L; }

void orc_level_info(const orc_hier* h, int k, int64_t* counts, uint64_t* hash) {
    const level_t* lv = &h->lv[k];
    counts[0] = lv->m.nv; counts[1] = lv->m.ne; counts[2] = lv->m.nt; counts[3] = lv->nnzL;
    *hash = lv->m.hash;
}

int64_t orc_level_nnz(const orc_hier* h, int k, const char* op) {
    const level_t* lv = &h->lv[k];
    if (op[0] == 'L') return lv->nnzL;
    if (op[0] == 'P') return lv->nnzP;
    if (op[0] == 'R') return lv->nnzR;
    return -1;
}

#define COPY_OUT(ptr, n, T) do { if (!(ptr)) return -1; if (out) memcpy(out, ptr, (size_t)(n) * sizeof(T)); return (int64_t)(n); } while (0)
int64_t orc_get(const orc_hier* h, int k, const char* name, void* out) {
    if (k < 0 || k >= h->L) return -1;
    const level_t* lv = &h->lv[k];
    const int nv = lv->m.nv;
    const int nvc = k + 1 < h->L ? h->lv[k + 1].m.nv : 0;
    if (!strcmp(name, "positions")) COPY_OUT(lv->m.pos, 3 * (int64_t)nv, double);
    if (!strcmp(name, "edges")) COPY_OUT(lv->m.edges, 2 * (int64_t)lv->m.ne, int);
    if (!strcmp(name, "triangles")) COPY_OUT(lv->m.tris, 3 * (int64_t)lv->m.nt, int);
    if (!strcmp(name, "corners")) COPY_OUT(lv->m.corners, 3 * (int64_t)lv->m.nt, int);
    if (!strcmp(name, "dual_areas")) COPY_OUT(lv->area, nv, double);
    if (!strcmp(name, "boundary")) COPY_OUT(lv->bd, nv, int);
    if (!strcmp(name, "L_rp")) COPY_OUT(lv->L_rp, nv + 1, int);
    if (!strcmp(name, "L_ci")) COPY_OUT(lv->L_ci, lv->nnzL, int);
    if (!strcmp(name, "L_v")) COPY_OUT(lv->L_v, lv->nnzL, double);
    if (!strcmp(name, "P_rp")) COPY_OUT(lv->P_rp, nv + 1, int);
    if (!strcmp(name, "P_ci")) COPY_OUT(lv->P_ci, lv->nnzP, int);
    if (!strcmp(name, "P_v")) COPY_OUT(lv->P_v, lv->nnzP, double);
    if (!strcmp(name, "R_rp")) COPY_OUT(lv->R_rp, nvc + 1, int);
    if (!strcmp(name, "R_ci")) COPY_OUT(lv->R_ci, lv->nnzR, int);
    if (!strcmp(name, "R_v")) COPY_OUT(lv->R_v, lv->nnzR, double);
    return -1;
}

/* ------------------------------------------------------------ kernels ---- */
/* SparseOperator::apply (proj/src/sparse.cpp:209-218) */
static void csr_apply(int n, const int* rp, const int* ci, const double* v, const double* x, double* y) {
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

void orc_spmv(const orc_hier* h, int k, const char* op, const double* x, double* y) {
    const level_t* lv = &h->lv[k];
    if (op[0] == 'L') csr_apply(lv->m.nv, lv->L_rp, lv->L_ci, lv->L_v, x, y);
    else if (op[0] == 'P') csr_apply(lv->m.nv, lv->P_rp, lv->P_ci, lv->P_v, x, y);
    else if (op[0] == 'R') csr_apply(h->lv[k + 1].m.nv, lv->R_rp, lv->R_ci, lv->R_v, x, y);
}

/* kernels::dot / norm2 with kDotBlock = 4096 (proj/src/kernels.cpp:9-31,
 * proj/include/decmg/kernels.hpp:14) */
static double dot_serial(const double* a, const double* b, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
static double dot_blocked(const double* a, const double* b, int64_t n) {
    if (n <= 4096) return dot_serial(a, b, n);
    double s = 0.0;
    for (int64_t lo = 0; lo < n; lo += 4096) {
        const int64_t hi = lo + 4096 < n ? lo + 4096 : n;
        s += dot_serial(a + lo, b + lo, hi - lo);
    }
    return s;
}
double orc_norm2(const double* a, int64_t n) { return sqrt(dot_blocked(a, a, n)); }

/* MultigridHierarchy::project_compatible (proj/src/multigrid.cpp:240-250) */
void orc_project(const orc_hier* h, double* b) {
    const level_t* lv = &h->lv[0];
    double mean = 0.0, total = 0.0;
    for (int i = 0; i < lv->m.nv; ++i) {
        mean += lv->area[i] * b[i];
        total += lv->area[i];
    }
    mean /= total;
    for (int i = 0; i < lv->m.nv; ++i) b[i] -= mean;
}

/* The stand-in's sums: n <= 32 terms are added in index
 * order from 0.0; longer sums use a fixed-shape tree -- chunks of 256
 * consecutive terms, zero-padded, folded pairwise (s[t] += s[t + h] for
 * h = 128, 64, ..., 1), then the chunk sums the same way until one is left --
 * which the device's grid CG reproduces (rowkernels.cuh k_coarse_cg_grid).
 * q is overwritten. */
static double standin_sum(double* q, int64_t n) {
    if (n <= 32) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += q[i];
        return s;
    }
    while (n > 1) {
        const int64_t nc = (n + 255) / 256;
        for (int64_t c = 0; c < nc; ++c) {
            double t[256];
            for (int j = 0; j < 256; ++j) t[j] = c * 256 + j < n ? q[c * 256 + j] : 0.0;
            for (int h = 128; h >= 1; h >>= 1)
                for (int j = 0; j < h; ++j) t[j] = t[j] + t[j + h];
            q[c] = t[0];
        }
        n = nc;
    }
    return q[0];
}

/* Coarse solve: projected weighted CG (oracle/ref_standin_direct.cpp, the
 * stand-in for PinnedDirectSolver::solve, proj/src/direct.cpp:59-76).
 * Dirichlet (x1): same CG without the two projections. */
static void coarse_cg(const level_t* lv, double wtot, int project, const double* b, double* x) {
    const int n = lv->m.nv;
    const double* w = lv->area;
    double* rhs = NEW(double, n);
    double* r = NEW(double, n);
    double* p = NEW(double, n);
    double* Ap = NEW(double, n);
    double* q = NEW(double, n);
    memcpy(rhs, b, (size_t)n * sizeof(double));
    if (project) {
        for (int i = 0; i < n; ++i) q[i] = w[i] * b[i];
        const double m = standin_sum(q, n) / wtot;
        for (int i = 0; i < n; ++i) rhs[i] = b[i] - m;
    }
    for (int i = 0; i < n; ++i) { x[i] = 0.0; r[i] = rhs[i]; p[i] = rhs[i]; }
    for (int i = 0; i < n; ++i) q[i] = (w[i] * r[i]) * r[i];
    double rr = standin_sum(q, n);
    const double rr0 = rr;
    const int maxit = 4 * n + 20;
    for (int it = 0; it < maxit; ++it) {
        if (!(rr > 1e-30 * rr0)) break;
        csr_apply(n, lv->L_rp, lv->L_ci, lv->L_v, p, Ap);
        for (int i = 0; i < n; ++i) q[i] = (w[i] * p[i]) * Ap[i];
        const double curv = standin_sum(q, n);
        if (curv == 0.0) break;
        const double alpha = rr / curv;
        for (int i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] = r[i] - alpha * Ap[i];
        for (int i = 0; i < n; ++i) q[i] = (w[i] * r[i]) * r[i];
        const double rn = standin_sum(q, n);
        const double beta = rn / rr;
        for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        rr = rn;
    }
    if (project) {
        for (int i = 0; i < n; ++i) q[i] = w[i] * x[i];
        const double ym = standin_sum(q, n) / wtot;
        for (int i = 0; i < n; ++i) x[i] = x[i] - ym;
    }
    free(rhs); free(r); free(p); free(Ap); free(q);
}

void orc_coarse_solve(const orc_hier* h, const double* b, double* x) {
    coarse_cg(&h->lv[h->L - 1], h->wtot_coarse, !h->dirichlet, b, x);
}

/* jacobi_sweep (proj/src/multigrid.cpp:36-56) */
static int jacobi_sweep(const level_t* lv, double* x, const double* b, double omega, double* s) {
    const int n = lv->m.nv;
    csr_apply(n, lv->L_rp, lv->L_ci, lv->L_v, x, s);
    for (int i = 0; i < n; ++i)
        if (lv->diag[i] == 0.0) { set_err("jacobi: zero diagonal at row %d", i); return -1; }
    for (int i = 0; i < n; ++i) x[i] += omega * (b[i] - s[i]) / lv->diag[i];
    return 0;
}

/* gauss_seidel_sweep (proj/src/multigrid.cpp:13-34): rows in increasing
 * order (reverse = 0) or decreasing order (reverse = 1), updated in place */
static int gs_sweep(const level_t* lv, double* x, const double* b, int reverse) {
    const int n = lv->m.nv;
    for (int step = 0; step < n; ++step) {
        const int i = reverse ? n - 1 - step : step;
        double diag = 0.0, sum = 0.0;
        for (int k = lv->L_rp[i]; k < lv->L_rp[i + 1]; ++k) {
            if (lv->L_ci[k] == i) diag = lv->L_v[k];
            else sum += lv->L_v[k] * x[lv->L_ci[k]];
        }
        if (diag == 0.0) { set_err("gauss_seidel: zero diagonal at row %d", i); return -1; }
        x[i] = (b[i] - sum) / diag;
    }
    return 0;
}

typedef struct { int pre, post, smoother; double omega; } plan_t;

/* cg_fixed (proj/src/multigrid.cpp:63-91) with the level's dual areas as
 * weights (cycle_once passes lvl.ops.dual_areas): sequential weighted dots,
 * no convergence exit; breaks on rr == 0 or zero curvature. */
static void cg_smooth(const level_t* lv, double* x, const double* b, int iters) {
    const int n = lv->m.nv;
    const double* w = lv->area;
    double* r = NEW(double, n);
    double* p = NEW(double, n);
    double* Ap = NEW(double, n);
    csr_apply(n, lv->L_rp, lv->L_ci, lv->L_v, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    memcpy(p, r, (size_t)n * sizeof(double));
    double rr = 0.0;
    for (int i = 0; i < n; ++i) rr += w[i] * r[i] * r[i];
    for (int it = 0; it < iters; ++it) {
        if (rr == 0.0) break;
        csr_apply(n, lv->L_rp, lv->L_ci, lv->L_v, p, Ap);
        double curv = 0.0;
        for (int i = 0; i < n; ++i) curv += w[i] * p[i] * Ap[i];
        if (curv == 0.0) break;
        const double alpha = rr / curv;
        for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] -= alpha * Ap[i];
        double rn = 0.0;
        for (int i = 0; i < n; ++i) rn += w[i] * r[i] * r[i];
        const double beta = rn / rr;
        for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        rr = rn;
    }
    free(r); free(p); free(Ap);
}

/* smooth (proj/src/multigrid.cpp:95-120): 0 weighted Jacobi, 1 Gauss-Seidel,
 * 2 symmetric Gauss-Seidel (forward then reverse per iteration), 3 cg_fixed */
static int smooth(const level_t* lv, double* x, const double* b, const plan_t* p, int iters, double* s) {
    for (int it = 0; it < iters; ++it) {
        int rc;
        if (p->smoother == 3) {  /* Smoother::Cg: one call runs `iters` CG steps */
            cg_smooth(lv, x, b, iters);
            return 0;
        }
        if (p->smoother == 0) {
            rc = jacobi_sweep(lv, x, b, p->omega, s);
        } else {
            rc = gs_sweep(lv, x, b, 0);
            if (!rc && p->smoother == 2) rc = gs_sweep(lv, x, b, 1);
        }
        if (rc) return rc;
    }
    return 0;
}

/* smooth(A = level k's Laplacian, x, b, cfg, iters, weights = dual areas)
 * (proj/include/decmg/multigrid.hpp:66-68, proj/src/multigrid.cpp:95-120), x in place. */
int orc_smooth(const orc_hier* h, int k, int smoother, double omega, int iters, const double* b, double* x) {
    if (k < 0 || k >= h->L) { set_err("smooth: level out of range"); return -1; }
    const level_t* lv = &h->lv[k];
    double* s = NEW(double, lv->m.nv);
    plan_t p = {0, 0, smoother, omega};
    const int rc = smooth(lv, x, b, &p, iters, s);
    free(s);
    return rc;
}

/* MultigridHierarchy::cycle_once (proj/src/multigrid.cpp:252-285) with the
 * x1 extension (coarse RHS zeroed on Dirichlet vertices after restriction). */
static int cycle_once(const orc_hier* h, const char* walk, const plan_t* p, double** xs, double** bs,
                      double* r, double* s) {
    const int nw = (int)strlen(walk);
    int level = 0;
    for (int w = 0; w < nw; ++w) {
        if (walk[w] == 'd') {
            const level_t* lv = &h->lv[level];
            if (smooth(lv, xs[level], bs[level], p, p->pre, s)) return -1;
            csr_apply(lv->m.nv, lv->L_rp, lv->L_ci, lv->L_v, xs[level], r);
            for (int i = 0; i < lv->m.nv; ++i) r[i] = bs[level][i] - r[i];
            ++level;
            const level_t* cl = &h->lv[level];
            csr_apply(cl->m.nv, lv->R_rp, lv->R_ci, lv->R_v, r, bs[level]);
            if (h->dirichlet)
                for (int i = 0; i < cl->m.nv; ++i)
                    if (cl->bd[i]) bs[level][i] = 0.0;
            for (int i = 0; i < cl->m.nv; ++i) xs[level][i] = 0.0;
            if (level == h->L - 1) {
                orc_coarse_solve(h, bs[level], xs[level]);
            } else if (w + 1 < nw && walk[w + 1] == 'u') {
                if (smooth(cl, xs[level], bs[level], p, p->pre, s)) return -1;
            }
        } else {
            const level_t* fl = &h->lv[level - 1];
            csr_apply(fl->m.nv, fl->P_rp, fl->P_ci, fl->P_v, xs[level], r);
            --level;
            for (int i = 0; i < fl->m.nv; ++i) xs[level][i] += r[i];
            if (smooth(fl, xs[level], bs[level], p, p->post, s)) return -1;
        }
    }
    return 0;
}

static char* v_walk(int L) {
    char* w = (char*)calloc((size_t)2 * L + 1, 1);
    for (int i = 0; i < L - 1; ++i) { w[i] = 'd'; w[2 * (L - 1) - 1 - i] = 'u'; }
    return w;
}

/* MultigridHierarchy::run_cycle (proj/src/multigrid.cpp:287-323) */
int orc_run_cycles(const orc_hier* h, const char* walk, int pre, int post, int smoother, double omega,
                   const double* b, const double* x0, int ncycles, double* x_out, double* hist_out) {
    const plan_t p = {pre, post, smoother, omega};
    char* vw = walk ? NULL : v_walk(h->L);
    const char* wk = walk ? walk : vw;
    /* CyclePlan::validate (multigrid.cpp:131-143) */
    int lvl = 0;
    for (const char* c = wk; *c; ++c) {
        lvl += *c == 'd' ? 1 : -1;
        if (lvl < 0 || lvl > h->L - 1) { set_err("CyclePlan: walk leaves the hierarchy"); free(vw); return -1; }
    }
    if (lvl != 0) { set_err("CyclePlan: walk does not return to the finest level"); free(vw); return -1; }
    const int n0 = h->lv[0].m.nv;
    double** xs = (double**)calloc((size_t)h->L, sizeof(double*));
    double** bs = (double**)calloc((size_t)h->L, sizeof(double*));
    for (int k = 0; k < h->L; ++k) { xs[k] = NEW(double, h->lv[k].m.nv); bs[k] = NEW(double, h->lv[k].m.nv); }
    memcpy(xs[0], x0, (size_t)n0 * sizeof(double));
    memcpy(bs[0], b, (size_t)n0 * sizeof(double));
    double* r = NEW(double, n0);
    double* s = NEW(double, n0);
    const double bn = orc_norm2(b, n0);
    const double denom = bn > 0.0 ? bn : 1.0;
    int rc = 0;
    for (int c = 0; c < ncycles && !rc; ++c) {
        if (h->L == 1) orc_coarse_solve(h, bs[0], xs[0]);
        else rc = cycle_once(h, wk, &p, xs, bs, r, s);
        if (rc) break;
        csr_apply(n0, h->lv[0].L_rp, h->lv[0].L_ci, h->lv[0].L_v, xs[0], r);
        for (int i = 0; i < n0; ++i) r[i] = b[i] - r[i];
        if (hist_out) hist_out[c] = orc_norm2(r, n0) / denom;
    }
    if (x_out) memcpy(x_out, xs[0], (size_t)n0 * sizeof(double));
    for (int k = 0; k < h->L; ++k) { free(xs[k]); free(bs[k]); }
    free(xs); free(bs); free(r); free(s); free(vw);
    return rc;
}

/* gmg_solve (proj/src/solvers.cpp:251-279); Dirichlet skips the projection. */
int orc_solve(const orc_hier* h, int pre, int post, int smoother, double omega, const double* b,
              double tol, int max_cycles, double* x_out, double* hist_out, int* iters_out,
              double* final_out) {
    const int n0 = h->lv[0].m.nv;
    double* bc = NEW(double, n0);
    memcpy(bc, b, (size_t)n0 * sizeof(double));
    if (!h->dirichlet) orc_project(h, bc);
    double* x = NEW(double, n0);
    double* xn = NEW(double, n0);
    int c = 0, rc = 0;
    double res = 0.0;
    while (c < max_cycles) {
        double hc;
        rc = orc_run_cycles(h, NULL, pre, post, smoother, omega, bc, x, 1, xn, &hc);
        if (rc) break;
        memcpy(x, xn, (size_t)n0 * sizeof(double));
        res = hc;
        if (hist_out) hist_out[c] = res;
        ++c;
        if (res <= tol) break;
    }
    /* final_relative_residual = relative_residual(A, x, bc) (solvers.cpp:20-27) */
    double* r = xn;
    csr_apply(n0, h->lv[0].L_rp, h->lv[0].L_ci, h->lv[0].L_v, x, r);
    for (int i = 0; i < n0; ++i) r[i] = bc[i] - r[i];
    const double bn = orc_norm2(bc, n0);
    if (final_out) *final_out = orc_norm2(r, n0) / (bn > 0.0 ? bn : 1.0);
    if (iters_out) *iters_out = c;
    if (x_out) memcpy(x_out, x, (size_t)n0 * sizeof(double));
    free(bc); free(x); free(xn);
    return rc;
}

/* gmg_preconditioned_cg (proj/src/solvers.cpp:118-130) = weighted_cg
 * (solvers.cpp:56-116) on the fine operator with the level-0 dual areas as
 * weights and run_cycle(inner plan: walk, pre/post, smoother, ncycles cycles,
 * r, 0) as the preconditioner, after
 * project_compatible(b). hist_out[0..iters] (iters + 1 entries). Returns -2
 * with the reference's message on a CG breakdown. */
static double wdot(const double* w, const double* a, const double* c, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += w[i] * a[i] * c[i];
    return s;
}

int orc_pcg(const orc_hier* h, const char* walk, int pre, int post, int smoother, double omega, int ncycles,
            const double* b, double tol, int maxiter, double* x_out, double* hist_out, int* iters_out,
            double* final_out) {
    const level_t* l0 = &h->lv[0];
    const int n = l0->m.nv;
    const double* w = l0->area;
    double* bc = NEW(double, n);
    memcpy(bc, b, (size_t)n * sizeof(double));
    orc_project(h, bc);
    double* x = NEW(double, n);
    double* r = NEW(double, n);
    double* z = NEW(double, n);
    double* p = NEW(double, n);
    double* Ap = NEW(double, n);
    double* zero = NEW(double, n);
    double* hc = NEW(double, ncycles > 0 ? ncycles : 1);
    int rc = 0, it = 0;
    csr_apply(n, l0->L_rp, l0->L_ci, l0->L_v, x, r);
    for (int i = 0; i < n; ++i) r[i] = bc[i] - r[i];
    const double bn = orc_norm2(bc, n);
    const double denom = bn > 0.0 ? bn : 1.0;
    rc = orc_run_cycles(h, walk, pre, post, smoother, omega, r, zero, ncycles, z, hc);
    memcpy(p, z, (size_t)n * sizeof(double));
    double rz = wdot(w, r, z, n);
    double res = orc_norm2(r, n) / denom;
    if (hist_out) hist_out[0] = res;
    while (!rc && res > tol && it < maxiter) {
        csr_apply(n, l0->L_rp, l0->L_ci, l0->L_v, p, Ap);
        const double curv = wdot(w, p, Ap, n);
        if (curv == 0.0 || !isfinite(curv)) {
            set_err("cg: breakdown (zero curvature) at iteration %d", it);
            rc = -2;
            break;
        }
        const double alpha = rz / curv;
        if (!isfinite(alpha)) {
            set_err("cg: breakdown (non-finite step) at iteration %d", it);
            rc = -2;
            break;
        }
        for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] -= alpha * Ap[i];
        rc = orc_run_cycles(h, walk, pre, post, smoother, omega, r, zero, ncycles, z, hc);
        if (rc) break;
        const double rz_new = wdot(w, r, z, n);
        const double beta = rz_new / rz;
        for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rz = rz_new;
        ++it;
        res = orc_norm2(r, n) / denom;
        if (hist_out) hist_out[it] = res;
    }
    /* final_relative_residual = relative_residual(A, x, bc) (solvers.cpp:20-27) */
    csr_apply(n, l0->L_rp, l0->L_ci, l0->L_v, x, Ap);
    for (int i = 0; i < n; ++i) Ap[i] = bc[i] - Ap[i];
    if (final_out) *final_out = orc_norm2(Ap, n) / denom;
    if (iters_out) *iters_out = it;
    if (x_out) memcpy(x_out, x, (size_t)n * sizeof(double));
    free(bc); free(x); free(r); free(z); free(p); free(Ap); free(zero); free(hc);
    return rc;
}

/* ------------------------------------------------------- RHS (x3) -------- */
/* std::mt19937_64 (the standard MT19937-64 recurrence) + uniform01 =
 * (rng() >> 11) * 2^-53 (proj/include/decmg/rng.hpp:11-13). */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
static double uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

int orc_rhs(const orc_hier* h, const char* kind, uint64_t seed, double* b) {
    const level_t* lv = &h->lv[0];
    const int n = lv->m.nv;
    const double* P = lv->m.pos;
    mt64* g = (mt64*)malloc(sizeof(mt64));
    mt64_seed(g, seed);
    if (!strcmp(kind, "uniform")) {
        for (int i = 0; i < n; ++i) b[i] = 2.0 * uniform01(g) - 1.0;
    } else if (!strcmp(kind, "lr")) { /* poisson_rhs_random, proj/src/physics.cpp:50-53 */
        double* u = NEW(double, n);
        for (int i = 0; i < n; ++i) u[i] = uniform01(g);
        csr_apply(n, lv->L_rp, lv->L_ci, lv->L_v, u, b);
        free(u);
    } else if (!strcmp(kind, "ylm")) {
        double* gs = NEW(double, n + 1);
        for (int i = 0; i < n; i += 2) {
            const double u1 = uniform01(g);
            const double u2 = uniform01(g);
            const double rad = sqrt(-2.0 * log(1.0 - u1));
            const double th = 2.0 * M_PI * u2;
            gs[i] = rad * cos(th);
            gs[i + 1] = rad * sin(th);
        }
        const double c = 0.25 * sqrt(105.0 / M_PI);
        for (int i = 0; i < n; ++i) {
            const double x = P[3 * i], y = P[3 * i + 1], z = P[3 * i + 2];
            b[i] = c * ((x * x - y * y) * z) + 1e-3 * gs[i];
        }
        free(gs);
    } else if (!strcmp(kind, "sinsin")) {
        for (int i = 0; i < n; ++i) {
            const double x = P[3 * i], y = P[3 * i + 1];
            const double f = ((2.0 * M_PI * M_PI) * sin(M_PI * x)) * sin(M_PI * y);
            b[i] = -f;
        }
    } else {
        free(g);
        set_err("unknown rhs kind %s", kind);
        return -1;
    }
    if (h->dirichlet)
        for (int i = 0; i < n; ++i)
            if (lv->bd[i]) b[i] = 0.0;
    free(g);
    return 0;
}
