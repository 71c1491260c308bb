// TEST INFRASTRUCTURE ONLY (oracle). The BASELINE cases built with the
// UNMODIFIED reference's own mesh and subdivision code (proj/src/mesh.cpp,
// subdivision.cpp, geometric_map.cpp), shared by oracle/ref_harness.cpp and the
// shim's reference-type caller tests/cpp/shim_reference.cpp:
//   x2 canonical icosahedron + projected binary/cubic subdivision
//   <base>[+cubic] specs: square | ico | grid:nx:ny:lx:ly | equi:rows:cols:side
#pragma once

#include "decmg/geometric_map.hpp"
#include "decmg/mesh.hpp"
#include "decmg/subdivision.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace refcases {
using namespace decmg;

// ---- extension x2: canonical icosahedron ------------------------
inline std::shared_ptr<EmbeddedComplex2D> ico_base() {
    const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
    const double raw[12][3] = {{-1, phi, 0}, {1, phi, 0},  {-1, -phi, 0}, {1, -phi, 0},
                               {0, -1, phi}, {0, 1, phi},  {0, -1, -phi}, {0, 1, -phi},
                               {phi, 0, -1}, {phi, 0, 1},  {-phi, 0, -1}, {-phi, 0, 1}};
    std::vector<Vec3> pos;
    for (const auto& r : raw) {
        Vec3 p(r[0], r[1], r[2]);
        const double s = 1.0 / p.norm();
        pos.push_back(p * s);
    }
    const std::vector<std::array<int, 3>> tris = {
        {0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
        {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
        {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
        {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
    return EmbeddedComplex2D::from_triangles(std::move(pos), tris);
}

// Projected subdivision: the reference's binary (or cubic) subdivide, then
// every new vertex is pushed to the unit sphere as p * (1.0 / |p|); copied
// vertices keep their bits. Map columns are unchanged.
inline SubdivisionResult projected_subdivide(const std::shared_ptr<const EmbeddedComplex2D>& c, bool cubic = false) {
    SubdivisionResult s = cubic ? cubic_subdivide(c) : binary_subdivide(c);
    const int nvc = c->num_vertices();
    std::vector<Vec3> pos = s.fine->positions;
    for (std::size_t v = nvc; v < pos.size(); ++v) {
        const double inv = 1.0 / pos[v].norm();
        pos[v] = pos[v] * inv;
    }
    std::vector<std::array<int, 3>> tris;
    tris.reserve(s.fine->num_triangles());
    for (int t = 0; t < s.fine->num_triangles(); ++t) tris.push_back(s.fine->corners(t));
    auto fine = EmbeddedComplex2D::from_triangles(std::move(pos), tris);
    SubdivisionResult out;
    out.map = GeometricMap::make(fine, c, s.map.columns());
    out.fine = fine;
    out.provenance = std::move(s.provenance);
    return out;
}

struct Case {
    std::shared_ptr<EmbeddedComplex2D> base;
    bool project = false;
    bool cubic = false;  // SubdivisionScheme::Cubic (1 -> 9) instead of Binary
};

// <base>[+cubic], base one of square | ico | grid:nx:ny:lx:ly | equi:rows:cols:side
inline Case make_case(const std::string& spec_in) {
    Case c;
    std::string spec = spec_in;
    const std::string suffix = "+cubic";
    if (spec.size() > suffix.size() && spec.compare(spec.size() - suffix.size(), suffix.size(), suffix) == 0) {
        c.cubic = true;
        spec = spec.substr(0, spec.size() - suffix.size());
    }
    if (spec == "square") {
        c.base = make_triangulated_grid(1, 1, 1.0, 1.0);
    } else if (spec == "ico") {
        c.base = ico_base();
        c.project = true;
    } else if (spec.rfind("grid:", 0) == 0) {
        int nx, ny;
        double lx, ly;
        if (std::sscanf(spec.c_str(), "grid:%d:%d:%lf:%lf", &nx, &ny, &lx, &ly) != 4)
            throw std::invalid_argument("bad grid spec");
        c.base = make_triangulated_grid(nx, ny, lx, ly);
    } else if (spec.rfind("equi:", 0) == 0) {
        int r, cc;
        double side;
        if (std::sscanf(spec.c_str(), "equi:%d:%d:%lf", &r, &cc, &side) != 3)
            throw std::invalid_argument("bad equi spec");
        c.base = make_equilateral_grid(r, cc, side);
    } else {
        throw std::invalid_argument("unknown case " + spec);
    }
    return c;
}

inline std::vector<SubdivisionResult> tower_of(const Case& c, int k) {
    if (k == 0) return {};
    if (!c.project)
        return subdivision_tower(c.base, c.cubic ? SubdivisionScheme::Cubic : SubdivisionScheme::Binary, k);
    std::vector<SubdivisionResult> chain;
    std::shared_ptr<const EmbeddedComplex2D> cur = c.base;
    for (int i = 0; i < k; ++i) {
        chain.push_back(projected_subdivide(cur, c.cubic));
        cur = chain.back().fine;
    }
    std::reverse(chain.begin(), chain.end());
    return chain;
}

}  // namespace refcases
