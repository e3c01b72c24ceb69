// Input generation for the CLI's `--grid kind:level` (the reference's build_grid,
// geometry.cpp:97-213) and its built-in Y_4^3 weights (real_sph_harm, applications.cpp:
// 14-49), restated on the host with the same operation order and the same libm, so the
// particle sets the CLI hands to the engine are bitwise the reference's
// (tests/test_cli.py::test_grid_matches_reference).  Not on the GPU path.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <unordered_map>

#include "io.hpp"

namespace csfs_b200::host {

namespace {

constexpr double kPi = 3.14159265358979323846;

Vec3 add(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
Vec3 sub(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
Vec3 cross(const Vec3& a, const Vec3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
Vec3 unit(const Vec3& a) {
    const double n = std::sqrt(dot(a, a));
    return {a.x / n, a.y / n, a.z / n};
}

// face_point_from_plane (geometry.cpp:37-48): the cube-face point (1, X, Y) in face
// coordinates, projected to the sphere
Vec3 plane_point(int face, double X, double Y) {
    const double s = 1.0 / std::sqrt(1.0 + X * X + Y * Y);
    switch (face) {
        case 0: return {s, s * X, s * Y};
        case 1: return {-s * X, s, s * Y};
        case 2: return {-s, -s * X, s * Y};
        case 3: return {s * X, -s, s * Y};
        case 4: return {-s * Y, s * X, s};
        default: return {s * Y, s * X, -s};
    }
}

// spherical triangle / quad areas (geometry.cpp:70-78): 2 atan2(a.(b x c), 1 + a.b + b.c + c.a)
double tri_area(const Vec3& a, const Vec3& b, const Vec3& c) {
    return 2.0 * std::atan2(dot(a, cross(b, c)), 1.0 + dot(a, b) + dot(b, c) + dot(c, a));
}
double quad_area(const Vec3& p0, const Vec3& p1, const Vec3& p2, const Vec3& p3) {
    return tri_area(p0, p1, p2) + tri_area(p0, p2, p3);
}

// equiangular cubed sphere: 6 x 2^L x 2^L cells, centres at the cell-centre angles,
// exact spherical cell areas; order face -> xi -> eta
Grid cubed_sphere(int level) {
    const int m = 1 << level;
    const double d = (kPi / 2.0) / m;
    std::vector<double> edge(m + 1);
    for (int i = 0; i <= m; ++i) edge[i] = std::tan(-kPi / 4.0 + i * d);
    Grid g;
    g.kind = "cubed_sphere";
    g.level = level;
    g.centers.reserve(std::size_t(6) * m * m);
    g.areas.reserve(std::size_t(6) * m * m);
    for (int f = 0; f < 6; ++f)
        for (int i = 0; i < m; ++i) {
            const double xc = -kPi / 4.0 + (i + 0.5) * d;
            for (int j = 0; j < m; ++j) {
                const double ec = -kPi / 4.0 + (j + 0.5) * d;
                g.centers.push_back(plane_point(f, std::tan(xc), std::tan(ec)));
                g.areas.push_back(quad_area(plane_point(f, edge[i], edge[j]), plane_point(f, edge[i + 1], edge[j]),
                                            plane_point(f, edge[i + 1], edge[j + 1]),
                                            plane_point(f, edge[i], edge[j + 1])));
            }
        }
    return g;
}

// icosahedral: the 12-vertex icosahedron, `level` midpoint subdivisions (vertices
// re-projected), control areas from the barycentric dual (each triangle gives each corner
// the quad corner - edge midpoint - centroid - edge midpoint)
Grid icosahedral(int level) {
    const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
    const double raw[12][3] = {{-1, phi, 0}, {1, phi, 0}, {-1, -phi, 0}, {1, -phi, 0},
                               {0, -1, phi}, {0, 1, phi}, {0, -1, -phi}, {0, 1, -phi},
                               {phi, 0, -1}, {phi, 0, 1}, {-phi, 0, -1}, {-phi, 0, 1}};
    const int faces[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                              {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                              {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                              {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
    std::vector<Vec3> V;
    for (const auto& r : raw) V.push_back(unit({r[0], r[1], r[2]}));
    std::vector<std::array<int, 3>> T;
    for (const auto& f : faces) {
        std::array<int, 3> t{f[0], f[1], f[2]};
        if (dot(V[t[0]], cross(sub(V[t[1]], V[t[0]]), sub(V[t[2]], V[t[0]]))) < 0.0) std::swap(t[1], t[2]);
        T.push_back(t);
    }
    for (int l = 0; l < level; ++l) {
        std::unordered_map<std::uint64_t, int> mids;
        mids.reserve(T.size() * 2);
        auto mid = [&](int a, int b) {
            const std::uint64_t key = (std::uint64_t(std::min(a, b)) << 32) | std::uint64_t(std::max(a, b));
            const auto it = mids.find(key);
            if (it != mids.end()) return it->second;
            V.push_back(unit(add(V[a], V[b])));
            mids.emplace(key, int(V.size()) - 1);
            return int(V.size()) - 1;
        };
        std::vector<std::array<int, 3>> next;
        next.reserve(T.size() * 4);
        for (const auto& t : T) {
            const int ab = mid(t[0], t[1]), bc = mid(t[1], t[2]), ca = mid(t[2], t[0]);
            next.push_back({t[0], ab, ca});
            next.push_back({t[1], bc, ab});
            next.push_back({t[2], ca, bc});
            next.push_back({ab, bc, ca});
        }
        T = std::move(next);
    }
    std::vector<double> area(V.size(), 0.0);
    for (const auto& t : T) {
        const Vec3 &a = V[t[0]], &b = V[t[1]], &c = V[t[2]];
        const Vec3 mab = unit(add(a, b)), mbc = unit(add(b, c)), mca = unit(add(c, a));
        const Vec3 g = unit(add(add(a, b), c));
        area[t[0]] += quad_area(a, mab, g, mca);
        area[t[1]] += quad_area(b, mbc, g, mab);
        area[t[2]] += quad_area(c, mca, g, mbc);
    }
    Grid g;
    g.kind = "icosahedral";
    g.level = level;
    g.centers = std::move(V);
    g.areas = std::move(area);
    return g;
}

// regular lat-lon cells: (45 * 2^(L-4)) rows x twice as many columns, exact band areas
Grid latlon(int level) {
    const int rows = 45 << (level - 4), cols = 2 * rows;
    const double dth = kPi / rows, dlm = 2.0 * kPi / cols;
    Grid g;
    g.kind = "latlon";
    g.level = level;
    g.centers.reserve(std::size_t(rows) * cols);
    g.areas.reserve(std::size_t(rows) * cols);
    for (int i = 0; i < rows; ++i) {
        const double thc = (i + 0.5) * dth;
        const double band = dlm * (std::cos(i * dth) - std::cos((i + 1) * dth));
        const double sth = std::sin(thc), cth = std::cos(thc);
        for (int j = 0; j < cols; ++j) {
            const double lm = (j + 0.5) * dlm;
            g.centers.push_back({sth * std::cos(lm), sth * std::sin(lm), cth});
            g.areas.push_back(band);
        }
    }
    return g;
}

// associated Legendre P_l^m(z), no Condon-Shortley phase: the standard upward recurrence
double legendre(int l, int m, double z) {
    double pmm = 1.0;
    if (m > 0) {
        const double s = std::sqrt(std::max(0.0, 1.0 - z * z));
        double fact = 1.0;
        for (int i = 1; i <= m; ++i) {
            pmm *= fact * s;
            fact += 2.0;
        }
    }
    if (l == m) return pmm;
    double pmm1 = z * (2.0 * m + 1.0) * pmm;
    if (l == m + 1) return pmm1;
    double pll = 0.0;
    for (int ll = m + 2; ll <= l; ++ll) {
        pll = (z * (2.0 * ll - 1.0) * pmm1 - (ll + m - 1.0) * pmm) / (ll - m);
        pmm = pmm1;
        pmm1 = pll;
    }
    return pll;
}

}  // namespace

Grid build_grid(const std::string& kind, int level) {
    if (kind != "icosahedral" && kind != "cubed_sphere" && kind != "latlon")
        throw std::invalid_argument("unknown grid kind: " + kind);
    if (level < 0) throw std::invalid_argument("grid level must be non-negative");
    if (kind == "icosahedral") {
        if (level > 9) throw std::invalid_argument("icosahedral grid supports levels 0..9");
        return icosahedral(level);
    }
    if (kind == "cubed_sphere") {
        if (level > 10) throw std::invalid_argument("cubed sphere grid supports levels 0..10");
        return cubed_sphere(level);
    }
    if (level < 4 || level > 9) throw std::invalid_argument("latlon grid supports levels 4..9");
    return latlon(level);
}

// orthonormal real spherical harmonic: sqrt((2l+1)/4pi (l-|m|)!/(l+|m|)!) P_l^|m|(z),
// times sqrt(2) cos(m lon) (m > 0) or sqrt(2) sin(|m| lon) (m < 0)
double real_sph_harm(int l, int m, const Vec3& p) {
    if (l < 0 || std::abs(m) > l) throw std::invalid_argument("invalid spherical harmonic degree/order");
    const int am = std::abs(m);
    double ratio = 1.0;
    for (int i = l - am + 1; i <= l + am; ++i) ratio /= double(i);
    const double norm = std::sqrt((2.0 * l + 1.0) / (4.0 * kPi) * ratio);
    const double plm = legendre(l, am, p.z);
    if (m == 0) return norm * plm;
    const double lon = std::atan2(p.y, p.x);
    const double trig = m > 0 ? std::cos(am * lon) : std::sin(am * lon);
    return std::sqrt(2.0) * norm * plm * trig;
}

double relative_l2_error(const std::vector<double>& phi1, const std::vector<double>& phi2,
                         const std::vector<double>& phi_exact, const std::vector<double>& areas, int out_dim) {
    const std::size_t n = areas.size();
    if (phi1.size() != n * out_dim || phi2.size() != n * out_dim || phi_exact.size() != n * out_dim)
        throw std::invalid_argument("field lengths do not match the area list");
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < n; ++i)
        for (int d = 0; d < out_dim; ++d) {
            const std::size_t k = i * out_dim + d;
            const double diff = phi1[k] - phi2[k];
            num += diff * diff * areas[i];
            den += phi_exact[k] * phi_exact[k] * areas[i];
        }
    if (den == 0.0) throw std::invalid_argument("reference field is identically zero");
    return std::sqrt(num / den);
}

}  // namespace csfs_b200::host
