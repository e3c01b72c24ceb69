// Input generation for the CLI's `--grid kind:level` and its built-in Y_4^3 weights.
//
// Contract: the particle sets equal the reference's build_grid (geometry.cpp:97-243) and
// real_sph_harm (applications.cpp:14-49) BIT FOR BIT (tests/test_cli.py::
// test_grid_matches_reference), because a user comparing the two front-ends must feed the
// engines identical inputs.  Bitwise equality with the host libm fixes the floating-point
// operations and their order — the code around them is this file's own: grids are built
// from shared vertex tables (corner lattices, an edge-midpoint index) and areas from one
// polygon-fan routine.  Not on the GPU path.
#include <algorithm>
#include <array>
#include <cmath>
#include <stdexcept>
#include <utility>

#include "io.hpp"

namespace csfs_b200::host {

namespace {

constexpr double kPi = 3.14159265358979323846;

// ---- 3-vector arithmetic in the reference build's order (no FMA contraction on this
// host build: g++ without -march) --------------------------------------------------------
inline Vec3 plus(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 minus(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double inner(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline Vec3 outer(const Vec3& a, const Vec3& b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline Vec3 to_sphere(const Vec3& a) {
    const double len = std::sqrt(inner(a, a));
    return {a.x / len, a.y / len, a.z / len};
}

// Area of the spherical polygon v[0..n) as a fan of triangles from v[0]; each triangle is
// 2 atan2(a.(b x c), 1 + a.b + b.c + c.a) (Van Oosterom-Strackee).
template <std::size_t N>
double fan_area(const std::array<Vec3, N>& v) {
    double area = 0.0;
    for (std::size_t k = 1; k + 1 < N; ++k) {
        const Vec3 &a = v[0], &b = v[k], &c = v[k + 1];
        const double num = inner(a, outer(b, c));
        const double den = 1.0 + inner(a, b) + inner(b, c) + inner(c, a);
        area = (k == 1) ? 2.0 * std::atan2(num, den) : area + 2.0 * std::atan2(num, den);
    }
    return area;
}

// Cube face f's point (1, X, Y) in face coordinates pushed onto the sphere (the
// face-specific signed axis permutation of geometry.cpp:37-48).
Vec3 cube_to_sphere(int f, double X, double Y) {
    const double s = 1.0 / std::sqrt(1.0 + X * X + Y * Y);
    const double sX = s * X, sY = s * Y;
    switch (f) {
        case 0: return {s, sX, sY};
        case 1: return {-sX, s, sY};
        case 2: return {-s, -sX, sY};
        case 3: return {sX, -s, sY};
        case 4: return {-sY, sX, s};
        default: return {sY, sX, -s};
    }
}

// ---- equiangular cubed sphere ------------------------------------------------------------
// 6 x m x m cells, m = 2^level; cell (f, i, j) spans angles [a_i, a_i+1] x [a_j, a_j+1],
// a_k = -pi/4 + k pi/(2m).  Centre = the sphere point of the centre angles, area = the
// exact spherical quad of its four corners.  Order: face, then xi, then eta.
Grid cubed_sphere(int level) {
    const int m = 1 << level;
    const double step = (kPi / 2.0) / m;
    std::vector<double> t_edge(m + 1), t_mid(m);
    for (int k = 0; k <= m; ++k) t_edge[k] = std::tan(-kPi / 4.0 + k * step);
    for (int k = 0; k < m; ++k) t_mid[k] = std::tan(-kPi / 4.0 + (k + 0.5) * step);
    Grid g;
    g.kind = "cubed_sphere";
    g.level = level;
    const std::size_t per_face = std::size_t(m) * m;
    g.centers.resize(6 * per_face);
    g.areas.resize(6 * per_face);
    std::vector<Vec3> lattice(std::size_t(m + 1) * (m + 1));  // one face's corner points
    for (int f = 0; f < 6; ++f) {
        for (int i = 0; i <= m; ++i)
            for (int j = 0; j <= m; ++j) lattice[std::size_t(i) * (m + 1) + j] = cube_to_sphere(f, t_edge[i], t_edge[j]);
        auto corner = [&](int i, int j) { return lattice[std::size_t(i) * (m + 1) + j]; };
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                const std::size_t c = f * per_face + std::size_t(i) * m + j;
                g.centers[c] = cube_to_sphere(f, t_mid[i], t_mid[j]);
                g.areas[c] = fan_area<4>({corner(i, j), corner(i + 1, j), corner(i + 1, j + 1), corner(i, j + 1)});
            }
    }
    return g;
}

// ---- icosahedral -------------------------------------------------------------------------
// The icosahedron (12 vertices on the golden-ratio rectangles, 20 outward-oriented faces)
// refined `level` times: every triangle splits into four through its edge midpoints, a
// midpoint being created the first time its edge is met (so vertex ids follow the triangle
// walk).  Control areas come from the barycentric dual: each triangle hands each corner the
// quad corner -> midpoint of the next edge -> centroid -> midpoint of the previous edge.
class IcoMesh {
public:
    IcoMesh() {
        const double gr = (1.0 + std::sqrt(5.0)) / 2.0;
        const double base[12][3] = {{-1, gr, 0}, {1, gr, 0}, {-1, -gr, 0}, {1, -gr, 0}, {0, -1, gr}, {0, 1, gr},
                                    {0, -1, -gr}, {0, 1, -gr}, {gr, 0, -1}, {gr, 0, 1}, {-gr, 0, -1}, {-gr, 0, 1}};
        for (const auto& b : base) vert_.push_back(to_sphere({b[0], b[1], b[2]}));
        static constexpr int kFaces[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                              {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                              {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                              {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
        for (const auto& f : kFaces) {
            Tri t{f[0], f[1], f[2]};
            const Vec3 n = outer(minus(vert_[t[1]], vert_[t[0]]), minus(vert_[t[2]], vert_[t[0]]));
            if (inner(vert_[t[0]], n) < 0.0) std::swap(t[1], t[2]);  // outward
            tri_.push_back(t);
        }
    }

    void refine() {
        edge_mid_.assign(vert_.size(), {});
        std::vector<Tri> finer;
        finer.reserve(4 * tri_.size());
        for (const Tri& t : tri_) {
            const int m01 = midpoint(t[0], t[1]), m12 = midpoint(t[1], t[2]), m20 = midpoint(t[2], t[0]);
            finer.push_back({t[0], m01, m20});
            finer.push_back({t[1], m12, m01});
            finer.push_back({t[2], m20, m12});
            finer.push_back({m01, m12, m20});
        }
        tri_.swap(finer);
    }

    Grid grid(int level) {
        Grid g;
        g.kind = "icosahedral";
        g.level = level;
        g.areas.assign(vert_.size(), 0.0);
        for (const Tri& t : tri_) {
            const Vec3 &p0 = vert_[t[0]], &p1 = vert_[t[1]], &p2 = vert_[t[2]];
            const Vec3 h01 = to_sphere(plus(p0, p1)), h12 = to_sphere(plus(p1, p2)), h20 = to_sphere(plus(p2, p0));
            const Vec3 cen = to_sphere(plus(plus(p0, p1), p2));
            g.areas[t[0]] += fan_area<4>({p0, h01, cen, h20});
            g.areas[t[1]] += fan_area<4>({p1, h12, cen, h01});
            g.areas[t[2]] += fan_area<4>({p2, h20, cen, h12});
        }
        g.centers = std::move(vert_);
        return g;
    }

private:
    using Tri = std::array<int, 3>;
    std::vector<Vec3> vert_;
    std::vector<Tri> tri_;
    // per lower vertex id: (higher vertex id, midpoint id) of the edges met at this level
    std::vector<std::vector<std::pair<int, int>>> edge_mid_;

    int midpoint(int a, int b) {
        const int lo = std::min(a, b), hi = std::max(a, b);
        for (const auto& e : edge_mid_[lo])
            if (e.first == hi) return e.second;
        const int id = int(vert_.size());
        vert_.push_back(to_sphere(plus(vert_[a], vert_[b])));
        edge_mid_[lo].push_back({hi, id});
        return id;
    }
};

// ---- regular longitude-latitude cells ------------------------------------------------------
// 45 * 2^(level-4) colatitude bands x twice as many longitudes; centre at the cell-centre
// angles, area = the exact band area dlon (cos th_i - cos th_i+1).
Grid latlon(int level) {
    const int nb = 45 << (level - 4), nl = 2 * nb;
    const double d_th = kPi / nb, d_lon = 2.0 * kPi / nl;
    Grid g;
    g.kind = "latlon";
    g.level = level;
    g.centers.resize(std::size_t(nb) * nl);
    g.areas.resize(std::size_t(nb) * nl);
    std::vector<double> cos_lon(nl), sin_lon(nl);
    for (int j = 0; j < nl; ++j) {
        cos_lon[j] = std::cos((j + 0.5) * d_lon);
        sin_lon[j] = std::sin((j + 0.5) * d_lon);
    }
    for (int b = 0; b < nb; ++b) {
        const double th = (b + 0.5) * d_th;
        const double ring = std::sin(th), height = std::cos(th);
        const double cell = d_lon * (std::cos(b * d_th) - std::cos((b + 1) * d_th));
        for (int j = 0; j < nl; ++j) {
            g.centers[std::size_t(b) * nl + j] = {ring * cos_lon[j], ring * sin_lon[j], height};
            g.areas[std::size_t(b) * nl + j] = cell;
        }
    }
    return g;
}

// ---- spherical harmonics -----------------------------------------------------------------
// P_l^m(z) (no Condon-Shortley phase): start on the diagonal P_m^m = (2m-1)!! (1-z^2)^(m/2),
// one step off it, then the three-term recurrence in l.
double assoc_legendre(int l, int m, double z) {
    double lower = 1.0;  // P_m^m
    if (m > 0) {
        const double sin_t = std::sqrt(std::max(0.0, 1.0 - z * z));
        for (int k = 0; k < m; ++k) lower *= double(2 * k + 1) * sin_t;
    }
    if (l == m) return lower;
    double upper = z * (2.0 * m + 1.0) * lower;  // P_{m+1}^m
    for (int deg = m + 2; deg <= l; ++deg) {
        const double next = (z * (2.0 * deg - 1.0) * upper - (deg + m - 1.0) * lower) / (deg - m);
        lower = upper;
        upper = next;
    }
    return upper;
}

// (l-m)! / (l+m)! as the running quotient 1 / ((l-m+1)(l-m+2)...(l+m))
double factorial_quotient(int l, int m) {
    double q = 1.0;
    for (int k = l - m + 1; k <= l + m; ++k) q /= double(k);
    return q;
}

}  // namespace

Grid build_grid(const std::string& kind, int level) {
    if (kind != "icosahedral" && kind != "cubed_sphere" && kind != "latlon")
        throw std::invalid_argument("unknown grid kind: " + kind);
    if (level < 0) throw std::invalid_argument("grid level must be non-negative");
    if (kind == "cubed_sphere") {
        if (level > 10) throw std::invalid_argument("cubed sphere grid supports levels 0..10");
        return cubed_sphere(level);
    }
    if (kind == "latlon") {
        if (level < 4 || level > 9) throw std::invalid_argument("latlon grid supports levels 4..9");
        return latlon(level);
    }
    if (level > 9) throw std::invalid_argument("icosahedral grid supports levels 0..9");
    IcoMesh mesh;
    for (int k = 0; k < level; ++k) mesh.refine();
    return mesh.grid(level);
}

// Orthonormal real spherical harmonic: N_lm P_l^|m|(z) with N_lm^2 = (2l+1)/(4 pi) (l-|m|)!/
// (l+|m|)!, times sqrt(2) cos(m lon) for m > 0 and sqrt(2) sin(|m| lon) for m < 0.
double real_sph_harm(int l, int m, const Vec3& p) {
    if (l < 0 || std::abs(m) > l) throw std::invalid_argument("invalid spherical harmonic degree/order");
    const int am = std::abs(m);
    const double n_lm = std::sqrt((2.0 * l + 1.0) / (4.0 * kPi) * factorial_quotient(l, am));
    const double p_lm = assoc_legendre(l, am, p.z);
    if (m == 0) return n_lm * p_lm;
    const double phi = std::atan2(p.y, p.x);
    return std::sqrt(2.0) * n_lm * p_lm * (m > 0 ? std::cos(am * phi) : std::sin(am * phi));
}

// Area-weighted relative L2 distance sqrt(sum_i A_i |phi1_i - phi2_i|^2 / sum_i A_i |phi_ex_i|^2)
// over out_dim components per point.
double relative_l2_error(const std::vector<double>& phi1, const std::vector<double>& phi2,
                         const std::vector<double>& phi_exact, const std::vector<double>& areas, int out_dim) {
    const std::size_t n = areas.size(), len = n * std::size_t(out_dim);
    if (phi1.size() != len || phi2.size() != len || phi_exact.size() != len)
        throw std::invalid_argument("field lengths do not match the area list");
    double err2 = 0.0, ref2 = 0.0;
    for (std::size_t k = 0; k < len; ++k) {
        const double a = areas[k / out_dim];
        const double d = phi1[k] - phi2[k];
        err2 += d * d * a;
        ref2 += phi_exact[k] * phi_exact[k] * a;
    }
    if (ref2 == 0.0) throw std::invalid_argument("reference field is identically zero");
    return std::sqrt(err2 / ref2);
}

}  // namespace csfs_b200::host
