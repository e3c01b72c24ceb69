// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (csfs, compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// It lets the Python parity tests, the golden-fixture generator and
// bench.py's reference arm call the reference's own `csfmm_sum`,
// `direct_sum`, `ClusterTree`, `upward_pass` and `dual_tree_traversal`
// (proj/include/csfs/summation.hpp:63-102, cluster_tree.hpp:52-81) on the
// same arrays the CUDA path receives.  Nothing here re-implements the
// algorithm; every function forwards to the reference.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "csfs/applications.hpp"
#include "csfs/cluster_tree.hpp"
#include "csfs/geometry.hpp"
#include "csfs/io.hpp"
#include "csfs/kernels.hpp"
#include "csfs/summation.hpp"

using namespace csfs;

namespace {

thread_local std::string g_err;

std::vector<Vec3> to_vec3(const double* xyz, size_t n) {
    std::vector<Vec3> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    return v;
}

Kernel make_kernel(int kind, const double* sal4) {
    Kernel k;
    switch (kind) {
        case 0: k.kind = KernelKind::Laplace; break;
        case 1: k.kind = KernelKind::Biharmonic; break;
        case 2: k.kind = KernelKind::BiotSavart; break;
        case 3: k.kind = KernelKind::Sal; break;
        default: throw std::invalid_argument("unknown kernel kind");
    }
    if (sal4) {
        k.sal.a1 = sal4[0];
        k.sal.b0 = sal4[1];
        k.sal.b1 = sal4[2];
        k.sal.rho_ratio = sal4[3];
    }
    return k;
}

void put_stats(const SumStats& s, double* st) {
    if (!st) return;
    st[0] = s.t_tree_build;
    st[1] = s.t_upward;
    st[2] = s.t_traversal;
    st[3] = s.t_downward;
    st[4] = s.t_total;
    st[5] = double(s.pp);
    st[6] = double(s.pc);
    st[7] = double(s.cp);
    st[8] = double(s.cc);
    st[9] = s.source_tree.depth;
    st[10] = s.source_tree.cluster_count;
    st[11] = s.source_tree.leaf_count;
    st[12] = s.target_tree.depth;
    st[13] = s.target_tree.cluster_count;
    st[14] = s.target_tree.leaf_count;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* csref_last_error() { return g_err.c_str(); }

// read_particles_csv (io.cpp:166-185): returns the particle count (fills when xyz != null),
// or -1 with last_error = "<code>: <message>" for the reference's CliError.
long long csref_read_particles(const char* path, double* xyz, double* w) {
    try {
        const ParticleSet p = read_particles_csv(path);
        if (xyz)
            for (size_t i = 0; i < p.size(); ++i) {
                xyz[3 * i] = p.positions[i].x;
                xyz[3 * i + 1] = p.positions[i].y;
                xyz[3 * i + 2] = p.positions[i].z;
                w[i] = p.weights[i];
            }
        return (long long)p.size();
    } catch (const CliError& e) {
        g_err = e.code + ": " + e.message;
        return -1;
    }
}

// build_grid (geometry.cpp:229-243): returns the cell count; fills when xyz != null.
long long csref_grid(int kind, int level, double* xyz, double* areas) {
    long long n = -1;
    int rc = guarded([&] {
        const GridKind gk = kind == 0 ? GridKind::Icosahedral
                            : kind == 1 ? GridKind::CubedSphere
                                        : GridKind::LatLon;
        const SphericalGrid g = build_grid(gk, level);
        n = (long long)g.size();
        if (xyz)
            for (size_t i = 0; i < g.size(); ++i) {
                xyz[3 * i] = g.centers[i].x;
                xyz[3 * i + 1] = g.centers[i].y;
                xyz[3 * i + 2] = g.centers[i].z;
            }
        if (areas)
            for (size_t i = 0; i < g.size(); ++i) areas[i] = g.areas[i];
    });
    return rc ? -1 : n;
}

// summed_potential (summation.cpp:423-440) with method 0 direct / 1 cstc / 2 csfmm.
int csref_sum(int method, const double* txyz, size_t nt, const double* sxyz, const double* sw,
              size_t ns, int kind, const double* sal4, double mac, int degree, int n0,
              int shrink, int threads, double* out, double* stats) {
    return guarded([&] {
        ParticleSet t, s;
        t.positions = to_vec3(txyz, nt);
        t.weights.assign(nt, 0.0);
        s.positions = to_vec3(sxyz, ns);
        s.weights.assign(sw, sw + ns);
        TraversalConfig cfg;
        cfg.method = method == 0 ? Method::Direct : method == 1 ? Method::Cstc : Method::Csfmm;
        cfg.mac = mac;
        cfg.degree = degree;
        cfg.n0 = n0;
        cfg.shrink = shrink != 0;
        cfg.threads = threads;
        SumStats st;
        const PotentialField f = summed_potential(t, s, make_kernel(kind, sal4), cfg, &st);
        std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
        put_stats(st, stats);
    });
}

// --- stepwise API (cluster_tree.hpp:52-81, summation.hpp:69-102) -----------------

void* csref_tree_new(const double* xyz, size_t n, int degree, int n0, int shrink) {
    ClusterTree* tree = nullptr;
    int rc = guarded([&] {
        ParticleSet p;
        p.positions = to_vec3(xyz, n);
        p.weights.assign(n, 0.0);
        tree = new ClusterTree(p, degree, n0, shrink != 0);
    });
    return rc ? nullptr : tree;
}

void csref_tree_free(void* h) { delete static_cast<ClusterTree*>(h); }

int csref_tree_ncl(void* h) { return int(static_cast<ClusterTree*>(h)->clusters.size()); }
int csref_tree_depth(void* h) { return int(static_cast<ClusterTree*>(h)->levels.size()) - 1; }

// ints: ncl x 10 = face, begin, end, parent, depth, child_count, children[4]
// dbls: ncl x 8  = xi0, xi1, eta0, eta1, cx, cy, cz, radius
// proxy: ncl x (p+1)^2 x 3 (nullable); xi/eta: n (tree order, nullable)
void csref_tree_export(void* h, int* perm, int* ints, double* dbls, double* proxy, double* xi,
                       double* eta) {
    const ClusterTree& t = *static_cast<ClusterTree*>(h);
    const size_t n = t.particle_count();
    if (perm) std::memcpy(perm, t.perm.data(), n * sizeof(int));
    if (xi) std::memcpy(xi, t.xi.data(), n * sizeof(double));
    if (eta) std::memcpy(eta, t.eta.data(), n * sizeof(double));
    for (size_t c = 0; c < t.clusters.size(); ++c) {
        const Cluster& k = t.clusters[c];
        if (ints) {
            int* r = ints + 10 * c;
            r[0] = k.face;
            r[1] = k.begin;
            r[2] = k.end;
            r[3] = k.parent;
            r[4] = k.depth;
            r[5] = k.child_count;
            for (int q = 0; q < 4; ++q) r[6 + q] = k.children[q];
        }
        if (dbls) {
            double* r = dbls + 8 * c;
            r[0] = k.bounds.xi0;
            r[1] = k.bounds.xi1;
            r[2] = k.bounds.eta0;
            r[3] = k.bounds.eta1;
            r[4] = k.center.x;
            r[5] = k.center.y;
            r[6] = k.center.z;
            r[7] = k.radius;
        }
        if (proxy) {
            const size_t npp = k.interp.proxy_points.size();
            for (size_t m = 0; m < npp; ++m) {
                double* r = proxy + 3 * (c * npp + m);
                r[0] = k.interp.proxy_points[m].x;
                r[1] = k.interp.proxy_points[m].y;
                r[2] = k.interp.proxy_points[m].z;
            }
        }
    }
}

// upward_pass (cluster_tree.cpp:163-220); pw: ncl x (p+1)^2 in cluster-id order.
int csref_upward(void* h, const double* w, double* pw) {
    return guarded([&] {
        ClusterTree& t = *static_cast<ClusterTree*>(h);
        std::vector<double> wv(w, w + t.particle_count());
        upward_pass(t, wv);
        if (pw) {
            size_t off = 0;
            for (const Cluster& c : t.clusters) {
                std::memcpy(pw + off, c.proxy_weights.data(), c.proxy_weights.size() * sizeof(double));
                off += c.proxy_weights.size();
            }
        }
    });
}

// dual_tree_traversal (summation.cpp:163-203).  counts[4] = |pp|,|pc|,|cp|,|cc|;
// each non-null list buffer receives (t, s) int pairs in the reference's emission order.
int csref_lists(void* ht, void* hs, double mac, int n0, long long* counts, int* pp, int* pc,
                int* cp, int* cc) {
    return guarded([&] {
        const ClusterTree& tt = *static_cast<ClusterTree*>(ht);
        const ClusterTree& ts = *static_cast<ClusterTree*>(hs);
        const InteractionLists l = dual_tree_traversal(tt, ts, mac, n0);
        const std::vector<std::pair<int, int>>* lists[4] = {&l.pp, &l.pc, &l.cp, &l.cc};
        int* outs[4] = {pp, pc, cp, cc};
        for (int k = 0; k < 4; ++k) {
            counts[k] = (long long)lists[k]->size();
            if (outs[k])
                for (size_t e = 0; e < lists[k]->size(); ++e) {
                    outs[k][2 * e] = (*lists[k])[e].first;
                    outs[k][2 * e + 1] = (*lists[k])[e].second;
                }
        }
    });
}

// --- numerics used by the fixtures -------------------------------------------------

double csref_dilog(double x) {
    double v = 0.0;
    guarded([&] { v = dilog(x); });
    return v;
}

// Kernel::try_eval (kernels.cpp: try_eval) — returns 1 when evaluated, 0 when guarded.
int csref_kernel_try_eval(int kind, const double* sal4, const double* x, const double* y,
                          double* out) {
    const Kernel k = make_kernel(kind, sal4);
    return k.try_eval({x[0], x[1], x[2]}, {y[0], y[1], y[2]}, out) ? 1 : 0;
}

void csref_bary_basis_1d(int degree, double x, double* out) {
    ChebyshevGrid1D g(degree);
    bary_basis_1d(g, x, out);
}

void csref_face_project(const double* p, int* face, double* xi, double* eta) {
    const FaceCoords fc = face_project({p[0], p[1], p[2]});
    *face = fc.face;
    *xi = fc.xi;
    *eta = fc.eta;
}

void csref_sph_harm_many(int l, int m, const double* xyz, size_t n, double* out) {
    for (size_t i = 0; i < n; ++i)
        out[i] = real_sph_harm(l, m, {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
}

void csref_rh_zeta_many(const double* xyz, size_t n, double* out) {
    for (size_t i = 0; i < n; ++i)
        out[i] = rossby_haurwitz_zeta({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
}

// One bve_step (applications.cpp:378-412) with remesh off: 4 CSFMM Biot-Savart sums.
int csref_bve_step(double* xyz, double* zeta, const double* areas, size_t n, double omega,
                   double dt, double mac, int degree, int n0, int threads) {
    return guarded([&] {
        BveState s;
        s.positions = to_vec3(xyz, n);
        s.zeta.assign(zeta, zeta + n);
        s.areas.assign(areas, areas + n);
        s.grid_centers = s.positions;
        s.omega = omega;
        BveStepOptions o;
        o.traversal.mac = mac;
        o.traversal.degree = degree;
        o.traversal.n0 = n0;
        o.traversal.threads = threads;
        o.remesh = false;
        bve_step(s, dt, o);
        for (size_t i = 0; i < n; ++i) {
            xyz[3 * i] = s.positions[i].x;
            xyz[3 * i + 1] = s.positions[i].y;
            xyz[3 * i + 2] = s.positions[i].z;
            zeta[i] = s.zeta[i];
        }
    });
}

// bve_remesh (applications.cpp:329-371): positions <- grid, zeta/tracer <- the LSQ fits.
int csref_bve_remesh(double* xyz, double* zeta, double* tracer, const double* grid, size_t n, int neighbors) {
    return guarded([&] {
        BveState s;
        s.positions = to_vec3(xyz, n);
        s.zeta.assign(zeta, zeta + n);
        if (tracer) s.tracer.assign(tracer, tracer + n);
        s.grid_centers = to_vec3(grid, n);
        s.areas.assign(n, 0.0);
        bve_remesh(s, neighbors);
        for (size_t i = 0; i < n; ++i) {
            xyz[3 * i] = s.positions[i].x;
            xyz[3 * i + 1] = s.positions[i].y;
            xyz[3 * i + 2] = s.positions[i].z;
            zeta[i] = s.zeta[i];
            if (tracer) tracer[i] = s.tracer[i];
        }
    });
}

// bve_step with BveStepOptions::remesh on (the reference's default): RK4 then remesh onto
// grid (n x 3).
int csref_bve_step_remesh(double* xyz, double* zeta, double* tracer, const double* areas, const double* grid,
                          size_t n, double omega, double dt, double mac, int degree, int n0, int neighbors,
                          int threads) {
    return guarded([&] {
        BveState s;
        s.positions = to_vec3(xyz, n);
        s.zeta.assign(zeta, zeta + n);
        if (tracer) s.tracer.assign(tracer, tracer + n);
        s.areas.assign(areas, areas + n);
        s.grid_centers = to_vec3(grid, n);
        s.omega = omega;
        BveStepOptions o;
        o.traversal.mac = mac;
        o.traversal.degree = degree;
        o.traversal.n0 = n0;
        o.traversal.threads = threads;
        o.remesh = true;
        o.remesh_neighbors = neighbors;
        bve_step(s, dt, o);
        for (size_t i = 0; i < n; ++i) {
            xyz[3 * i] = s.positions[i].x;
            xyz[3 * i + 1] = s.positions[i].y;
            xyz[3 * i + 2] = s.positions[i].z;
            zeta[i] = s.zeta[i];
            if (tracer) tracer[i] = s.tracer[i];
        }
    });
}

}  // extern "C"
