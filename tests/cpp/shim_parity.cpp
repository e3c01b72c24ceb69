// TEST (GPU): the C++ shim (paper_2508_13550_b200/host/csfs_b200_shim.cpp), built against
// the reference's own headers and types, against the reference library's csfs::csfmm_sum /
// direct_sum on the reference's own grids and weights — the drop-in exercised from C++.
// Prints one line per case: name rel_l2 pp pc cp cc (GPU) pp pc cp cc (reference).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "csfs/applications.hpp"
#include "csfs/cluster_tree.hpp"
#include "csfs/summation.hpp"

namespace csfs_gpu {
csfs::PotentialField csfmm_sum(const csfs::ParticleSet&, const csfs::ParticleSet&, const csfs::Kernel&,
                               const csfs::TraversalConfig&, csfs::SumStats*);
csfs::PotentialField direct_sum(const csfs::ParticleSet&, const csfs::ParticleSet&, const csfs::Kernel&, int);
csfs::PotentialField summed_potential(const csfs::ParticleSet&, const csfs::ParticleSet&, const csfs::Kernel&,
                                      const csfs::TraversalConfig&, csfs::SumStats*);
void bve_step(csfs::BveState&, double, const csfs::BveStepOptions&);
void fill_cluster_tree(csfs::ClusterTree&, const csfs::ParticleSet&);
void upward_pass(csfs::ClusterTree&, const std::vector<double>&);
void downward_pass(csfs::ClusterTree&, int, std::vector<double>&);
csfs::InteractionLists dual_tree_traversal(const csfs::ClusterTree&, const csfs::ClusterTree&, double, int);
void evaluate_pp(const csfs::ClusterTree&, const csfs::ClusterTree&, const std::vector<double>&, const csfs::Kernel&,
                 const std::vector<std::pair<int, int>>&, csfs::PotentialField&, int);
void evaluate_pc(const csfs::ClusterTree&, const csfs::ClusterTree&, const csfs::Kernel&,
                 const std::vector<std::pair<int, int>>&, csfs::PotentialField&, int);
void accumulate_cp_cc(csfs::ClusterTree&, const csfs::ClusterTree&, const std::vector<double>&, const csfs::Kernel&,
                      const std::vector<std::pair<int, int>>&, const std::vector<std::pair<int, int>>&, int);
}  // namespace csfs_gpu

using namespace csfs;

static double rel_l2(const PotentialField& a, const PotentialField& b);

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, std::fabs(a[i] - b[i]));
        den = std::max(den, std::fabs(b[i]));
    }
    return a.size() == b.size() ? num / (den > 0 ? den : 1.0) : 1e300;
}

static bool same_sets(std::vector<std::pair<int, int>> a, std::vector<std::pair<int, int>> b) {
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    return a == b;
}

// The stepwise API on the GPU (csfs_gpu::*) against the reference's own (csfs::*), piece by
// piece on the same trees: ClusterTree, upward_pass, dual_tree_traversal, evaluate_pp /
// evaluate_pc / accumulate_cp_cc, downward_pass, and the pieces chained into a whole sum.
static int stepwise_case(const char* name, const ParticleSet& p, const char* kname, int degree, int n0,
                         double mac) {
    int bad = 0;
    const Kernel k = Kernel::parse(kname);
    const int dim = k.out_dim();
    ClusterTree r(p, degree, n0, true);  // the reference's tree
    ClusterTree g = r;                   // same members, refilled by the GPU
    csfs_gpu::fill_cluster_tree(g, p);
    bool topo = g.perm == r.perm && g.clusters.size() == r.clusters.size() && g.levels == r.levels;
    double geo = 0;
    for (size_t i = 0; topo && i < r.clusters.size(); ++i) {
        const Cluster &a = g.clusters[i], &b = r.clusters[i];
        topo = a.face == b.face && a.begin == b.begin && a.end == b.end && a.parent == b.parent &&
               a.depth == b.depth && a.child_count == b.child_count && a.children == b.children;
        const double d[] = {a.bounds.xi0 - b.bounds.xi0, a.bounds.xi1 - b.bounds.xi1, a.bounds.eta0 - b.bounds.eta0,
                            a.bounds.eta1 - b.bounds.eta1, a.radius - b.radius, norm(a.center - b.center),
                            a.interp.xi_mid - b.interp.xi_mid, a.interp.eta_half - b.interp.eta_half};
        for (double x : d) geo = std::max(geo, std::fabs(x));
        for (size_t q = 0; q < a.interp.proxy_points.size(); ++q)
            geo = std::max(geo, norm(a.interp.proxy_points[q] - b.interp.proxy_points[q]));
    }
    for (size_t t = 0; topo && t < r.xi.size(); ++t) {
        geo = std::max(geo, std::fabs(g.xi[t] - r.xi[t]) + std::fabs(g.eta[t] - r.eta[t]));
        geo = std::max(geo, norm(g.points[t] - r.points[t]));
    }
    // upward pass
    csfs_gpu::upward_pass(g, p.weights);
    upward_pass(r, p.weights);
    std::vector<double> pwg, pwr;
    for (size_t i = 0; i < r.clusters.size(); ++i) {
        pwg.insert(pwg.end(), g.clusters[i].proxy_weights.begin(), g.clusters[i].proxy_weights.end());
        pwr.insert(pwr.end(), r.clusters[i].proxy_weights.begin(), r.clusters[i].proxy_weights.end());
    }
    const double up = max_rel(pwg, pwr);
    // traversal
    const InteractionLists lg = csfs_gpu::dual_tree_traversal(g, g, mac, n0);
    const InteractionLists lr = dual_tree_traversal(r, r, mac, n0);
    const bool lists = same_sets(lg.pp, lr.pp) && same_sets(lg.pc, lr.pc) && same_sets(lg.cp, lr.cp) &&
                       same_sets(lg.cc, lr.cc);
    // the evaluations, each on the reference's own lists
    PotentialField fg{dim, std::vector<double>(p.size() * dim, 0.0)}, fr = fg;
    csfs_gpu::evaluate_pp(g, g, p.weights, k, lr.pp, fg, 0);
    evaluate_pp(r, r, p.weights, k, lr.pp, fr, 0);
    const double epp = max_rel(fg.values, fr.values);
    csfs_gpu::evaluate_pc(g, g, k, lr.pc, fg, 0);
    evaluate_pc(r, r, k, lr.pc, fr, 0);
    clear_proxy_potentials(g, dim);
    clear_proxy_potentials(r, dim);
    csfs_gpu::accumulate_cp_cc(g, g, p.weights, k, lr.cp, lr.cc, 0);
    accumulate_cp_cc(r, r, p.weights, k, lr.cp, lr.cc, 0);
    std::vector<double> qg, qr;
    for (size_t i = 0; i < r.clusters.size(); ++i) {
        qg.insert(qg.end(), g.clusters[i].proxy_potentials.begin(), g.clusters[i].proxy_potentials.end());
        qr.insert(qr.end(), r.clusters[i].proxy_potentials.begin(), r.clusters[i].proxy_potentials.end());
    }
    const double ecc = max_rel(qg, qr);
    // downward pass of the accumulated proxy potentials, into the near field
    csfs_gpu::downward_pass(g, dim, fg.values);
    downward_pass(r, dim, fr.values);
    const double whole = rel_l2(fg, fr);
    const PotentialField ref_sum = csfmm_sum(p, p, k, [&] {
        TraversalConfig c;
        c.degree = degree;
        c.n0 = n0;
        c.mac = mac;
        return c;
    }());
    const double vs_csfmm = rel_l2(fg, ref_sum);
    std::printf("stepwise_%s topo %d geo %.1e upward %.1e lists %d pp %.1e cpcc %.1e chain %.1e vs_csfmm %.1e\n", name,
                int(topo), geo, up, int(lists), epp, ecc, whole, vs_csfmm);
    if (!topo || !(geo < 1e-13) || !(up < 1e-12) || !lists || !(epp < 1e-12) || !(ecc < 1e-12) || !(whole < 1e-10) ||
        !(vs_csfmm < 1e-10))
        ++bad;
    // downward pass identity (acceptance.cpp:249-279): random potentials on every cluster
    {
        std::mt19937 rng(7);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        clear_proxy_potentials(r, 1);
        for (Cluster& c : r.clusters)
            for (double& v : c.proxy_potentials) v = u(rng);
        ClusterTree g2 = r;
        std::vector<double> og(p.size(), 0.5), orr(p.size(), 0.5);
        csfs_gpu::downward_pass(g2, 1, og);
        downward_pass(r, 1, orr);
        std::vector<double> pg, pr;
        for (size_t i = 0; i < r.clusters.size(); ++i) {
            pg.insert(pg.end(), g2.clusters[i].proxy_potentials.begin(), g2.clusters[i].proxy_potentials.end());
            pr.insert(pr.end(), r.clusters[i].proxy_potentials.begin(), r.clusters[i].proxy_potentials.end());
        }
        const double d = max_rel(og, orr), dq = max_rel(pg, pr);
        std::printf("stepwise_%s_downward out %.1e pushed %.1e\n", name, d, dq);
        if (!(d < 1e-12) || !(dq < 1e-12)) ++bad;
    }
    return bad;
}

static double rel_l2(const PotentialField& a, const PotentialField& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.values.size(); ++i) {
        num += (a.values[i] - b.values[i]) * (a.values[i] - b.values[i]);
        den += b.values[i] * b.values[i];
    }
    return std::sqrt(num / den);
}

int main() {
    int bad = 0;
    struct Case { const char* name; GridKind g; int level; const char* kernel; int degree; double mac; int n0; };
    const Case cases[] = {{"ico4_laplace", GridKind::Icosahedral, 4, "laplace", 6, 0.7, -1},
                          {"cs5_sal", GridKind::CubedSphere, 5, "sal", 10, 0.6, 64},
                          {"ico4_bs", GridKind::Icosahedral, 4, "biot_savart", 6, 0.7, 40},
                          {"latlon4_biharmonic", GridKind::LatLon, 4, "biharmonic", 8, 0.6, 50}};
    for (const Case& c : cases) {
        const SphericalGrid g = build_grid(c.g, c.level);
        ParticleSet p;
        p.positions = g.centers;
        p.weights.resize(g.size());
        for (size_t i = 0; i < g.size(); ++i) p.weights[i] = real_sph_harm(4, 3, g.centers[i]) * g.areas[i];
        TraversalConfig cfg;
        cfg.degree = c.degree;
        cfg.mac = c.mac;
        cfg.n0 = c.n0;
        const Kernel k = Kernel::parse(c.kernel);
        SumStats sg, sr;
        const PotentialField fg = csfs_gpu::csfmm_sum(p, p, k, cfg, &sg);
        const PotentialField fr = csfs::csfmm_sum(p, p, k, cfg, &sr);
        const double e = rel_l2(fg, fr);
        const bool same_lists = sg.pp == sr.pp && sg.pc == sr.pc && sg.cp == sr.cp && sg.cc == sr.cc &&
                                sg.target_tree.cluster_count == sr.target_tree.cluster_count &&
                                sg.target_tree.leaf_count == sr.target_tree.leaf_count;
        std::printf("%s %.3e %zu %zu %zu %zu | %zu %zu %zu %zu\n", c.name, e, sg.pp, sg.pc, sg.cp, sg.cc, sr.pp,
                    sr.pc, sr.cp, sr.cc);
        if (!(e < 1e-10) || !same_lists) ++bad;
    }
    {  // the stepwise API
        std::mt19937 rng(424242);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        const SphericalGrid ico = build_grid(GridKind::Icosahedral, 5);
        ParticleSet p;
        p.positions = ico.centers;
        p.weights.resize(ico.size());
        for (double& w : p.weights) w = u(rng);
        bad += stepwise_case("ico5_laplace", p, "laplace", 6, 144, 0.7);
        bad += stepwise_case("ico5_bs", p, "biot_savart", 5, 60, 0.6);
        const SphericalGrid cs = build_grid(GridKind::CubedSphere, 5);
        ParticleSet q;
        q.positions = cs.centers;
        q.weights.resize(cs.size());
        for (size_t i = 0; i < cs.size(); ++i) q.weights[i] = real_sph_harm(4, 3, cs.centers[i]) * cs.areas[i];
        bad += stepwise_case("cs5_sal", q, "sal", 10, 64, 0.6);
        bad += stepwise_case("cs5_biharmonic", q, "biharmonic", 8, 50, 0.7);
        // clustered blobs: deep unbalanced trees with PC entries
        std::normal_distribution<double> nrm(0.0, 1.0);
        ParticleSet b;
        for (int c = 0; c < 4; ++c) {
            const Vec3 ctr = normalized({nrm(rng), nrm(rng), nrm(rng)});
            for (int i = 0; i < 1500; ++i)
                b.positions.push_back(normalized(ctr + Vec3{0.05 * nrm(rng), 0.05 * nrm(rng), 0.05 * nrm(rng)}));
        }
        for (int i = 0; i < 2000; ++i) b.positions.push_back(normalized({nrm(rng), nrm(rng), nrm(rng)}));
        b.weights.resize(b.positions.size());
        for (double& w : b.weights) w = u(rng);
        bad += stepwise_case("blobs_laplace", b, "laplace", 6, 48, 0.7);
    }
    {  // TreeStats::leaf_size_histogram through csfmm_sum's SumStats
        const SphericalGrid g = build_grid(GridKind::CubedSphere, 5);
        ParticleSet p;
        p.positions = g.centers;
        p.weights.assign(g.size(), 1.0);
        TraversalConfig cfg;
        cfg.n0 = 50;
        SumStats sg, sr;
        csfs_gpu::csfmm_sum(p, p, Kernel::parse("laplace"), cfg, &sg);
        csfmm_sum(p, p, Kernel::parse("laplace"), cfg, &sr);
        const bool same = sg.source_tree.leaf_size_histogram == sr.source_tree.leaf_size_histogram &&
                          sg.target_tree.leaf_size_histogram == sr.target_tree.leaf_size_histogram &&
                          !sr.target_tree.leaf_size_histogram.empty();
        std::printf("leaf_histogram %d (%zu buckets)\n", int(same), sr.target_tree.leaf_size_histogram.size());
        if (!same) ++bad;
    }
    {  // direct sum
        const SphericalGrid g = build_grid(GridKind::Icosahedral, 3);
        ParticleSet p;
        p.positions = g.centers;
        p.weights.assign(g.size(), 0.0);
        for (size_t i = 0; i < g.size(); ++i) p.weights[i] = real_sph_harm(4, 3, g.centers[i]) * g.areas[i];
        const double e = rel_l2(csfs_gpu::direct_sum(p, p, Kernel::parse("sal"), 0),
                                csfs::direct_sum(p, p, Kernel::parse("sal"), 0));
        std::printf("direct_sal %.3e\n", e);
        if (!(e < 1e-12)) ++bad;
    }
    {  // summed_potential dispatch: the treecode
        const SphericalGrid g = build_grid(GridKind::Icosahedral, 4);
        ParticleSet p;
        p.positions = g.centers;
        p.weights.resize(g.size());
        for (size_t i = 0; i < g.size(); ++i) p.weights[i] = real_sph_harm(4, 3, g.centers[i]) * g.areas[i];
        TraversalConfig cfg;
        cfg.method = Method::Cstc;
        SumStats sg, sr;
        const double e = rel_l2(csfs_gpu::summed_potential(p, p, Kernel::parse("sal"), cfg, &sg),
                                csfs::summed_potential(p, p, Kernel::parse("sal"), cfg, &sr));
        std::printf("cstc_sal %.3e %zu %zu | %zu %zu\n", e, sg.pp, sg.pc, sr.pp, sr.pc);
        if (!(e < 1e-10) || sg.pp != sr.pp || sg.pc != sr.pc) ++bad;
    }
    {  // bve_step with the reference's default options (remesh on, 12 neighbours), with a tracer
        const SphericalGrid g = build_grid(GridKind::CubedSphere, 4);
        BveState a = bve_initial(BveInit::RossbyHaurwitz, g, true), b = a;
        BveStepOptions o;
        o.traversal.degree = 6;
        o.traversal.mac = 0.7;
        csfs_gpu::bve_step(a, 0.05, o);
        bve_step(b, 0.05, o);
        double num = 0, den = 0, pos = 0;
        for (size_t i = 0; i < a.zeta.size(); ++i) {
            num += (a.zeta[i] - b.zeta[i]) * (a.zeta[i] - b.zeta[i]) + (a.tracer[i] - b.tracer[i]) * (a.tracer[i] - b.tracer[i]);
            den += b.zeta[i] * b.zeta[i] + b.tracer[i] * b.tracer[i];
            pos = std::max(pos, std::fabs(a.positions[i].x - b.positions[i].x));
        }
        const double e = std::sqrt(num / den);
        std::printf("bve_step_remesh %.3e pos %.1e time %g %g\n", e, pos, a.time, b.time);
        if (!(e < 1e-9) || pos != 0.0 || a.time != b.time) ++bad;
    }
    {  // the reference's exception contract
        ParticleSet empty, one;
        one.positions = {{0, 0, 1}};
        one.weights = {1.0};
        TraversalConfig cfg;
        for (int which = 0; which < 2; ++which) {
            std::string got_g, got_r;
            try { csfs_gpu::csfmm_sum(which ? one : empty, one, Kernel::parse("laplace"), cfg, nullptr); }
            catch (const std::invalid_argument& e) { got_g = e.what(); }
            try { csfs::csfmm_sum(which ? one : empty, one, Kernel::parse("laplace"), cfg, nullptr); }
            catch (const std::invalid_argument& e) { got_r = e.what(); }
            if (which == 1) {  // n0 = 0
                TraversalConfig z;
                z.n0 = 0;
                got_g.clear();
                got_r.clear();
                try { csfs_gpu::csfmm_sum(one, one, Kernel::parse("laplace"), z, nullptr); }
                catch (const std::invalid_argument& e) { got_g = e.what(); }
                try { csfs::csfmm_sum(one, one, Kernel::parse("laplace"), z, nullptr); }
                catch (const std::invalid_argument& e) { got_r = e.what(); }
            }
            std::printf("error '%s' | '%s'\n", got_g.c_str(), got_r.c_str());
            if (got_g != got_r || got_g.empty()) ++bad;
        }
    }
    std::printf(bad ? "FAIL %d\n" : "OK\n", bad);
    return bad ? 1 : 0;
}
