// TEST (GPU): the C++ shim (paper_2508_13550_b200/host/csfs_b200_shim.cpp), built against
// the reference's own headers and types, against the reference library's csfs::csfmm_sum /
// direct_sum on the reference's own grids and weights — the drop-in exercised from C++.
// Prints one line per case: name rel_l2 pp pc cp cc (GPU) pp pc cp cc (reference).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "csfs/applications.hpp"
#include "csfs/summation.hpp"

namespace csfs_gpu {
csfs::PotentialField csfmm_sum(const csfs::ParticleSet&, const csfs::ParticleSet&, const csfs::Kernel&,
                               const csfs::TraversalConfig&, csfs::SumStats*);
csfs::PotentialField direct_sum(const csfs::ParticleSet&, const csfs::ParticleSet&, const csfs::Kernel&, int);
csfs::PotentialField summed_potential(const csfs::ParticleSet&, const csfs::ParticleSet&, const csfs::Kernel&,
                                      const csfs::TraversalConfig&, csfs::SumStats*);
void bve_step(csfs::BveState&, double, const csfs::BveStepOptions&);
}  // namespace csfs_gpu

using namespace csfs;

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
