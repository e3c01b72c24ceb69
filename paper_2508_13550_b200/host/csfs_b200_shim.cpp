// C++ host shim: the reference's summation and cluster-tree API
// (/root/reference/proj/include/csfs/summation.hpp:14-102, cluster_tree.hpp:52-81) and the
// BVE driver's bve_step / bve_remesh (applications.hpp:89-94) implemented on the B200 C-ABI
// (include/csfs_b200.h).  Compiled against the reference's headers, it replaces
// summation.cpp AND cluster_tree.cpp in a link: the whole-sum entry points
// (csfmm_sum, cstc_sum, direct_sum, summed_potential) and the stepwise ones (the ClusterTree
// constructor, upward_pass, clear_proxy_potentials, downward_pass, dual_tree_traversal,
// evaluate_pp / evaluate_pc / accumulate_cp_cc) all run on the GPU.
//
// Build switches:
//   CSFS_B200_SHIM_NAMESPACE=csfs_gpu  side by side with the reference library (tests):
//                                      free functions land in csfs_gpu; the ClusterTree
//                                      members cannot be renamed, so fill_cluster_tree()
//                                      (the constructor's body) is exported instead
//   CSFS_B200_SHIM_BVE=0               leave bve_step / bve_remesh to the reference's
//                                      applications.cpp (they then call summed_potential,
//                                      i.e. this file, for their sums)
//   CSFS_B200_DEVICES=a,b,...          (environment) the devices of the shim's context: more
//                                      than one makes csfmm_sum run target-partitioned over
//                                      all of them (csfs_b200_create_multi, NCCL)
#include <chrono>
#include <cstdlib>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "csfs/applications.hpp"
#include "csfs/cluster_tree.hpp"
#include "csfs/summation.hpp"
#include "csfs_b200.h"

#ifndef CSFS_B200_SHIM_NAMESPACE
#define CSFS_B200_SHIM_NAMESPACE csfs
#define CSFS_B200_SHIM_DROP_IN 1
#else
#define CSFS_B200_SHIM_DROP_IN 0
#endif
#ifndef CSFS_B200_SHIM_BVE
#define CSFS_B200_SHIM_BVE 1
#endif

namespace CSFS_B200_SHIM_NAMESPACE {

using csfs::Cluster;
using csfs::ClusterTree;
using csfs::InteractionLists;
using csfs::Kernel;
using csfs::ParticleSet;
using csfs::PotentialField;
using csfs::SumStats;
using csfs::TraversalConfig;

namespace {

std::vector<int> devices_from_env() {
    std::vector<int> d;
    if (const char* e = std::getenv("CSFS_B200_DEVICES")) {
        std::stringstream ss(e);
        std::string tok;
        while (std::getline(ss, tok, ','))
            if (!tok.empty()) d.push_back(std::stoi(tok));
    }
    if (d.empty()) d.push_back(0);
    return d;
}

// One context per host thread (the C-ABI contract: calls on a context are serialized).
csfs_b200_ctx* thread_ctx() {
    thread_local struct Holder {
        csfs_b200_ctx* c = nullptr;
        Holder() {
            const std::vector<int> dev = devices_from_env();
            const int rc = dev.size() == 1 ? csfs_b200_create(&c, dev[0])
                                           : csfs_b200_create_multi(&c, int(dev.size()), dev.data());
            if (rc != CSFS_B200_OK)
                throw std::runtime_error("csfs_b200: no usable sm_100 device (there is no CPU fallback); code " +
                                         std::to_string(rc));
        }
        ~Holder() { csfs_b200_destroy(c); }
    } holder;
    return holder.c;
}

void check(int rc) {
    if (rc == CSFS_B200_OK) return;
    const std::string msg = csfs_b200_last_error(thread_ctx());
    if (rc == CSFS_B200_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error("csfs_b200: " + msg);
}

csfs_b200_kernel to_c(const Kernel& k) { return {int(k.kind), k.sal.a1, k.sal.b0, k.sal.b1, k.sal.rho_ratio}; }

const double* xyz_of(const std::vector<csfs::Vec3>& v) { return v.empty() ? nullptr : &v[0].x; }

// A reference ClusterTree as the C-ABI's csfs_b200_tree_desc (reference ids, tree order).
struct TreeArrays {
    std::vector<int> ints;
    std::vector<double> dbls, proxy;
    csfs_b200_tree_desc d{};

    explicit TreeArrays(const ClusterTree& t) {
        const int ncl = int(t.clusters.size());
        const int np = t.degree + 1, npp = np * np;
        ints.resize(size_t(ncl) * 10);
        dbls.resize(size_t(ncl) * 8);
        proxy.resize(size_t(ncl) * npp * 3);
        for (int i = 0; i < ncl; ++i) {
            const Cluster& c = t.clusters[i];
            int* r = &ints[size_t(i) * 10];
            r[0] = c.face;
            r[1] = c.begin;
            r[2] = c.end;
            r[3] = c.parent;
            r[4] = c.depth;
            r[5] = c.child_count;
            for (int q = 0; q < 4; ++q) r[6 + q] = q < c.child_count ? c.children[q] : -1;
            double* g = &dbls[size_t(i) * 8];
            g[0] = c.bounds.xi0;
            g[1] = c.bounds.xi1;
            g[2] = c.bounds.eta0;
            g[3] = c.bounds.eta1;
            g[4] = c.center.x;
            g[5] = c.center.y;
            g[6] = c.center.z;
            g[7] = c.radius;
            if (int(c.interp.proxy_points.size()) != npp)
                throw std::invalid_argument("cluster interpolant does not match the tree degree");
            for (int k = 0; k < npp; ++k) {
                double* q = &proxy[(size_t(i) * npp + k) * 3];
                q[0] = c.interp.proxy_points[k].x;
                q[1] = c.interp.proxy_points[k].y;
                q[2] = c.interp.proxy_points[k].z;
            }
        }
        d.n = t.particle_count();
        d.n_clusters = ncl;
        d.degree = t.degree;
        d.perm = t.perm.data();
        d.xyz = xyz_of(t.points);
        d.xi = t.xi.data();
        d.eta = t.eta.data();
        d.ints = ints.data();
        d.dbls = dbls.data();
        d.proxy = proxy.data();
    }
};

// Per-cluster vectors of a tree as one flat array (reference ids); empty ones as zeros.
std::vector<double> flatten(const ClusterTree& t, std::vector<double> Cluster::*field, size_t per) {
    std::vector<double> f(t.clusters.size() * per, 0.0);
    for (size_t i = 0; i < t.clusters.size(); ++i) {
        const std::vector<double>& v = t.clusters[i].*field;
        if (v.empty()) continue;
        if (v.size() != per) throw std::invalid_argument("per-cluster proxy data has the wrong size");
        std::copy(v.begin(), v.end(), f.begin() + i * per);
    }
    return f;
}

std::vector<int> flat_pairs(const std::vector<std::pair<int, int>>& l) {
    std::vector<int> f(2 * l.size());
    for (size_t e = 0; e < l.size(); ++e) {
        f[2 * e] = l[e].first;
        f[2 * e + 1] = l[e].second;
    }
    return f;
}

}  // namespace

// ---- the ClusterTree constructor's body (cluster_tree.cpp:29-147) on the device ----------
// `tree` must carry degree / n0 / shrunk / cheb (the constructor's member initialisers).
void fill_cluster_tree(ClusterTree& tree, const ParticleSet& particles) {
    csfs_b200_ctx* c = thread_ctx();
    int ncl = 0, depth = 0;
    check(csfs_b200_tree_build(c, xyz_of(particles.positions), particles.size(), tree.degree, tree.n0,
                               tree.shrunk ? 1 : 0, &ncl, &depth));
    const size_t n = particles.size();
    const int np = tree.degree + 1, npp = np * np;
    std::vector<int> ints(size_t(ncl) * 10);
    std::vector<double> dbls(size_t(ncl) * 8), proxy(size_t(ncl) * npp * 3), xyz(3 * n);
    tree.perm.resize(n);
    tree.xi.resize(n);
    tree.eta.resize(n);
    check(csfs_b200_tree_export(c, 0, tree.perm.data(), ints.data(), dbls.data(), proxy.data()));
    check(csfs_b200_tree_particles(c, 0, xyz.data(), tree.xi.data(), tree.eta.data()));
    tree.points.resize(n);
    for (size_t i = 0; i < n; ++i) tree.points[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    tree.clusters.assign(ncl, Cluster{});
    for (int i = 0; i < ncl; ++i) {
        Cluster& k = tree.clusters[i];
        const int* r = &ints[size_t(i) * 10];
        const double* g = &dbls[size_t(i) * 8];
        k.face = r[0];
        k.begin = r[1];
        k.end = r[2];
        k.parent = r[3];
        k.depth = r[4];
        k.child_count = r[5];
        for (int q = 0; q < 4; ++q) k.children[q] = q < r[5] ? r[6 + q] : -1;
        k.bounds = {g[0], g[1], g[2], g[3]};
        k.center = {g[4], g[5], g[6]};
        k.radius = g[7];
        // CellInterpolant (interpolation.cpp:51-68): mid / half / mapped nodes in its
        // arithmetic; the proxy points are the device's
        csfs::CellInterpolant& ip = k.interp;
        ip.face = k.face;
        ip.rect = k.bounds;
        ip.degree = tree.degree;
        ip.xi_mid = 0.5 * (k.bounds.xi0 + k.bounds.xi1);
        ip.xi_half = 0.5 * (k.bounds.xi1 - k.bounds.xi0);
        ip.eta_mid = 0.5 * (k.bounds.eta0 + k.bounds.eta1);
        ip.eta_half = 0.5 * (k.bounds.eta1 - k.bounds.eta0);
        ip.xi_nodes.resize(np);
        ip.eta_nodes.resize(np);
        for (int q = 0; q < np; ++q) {
            ip.xi_nodes[q] = ip.xi_mid + ip.xi_half * tree.cheb.nodes[q];
            ip.eta_nodes[q] = ip.eta_mid + ip.eta_half * tree.cheb.nodes[q];
        }
        ip.proxy_points.resize(npp);
        for (int q = 0; q < npp; ++q) {
            const double* p = &proxy[(size_t(i) * npp + q) * 3];
            ip.proxy_points[q] = {p[0], p[1], p[2]};
        }
    }
    tree.levels.assign(depth + 1, {});
    for (int i = 0; i < ncl; ++i) tree.levels[tree.clusters[i].depth].push_back(i);
}

// ---- stepwise API (cluster_tree.hpp:69-81, summation.hpp:63-102) ------------------------

void upward_pass(ClusterTree& tree, const std::vector<double>& weights) {
    if (weights.size() != tree.particle_count())
        throw std::invalid_argument("weight count does not match the tree's particle count");
    const TreeArrays a(tree);
    const size_t npp = size_t(tree.degree + 1) * (tree.degree + 1);
    std::vector<double> pw(tree.clusters.size() * npp);
    check(csfs_b200_upward_tree(thread_ctx(), &a.d, weights.data(), pw.data()));
    for (size_t i = 0; i < tree.clusters.size(); ++i)
        tree.clusters[i].proxy_weights.assign(pw.begin() + i * npp, pw.begin() + (i + 1) * npp);
}

void clear_proxy_potentials(ClusterTree& tree, int out_dim) {
    const size_t per = size_t(tree.degree + 1) * (tree.degree + 1) * out_dim;
    for (Cluster& c : tree.clusters) c.proxy_potentials.assign(per, 0.0);
}

void downward_pass(ClusterTree& tree, int out_dim, std::vector<double>& out) {
    if (out.size() != tree.particle_count() * size_t(out_dim))
        throw std::invalid_argument("output size does not match particle count and out_dim");
    bool any = false;
    for (const Cluster& c : tree.clusters) any = any || !c.proxy_potentials.empty();
    if (!any) return;  // nothing accumulated: the reference skips every cluster
    const size_t per = size_t(tree.degree + 1) * (tree.degree + 1) * out_dim;
    std::vector<double> q = flatten(tree, &Cluster::proxy_potentials, per);
    const TreeArrays a(tree);
    check(csfs_b200_downward_tree(thread_ctx(), &a.d, out_dim, q.data(), out.data()));
    for (size_t i = 0; i < tree.clusters.size(); ++i)  // children received their parents' share
        if (!tree.clusters[i].proxy_potentials.empty())
            std::copy(q.begin() + i * per, q.begin() + (i + 1) * per, tree.clusters[i].proxy_potentials.begin());
}

const char* method_name(csfs::Method m) {
    return m == csfs::Method::Direct ? "direct" : m == csfs::Method::Cstc ? "cstc" : "csfmm";
}

csfs::Method parse_method(const std::string& name) {
    static const std::pair<const char*, csfs::Method> kNames[] = {
        {"direct", csfs::Method::Direct}, {"cstc", csfs::Method::Cstc}, {"csfmm", csfs::Method::Csfmm}};
    for (const auto& kv : kNames)
        if (name == kv.first) return kv.second;
    throw std::invalid_argument("unknown method: " + name);
}

// The multipole acceptance test (summation.cpp:123-134); the device restates it in
// traverse.cu with the same operation order.
bool well_separated(const csfs::Vec3& c0, double r0, const csfs::Vec3& c1, double r1, double mac) {
    const double R = csfs::chordal_distance(c0, c1);
    return R > 0.0 && r0 + r1 < mac * R;
}
bool well_separated_pc(const csfs::Vec3& target, const Cluster& cluster, double mac) {
    return CSFS_B200_SHIM_NAMESPACE::well_separated(target, 0.0, cluster.center, cluster.radius, mac);
}
bool well_separated_cc(const Cluster& ct, const Cluster& cs, double mac) {
    return CSFS_B200_SHIM_NAMESPACE::well_separated(ct.center, ct.radius, cs.center, cs.radius, mac);
}

InteractionLists dual_tree_traversal(const ClusterTree& targets, const ClusterTree& sources, double mac, int n0) {
    const TreeArrays t(targets), s(sources);
    csfs_b200_ctx* c = thread_ctx();
    long long counts[4] = {0, 0, 0, 0};
    check(csfs_b200_traversal_tree(c, &t.d, &s.d, mac, n0, counts));
    std::vector<int> f[4];
    for (int k = 0; k < 4; ++k) f[k].resize(2 * size_t(counts[k]) + 2);
    check(csfs_b200_lists_export(c, counts, f[0].data(), f[1].data(), f[2].data(), f[3].data()));
    InteractionLists L;
    std::vector<std::pair<int, int>>* dst[4] = {&L.pp, &L.pc, &L.cp, &L.cc};
    for (int k = 0; k < 4; ++k) {
        dst[k]->resize(size_t(counts[k]));
        for (long long e = 0; e < counts[k]; ++e) (*dst[k])[e] = {f[k][2 * e], f[k][2 * e + 1]};
    }
    return L;
}

void evaluate_pp(const ClusterTree& targets, const ClusterTree& sources, const std::vector<double>& source_weights,
                 const Kernel& kernel, const std::vector<std::pair<int, int>>& list, PotentialField& out,
                 int /*threads*/) {
    if (source_weights.size() != sources.particle_count())
        throw std::invalid_argument("weight count does not match particle count");
    if (out.values.size() < targets.particle_count() * size_t(kernel.out_dim()))
        throw std::invalid_argument("output field is smaller than the target set");
    const TreeArrays t(targets), s(sources);
    const csfs_b200_kernel k = to_c(kernel);
    const std::vector<int> pp = flat_pairs(list);
    check(csfs_b200_evaluate_tree(thread_ctx(), &t.d, &s.d, source_weights.data(), nullptr, &k, pp.data(),
                                  (long long)list.size(), nullptr, 0, nullptr, 0, nullptr, 0, out.values.data(),
                                  nullptr));
}

void evaluate_pc(const ClusterTree& targets, const ClusterTree& sources, const Kernel& kernel,
                 const std::vector<std::pair<int, int>>& list, PotentialField& out, int /*threads*/) {
    if (out.values.size() < targets.particle_count() * size_t(kernel.out_dim()))
        throw std::invalid_argument("output field is smaller than the target set");
    const TreeArrays t(targets), s(sources);
    const size_t npp = size_t(sources.degree + 1) * (sources.degree + 1);
    const std::vector<double> pw = flatten(sources, &Cluster::proxy_weights, npp);
    const csfs_b200_kernel k = to_c(kernel);
    const std::vector<int> pc = flat_pairs(list);
    check(csfs_b200_evaluate_tree(thread_ctx(), &t.d, &s.d, nullptr, pw.data(), &k, nullptr, 0, pc.data(),
                                  (long long)list.size(), nullptr, 0, nullptr, 0, out.values.data(), nullptr));
}

void accumulate_cp_cc(ClusterTree& targets, const ClusterTree& sources, const std::vector<double>& source_weights,
                      const Kernel& kernel, const std::vector<std::pair<int, int>>& cp,
                      const std::vector<std::pair<int, int>>& cc, int /*threads*/) {
    if (source_weights.size() != sources.particle_count())
        throw std::invalid_argument("weight count does not match particle count");
    const TreeArrays t(targets), s(sources);
    const size_t npp = size_t(targets.degree + 1) * (targets.degree + 1);
    const size_t per = npp * kernel.out_dim();
    std::vector<double> q = flatten(targets, &Cluster::proxy_potentials, per);
    const std::vector<double> pw =
        cc.empty() ? std::vector<double>() : flatten(sources, &Cluster::proxy_weights, npp);
    const csfs_b200_kernel k = to_c(kernel);
    const std::vector<int> fcp = flat_pairs(cp), fcc = flat_pairs(cc);
    check(csfs_b200_evaluate_tree(thread_ctx(), &t.d, &s.d, source_weights.data(), cc.empty() ? nullptr : pw.data(),
                                  &k, nullptr, 0, nullptr, 0, fcp.data(), (long long)cp.size(), fcc.data(),
                                  (long long)cc.size(), nullptr, q.data()));
    for (size_t i = 0; i < targets.clusters.size(); ++i) {
        std::vector<double>& v = targets.clusters[i].proxy_potentials;
        if (v.empty()) v.assign(per, 0.0);
        std::copy(q.begin() + i * per, q.begin() + (i + 1) * per, v.begin());
    }
}

// ---- whole sums (summation.hpp:74-88) ----------------------------------------------------

namespace {
void copy_stats(const csfs_b200_stats& st, SumStats* stats, int which_trees) {
    *stats = SumStats{};
    stats->t_tree_build = st.t_tree_build;
    stats->t_upward = st.t_upward;
    stats->t_traversal = st.t_traversal;
    stats->t_downward = st.t_downward;
    stats->t_total = st.t_total;
    stats->pp = st.pp;
    stats->pc = st.pc;
    stats->cp = st.cp;
    stats->cc = st.cc;
    csfs_b200_ctx* c = thread_ctx();
    auto tree = [&](csfs::TreeStats& t, int which, int depth, int ncl, int leaves) {
        t.depth = depth;
        t.cluster_count = ncl;
        t.leaf_count = leaves;
        int len = 0;
        check(csfs_b200_leaf_histogram(c, which, nullptr, 0, &len));
        t.leaf_size_histogram.assign(len, 0);
        check(csfs_b200_leaf_histogram(c, which, t.leaf_size_histogram.data(), len, &len));
    };
    tree(stats->source_tree, 1, st.src_depth, st.src_clusters, st.src_leaves);
    if (which_trees == 2) tree(stats->target_tree, 0, st.tgt_depth, st.tgt_clusters, st.tgt_leaves);
}
}  // namespace

PotentialField csfmm_sum(const ParticleSet& targets, const ParticleSet& sources, const Kernel& kernel,
                         const TraversalConfig& config, SumStats* stats) {
    if (sources.weights.size() != sources.positions.size())
        throw std::invalid_argument("weight count does not match the tree's particle count");
    const csfs_b200_kernel k = to_c(kernel);
    const csfs_b200_config c{config.mac, config.degree, config.n0, config.shrink ? 1 : 0};
    PotentialField f;
    f.out_dim = kernel.out_dim();
    f.values.resize(targets.size() * f.out_dim);
    csfs_b200_stats st{};
    check(csfs_b200_csfmm(thread_ctx(), xyz_of(targets.positions), targets.size(), xyz_of(sources.positions),
                          sources.weights.data(), sources.size(), &k, &c, f.values.data(), &st));
    if (stats) copy_stats(st, stats, 2);
    return f;
}

PotentialField cstc_sum(const ParticleSet& targets, const ParticleSet& sources, const Kernel& kernel,
                        const TraversalConfig& config, SumStats* stats) {
    if (sources.weights.size() != sources.positions.size())
        throw std::invalid_argument("weight count does not match the tree's particle count");
    const csfs_b200_kernel k = to_c(kernel);
    const csfs_b200_config c{config.mac, config.degree, config.n0, config.shrink ? 1 : 0};
    PotentialField f;
    f.out_dim = kernel.out_dim();
    f.values.resize(targets.size() * f.out_dim);
    csfs_b200_stats st{};
    check(csfs_b200_cstc(thread_ctx(), xyz_of(targets.positions), targets.size(), xyz_of(sources.positions),
                         sources.weights.data(), sources.size(), &k, &c, f.values.data(), &st));
    if (stats) copy_stats(st, stats, 1);  // the treecode builds the source tree only
    return f;
}

PotentialField direct_sum(const ParticleSet& targets, const ParticleSet& sources, const Kernel& kernel,
                          int /*threads*/) {
    if (sources.weights.size() != sources.positions.size())
        throw std::invalid_argument("source weights and positions differ in length");
    const csfs_b200_kernel k = to_c(kernel);
    PotentialField f;
    f.out_dim = kernel.out_dim();
    f.values.assign(targets.size() * f.out_dim, 0.0);
    check(csfs_b200_direct(thread_ctx(), xyz_of(targets.positions), targets.size(), xyz_of(sources.positions),
                           sources.weights.data(), sources.size(), &k, f.values.data()));
    return f;
}

// summed_potential (summation.cpp:423-440): dispatch on config.method.
PotentialField summed_potential(const ParticleSet& targets, const ParticleSet& sources, const Kernel& kernel,
                                const TraversalConfig& config, SumStats* stats) {
    switch (config.method) {
        case csfs::Method::Direct: {
            const auto t0 = std::chrono::steady_clock::now();
            PotentialField f = CSFS_B200_SHIM_NAMESPACE::direct_sum(targets, sources, kernel, config.threads);
            if (stats) {
                *stats = SumStats{};
                stats->t_traversal = stats->t_total =
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                stats->pp = targets.size() * sources.size();
            }
            return f;
        }
        case csfs::Method::Cstc: return CSFS_B200_SHIM_NAMESPACE::cstc_sum(targets, sources, kernel, config, stats);
        default: return CSFS_B200_SHIM_NAMESPACE::csfmm_sum(targets, sources, kernel, config, stats);
    }
}

#if CSFS_B200_SHIM_BVE
// bve_remesh (applications.hpp:94, applications.cpp:329-371)
void bve_remesh(csfs::BveState& state, int neighbors) {
    const size_t n = state.positions.size();
    if (state.zeta.size() != n || state.grid_centers.size() != n || (!state.tracer.empty() && state.tracer.size() != n))
        throw std::invalid_argument("positions, zeta, tracer and grid centres must have one entry per particle");
    if (n == 0) return;
    check(csfs_b200_bve_remesh(thread_ctx(), &state.positions[0].x, state.zeta.data(),
                               state.tracer.empty() ? nullptr : state.tracer.data(), &state.grid_centers[0].x, n,
                               neighbors));
}

// bve_step (applications.hpp:89, applications.cpp:378-412): RK4 on the device, then the
// remesh when options.remesh.
void bve_step(csfs::BveState& state, double dt, const csfs::BveStepOptions& options) {
    const TraversalConfig& t = options.traversal;
    const csfs_b200_config c{t.mac, t.degree, t.n0, t.shrink ? 1 : 0};
    check(csfs_b200_bve_step(thread_ctx(), state.positions.empty() ? nullptr : &state.positions[0].x,
                             state.zeta.data(), state.areas.data(), state.positions.size(), state.omega, dt, &c,
                             nullptr));
    state.time += dt;
    if (options.remesh) CSFS_B200_SHIM_NAMESPACE::bve_remesh(state, options.remesh_neighbors);
}
#endif

}  // namespace CSFS_B200_SHIM_NAMESPACE

#if CSFS_B200_SHIM_DROP_IN
namespace csfs {

// The reference's ClusterTree members (cluster_tree.hpp:54, :65): the constructor's member
// initialisers as declared, its body on the device.
ClusterTree::ClusterTree(const ParticleSet& particles, int degree_, int n0_, bool shrink)
    : degree(degree_), n0(n0_), shrunk(shrink), cheb(degree_) {
    fill_cluster_tree(*this, particles);
}

TreeStats ClusterTree::stats() const {
    TreeStats s;
    s.depth = int(levels.size()) - 1;
    s.cluster_count = int(clusters.size());
    for (const Cluster& c : clusters) {
        if (c.child_count != 0) continue;
        const int k = c.end - c.begin;
        s.leaf_count += 1;
        if (k >= int(s.leaf_size_histogram.size())) s.leaf_size_histogram.resize(size_t(k) + 1, 0);
        s.leaf_size_histogram[size_t(k)] += 1;
    }
    return s;
}

}  // namespace csfs
#endif
