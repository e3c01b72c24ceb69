// C++ host shim: the reference's csfs::csfmm_sum / cstc_sum / direct_sum / summed_potential
// signatures (/root/reference/proj/include/csfs/summation.hpp:74-88) and the BVE driver's
// bve_step / bve_remesh (applications.hpp:89-94) implemented on the B200 C-ABI
// (include/csfs_b200.h).  A maintainer compiles this file against the reference's headers
// and links libcsfs_b200.so in place of summation.cpp's csfmm_sum.
// CSFS_B200_SHIM_NAMESPACE lets the tests build it side by side with the reference
// (tests/cpp/shim_parity.cpp) without a symbol clash.
#include <chrono>
#include <stdexcept>
#include <string>

#include "csfs/applications.hpp"
#include "csfs/summation.hpp"
#include "csfs_b200.h"

#ifndef CSFS_B200_SHIM_NAMESPACE
#define CSFS_B200_SHIM_NAMESPACE csfs
#endif

namespace CSFS_B200_SHIM_NAMESPACE {

using csfs::Kernel;
using csfs::ParticleSet;
using csfs::PotentialField;
using csfs::SumStats;
using csfs::TraversalConfig;

namespace {

// One context per host thread (the C-ABI contract: calls on a context are serialized).
csfs_b200_ctx* thread_ctx() {
    thread_local struct Holder {
        csfs_b200_ctx* c = nullptr;
        Holder() {
            if (csfs_b200_create(&c, 0) != CSFS_B200_OK)
                throw std::runtime_error("csfs_b200: no usable sm_100 device (there is no CPU fallback)");
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

csfs_b200_kernel to_c(const Kernel& k) {
    return {int(k.kind), k.sal.a1, k.sal.b0, k.sal.b1, k.sal.rho_ratio};
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
    const double* tx = targets.positions.empty() ? nullptr : &targets.positions[0].x;
    const double* sx = sources.positions.empty() ? nullptr : &sources.positions[0].x;
    check(csfs_b200_csfmm(thread_ctx(), tx, targets.size(), sx, sources.weights.data(), sources.size(), &k,
                          &c, f.values.data(), &st));
    if (stats) {
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
        stats->source_tree.depth = st.src_depth;
        stats->source_tree.cluster_count = st.src_clusters;
        stats->source_tree.leaf_count = st.src_leaves;
        stats->target_tree.depth = st.tgt_depth;
        stats->target_tree.cluster_count = st.tgt_clusters;
        stats->target_tree.leaf_count = st.tgt_leaves;
    }
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
    const double* tx = targets.positions.empty() ? nullptr : &targets.positions[0].x;
    const double* sx = sources.positions.empty() ? nullptr : &sources.positions[0].x;
    check(csfs_b200_cstc(thread_ctx(), tx, targets.size(), sx, sources.weights.data(), sources.size(), &k, &c,
                         f.values.data(), &st));
    if (stats) {
        *stats = SumStats{};
        stats->t_tree_build = st.t_tree_build;
        stats->t_upward = st.t_upward;
        stats->t_traversal = st.t_traversal;
        stats->t_total = st.t_total;
        stats->pp = st.pp;
        stats->pc = st.pc;
        stats->source_tree.depth = st.src_depth;
        stats->source_tree.cluster_count = st.src_clusters;
        stats->source_tree.leaf_count = st.src_leaves;
    }
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
    const double* tx = targets.positions.empty() ? nullptr : &targets.positions[0].x;
    const double* sx = sources.positions.empty() ? nullptr : &sources.positions[0].x;
    check(csfs_b200_direct(thread_ctx(), tx, targets.size(), sx, sources.weights.data(), sources.size(), &k,
                           f.values.data()));
    return f;
}

}  // namespace CSFS_B200_SHIM_NAMESPACE

namespace CSFS_B200_SHIM_NAMESPACE {

// summed_potential (summation.cpp:423-440): dispatch on config.method.
csfs::PotentialField summed_potential(const csfs::ParticleSet& targets, const csfs::ParticleSet& sources,
                                      const csfs::Kernel& kernel, const csfs::TraversalConfig& config,
                                      csfs::SumStats* stats) {
    switch (config.method) {
        case csfs::Method::Direct: {
            const auto t0 = std::chrono::steady_clock::now();
            csfs::PotentialField f = CSFS_B200_SHIM_NAMESPACE::direct_sum(targets, sources, kernel, config.threads);
            if (stats) {
                *stats = csfs::SumStats{};
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

}  // namespace CSFS_B200_SHIM_NAMESPACE

namespace CSFS_B200_SHIM_NAMESPACE {

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
    const csfs::TraversalConfig& t = options.traversal;
    const csfs_b200_config c{t.mac, t.degree, t.n0, t.shrink ? 1 : 0};
    check(csfs_b200_bve_step(thread_ctx(), state.positions.empty() ? nullptr : &state.positions[0].x,
                             state.zeta.data(), state.areas.data(), state.positions.size(), state.omega, dt, &c,
                             nullptr));
    state.time += dt;
    if (options.remesh) CSFS_B200_SHIM_NAMESPACE::bve_remesh(state, options.remesh_neighbors);
}

}  // namespace CSFS_B200_SHIM_NAMESPACE
