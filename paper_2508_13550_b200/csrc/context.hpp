// The C-ABI context (include/csfs_b200.h: csfs_b200_ctx) and the host helpers shared by
// capi.cu (single-device entry points) and partition.cu (the multi-GPU runtime).
//
// A context owns one device, its streams and every device buffer of the engine.  A
// multi-GPU context (csfs_b200_create_multi / _rank / _emulated) is rank 0 of a group:
// it holds an NCCL communicator (rank mode: this process's only rank; multi mode: one
// communicator per device from ncclCommInitAll, the peer contexts owned here), and the
// csfmm entry points run the target-partitioned evaluation of partition.cu on it.
#pragma once

#include <nccl.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/csfs_b200.h"
#include "engine.hpp"

struct csfs_b200_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t aux = nullptr;  // the upward pass, overlapped with the dual traversal
    cudaStream_t hi = nullptr;   // the list phase (traversal, items, symmetric pairs): greatest priority
    cudaEvent_t w_copied = nullptr;  // host API: the weights' H2D copy (on aux) is done
    std::string err;
    csfs_b200::DeviceTree ttree, stree;
    bool shared = false;
    csfs_b200::Scratch sc;
    csfs_b200::Lists lists;
    csfs_b200::Items items;
    csfs_b200::DevBuf<double> phi_near;
    csfs_b200::DevBuf<int> counter;
    csfs_b200::DevBuf<double> h_txyz, h_sxyz, h_w, h_out;  // staging for the host-pointer API
    // pinned bounce buffers of the host-pointer API for PAGEABLE caller memory (capi.cu
    // h2d_staged / d2h_staged): allocated on first use, two so a copy overlaps the DMA
    void* stage_pin[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};  // the last DMA that used each buffer
    csfs_b200::DevBuf<double> d_soa;
    csfs_b200::DevBuf<int4> d_items;
    csfs_b200::DevBuf<int2> d_segs;
    csfs_b200::DevBuf<double2> log_tab;  // fastmath.cuh table, uploaded once per context
    csfs_b200::DevBuf<double> bve;       // RK4 stage buffers (csfs_b200_bve_step)
    csfs_b200::DevBuf<int> rm_i;         // remesh buckets (csfs_b200_bve_remesh)
    csfs_b200::DevBuf<double> rm_d, rm_h;
    cudaEvent_t ev[12] = {};
    csfs_b200::Cheb cheb{};
    csfs_b200::KernelSpec kspec;
    csfs_b200::FmmConfig cfg;
    bool have_state = false;
    bool have_src_tree = false;  // the last call was cstc: only the source tree exists
    bool have_tree = false;      // the last call was csfs_b200_tree_build: only ttree exists
    // trees uploaded by the stepwise API: reference id of every internal cluster (target,
    // source); empty = trees built here (ids reconstructed by reference_ids)
    std::vector<int> ref_of[2];
    int dim = 1;
    bool use_mutual = true;  // symmetric PP/CC evaluation (CSFS_B200_NO_SYMMETRIC=1 disables)
    bool mutual_unit_scope = false;  // CSFS_B200_MUTUAL_SCOPE=unit: single-GPU pairs like the partitioned path
    // partition state (csfs_b200_part_* and the partitioned csfmm)
    bool part_planned = false;
    cudaStream_t part_stream = nullptr;
    csfs_b200::DevBuf<double> phi_tree;
    std::vector<long long> unit_b[2], unit_e[2];
    std::vector<double> unit_cost[2];

    // ---- multi-GPU group (partition.cu) ----------------------------------------------
    enum class Mode { Single, Rank, Multi, Emulated };
    Mode mode = Mode::Single;
    int nranks = 1, rank = 0;
    ncclComm_t comm = nullptr;
    std::vector<std::unique_ptr<csfs_b200_ctx>> peers;  // ranks 1..n-1 (Multi / Emulated)
    csfs_b200::DevBuf<double> xq;      // proxy-weight exchange buffer, owner-packed
    csfs_b200::DevBuf<int> xidx;       // source clusters in exchange order (rank by rank)
    csfs_b200::DevBuf<unsigned long long> xcount;  // executed evaluations of the owned items
    csfs_b200::DevBuf<long long> ubeg;             // partition units' first particles (device)
    csfs_b200::DevBuf<unsigned long long> ucost;   // per unit: pair evaluations of its items
    std::vector<long long> xq_off;     // per rank: first cluster of its segment in xidx (+ end)
    std::vector<long long> t_range, s_range;  // per rank: owned tree-order [b, e) x 2
    double t_exchange = 0.0;           // last call: seconds in the two exchanges (rank 0)
    // last call, per rank of this process: plan, upward + pack, interact, downward, finish (ms)
    // and the bytes the rank broadcasts in the two exchanges
    std::vector<double> rank_phases;
};

namespace csfs_b200 {

// NCCL failures map onto CSFS_B200_NCCL_ERROR (3).
struct NcclFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
inline void nccl_check(ncclResult_t r, const char* what, const char* file, int line) {
    if (r == ncclSuccess) return;
    throw NcclFailure(std::string(what) + " failed at " + file + ":" + std::to_string(line) + ": " +
                      ncclGetErrorString(r));
}
#define CSFS_NCCL(x) ::csfs_b200::nccl_check((x), #x, __FILE__, __LINE__)

namespace capi {

// Runs f with the context's device current; maps the engine's exceptions onto the return
// codes of csfs_b200.h and stores the message for csfs_b200_last_error.
int guarded_call(csfs_b200_ctx* c, void (*f)(void*), void* arg);
template <class F>
int guarded(csfs_b200_ctx* c, F&& f) {
    return guarded_call(c, [](void* a) { (*static_cast<F*>(a))(); }, &f);
}
// Re-raises a nested entry point's return code as the matching exception.
void rethrow(csfs_b200_ctx* c, int rc);

KernelSpec to_spec(const csfs_b200_kernel* k);
FmmConfig to_cfg(const csfs_b200_config* c);
// Validation in the reference's order (interpolation.cpp:15, cluster_tree.cpp:32-33).
void validate(const FmmConfig& f, size_t nt, size_t ns);
Cheb make_cheb(int degree);
float ev_ms(cudaEvent_t a, cudaEvent_t b);
int count_internal(const DeviceTree& t);
// Fresh single-device context on `device` (streams, events, log table); throws.
std::unique_ptr<csfs_b200_ctx> new_context(int device);
void free_context(csfs_b200_ctx* c);

// One whole csfmm_sum on ONE device (device pointers, out in input order).
void run_csfmm(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw, size_t ns,
               const KernelSpec& ks, const FmmConfig& f, double* out, csfs_b200_stats* st, cudaStream_t s,
               cudaEvent_t w_ready = nullptr);
// The partition plan of one rank (full trees, lists, items with unit-scope symmetric
// pairs, partition units and their costs) — csfs_b200_part_plan.
// early_upward (the group rank program): the rank's source split (by particle count) is
// known once the trees are built, so its upward pass starts then on the aux stream, under
// the traversal; c->ev[11] marks its end and c->s_range holds every rank's sources.
void part_plan(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw, size_t ns,
               const KernelSpec& ks, const FmmConfig& f, cudaStream_t s, bool early_upward = false);
void fill_stats(csfs_b200_ctx* c, csfs_b200_stats* st);

}  // namespace capi

// partition.cu: csfmm over every rank of c's group (c = rank 0 in Multi / Emulated mode,
// this process's rank in Rank mode).  Device pointers on c's device; out complete on
// c's device (and, in Rank mode, on every rank's).
void run_csfmm_group(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw,
                     size_t ns, const KernelSpec& ks, const FmmConfig& f, double* out, csfs_b200_stats* st,
                     cudaStream_t s, cudaEvent_t w_ready = nullptr);
// Contiguous split of `costs` (units in tree order) into `world` runs of about equal
// cost (distributed.py split_contiguous restated): the cut k sits at the unit boundary
// whose prefix cost is closest to k*total/world, never moving backwards.
std::vector<std::pair<int, int>> split_contiguous(const std::vector<double>& costs, int world);
// partition.cu: exchange order of the owned source clusters (needs c->s_range)
void exchange_order(csfs_b200_ctx* c, const DeviceTree& S, cudaStream_t s);

}  // namespace csfs_b200
