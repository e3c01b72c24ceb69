/*
 * csfs_b200 — C-ABI of the B200-native (sm_100a) cubed-sphere FMM.
 *
 * Drop-in boundary for the reference library's summation engine
 * (/root/reference/proj/include/csfs/summation.hpp).  Plain pointers and sizes only;
 * positions are AoS x,y,z doubles exactly as std::vector<csfs::Vec3>::data() lays them
 * out, weights/outputs are in INPUT order like the reference's ParticleSet /
 * PotentialField (summation.hpp:34-41).  The C++ shim (paper_2508_13550_b200/host/
 * csfs_b200_shim.cpp) re-exposes the reference's csfs:: signatures on top of these entry
 * points and rethrows std::invalid_argument on code 1 with the reference's messages.
 *
 * Return codes: 0 ok, 1 invalid argument (reference's std::invalid_argument),
 * 2 CUDA error, 3 NCCL/collective error, 4 device out of memory.
 * One context per host thread; a context owns its device(s), streams, buffers and NCCL
 * communicators; calls on one context are serialized by the caller.
 */
#ifndef CSFS_B200_H
#define CSFS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CSFS_B200_API __attribute__((visibility("default")))
#else
#define CSFS_B200_API
#endif

#define CSFS_B200_OK 0
#define CSFS_B200_INVALID_ARGUMENT 1
#define CSFS_B200_CUDA_ERROR 2
#define CSFS_B200_NCCL_ERROR 3
#define CSFS_B200_OUT_OF_MEMORY 4

typedef struct csfs_b200_ctx csfs_b200_ctx;

/* csfs::Kernel (kernels.hpp:32-49): kind in KernelKind order
 * 0 laplace, 1 biharmonic, 2 biot_savart (out_dim 3), 3 sal; SalParams defaults
 * a1=-2.7, b0=-6.21196, b1=6.1, rho_ratio=1025/5517 (kernels.hpp:18-23). */
typedef struct {
    int kind;
    double a1, b0, b1, rho_ratio;
} csfs_b200_kernel;

/* csfs::TraversalConfig (summation.hpp:22-31) minus method/threads:
 * n0 < 0 selects 4*degree^2 (resolved_n0). */
typedef struct {
    double mac;
    int degree;
    int n0;
    int shrink;
} csfs_b200_config;

/* csfs::SumStats (summation.hpp:44-53) plus B200 extras. Times in seconds, measured
 * with CUDA events on the context stream. t_traversal = lists + PP/PC/CP/CC, as in the
 * reference's csfmm_sum (summation.cpp:397-402). */
typedef struct {
    double t_tree_build, t_upward, t_traversal, t_downward, t_total;
    uint64_t pp, pc, cp, cc;
    int src_depth, src_clusters, src_leaves;
    int tgt_depth, tgt_clusters, tgt_leaves;
    double t_lists, t_interact;                  /* sub-phases of t_traversal */
    uint64_t evals_pp, evals_pc, evals_cp, evals_cc; /* pairwise kernel evaluations */
    int shared_tree;                             /* targets == sources: one tree built */
    uint64_t evals_executed;  /* kernel evaluations actually performed (symmetric PP/CC pairs once) */
    int symmetric_pairs;      /* PP leaf / CC cluster pairs evaluated once for both directions */
    int n_ranks;              /* ranks that evaluated the call (1: one GPU) */
    double t_exchange;        /* seconds in the two NCCL all-gathers (rank 0; 0 on one GPU) */
    int traversal_fallback;   /* 1: a host-free traversal sweep overflowed its buffers and the
                                 synchronous sweep loop re-ran it (the buffers then stay grown) */
    uint64_t symmetric_partials; /* doubles in the symmetric pairs' partial-sum buffer (64-bit offsets) */
} csfs_b200_stats;

/* --- lifetime ------------------------------------------------------------------------ */
/* One device.  (SURVEY.md §8b's csfs_b200_create(ctx, num_gpus, device_ids) is
 * csfs_b200_create_multi below; this single-device form is its num_gpus = 1 case.) */
CSFS_B200_API int csfs_b200_create(csfs_b200_ctx** out, int device);
CSFS_B200_API void csfs_b200_destroy(csfs_b200_ctx* ctx);
/* Message of the last failing call on this context ("" if none). */
CSFS_B200_API const char* csfs_b200_last_error(const csfs_b200_ctx* ctx);

/* --- the hot path ---------------------------------------------------------------------
 * csfs::csfmm_sum (summation.hpp:81-83, summation.cpp:383-421).  HOST pointers:
 * tgt_xyz nt x 3, src_xyz ns x 3, src_w ns, out nt x out_dim (overwritten).
 * stats may be NULL.  Synchronous. */
CSFS_B200_API int csfs_b200_csfmm(csfs_b200_ctx* ctx, const double* tgt_xyz, size_t nt, const double* src_xyz,
                    const double* src_w, size_t ns, const csfs_b200_kernel* kernel,
                    const csfs_b200_config* config, double* out, csfs_b200_stats* stats);

/* Same, DEVICE pointers (on the context's device), work ordered on `stream`
 * (cudaStream_t; NULL = CUDA's legacy default stream).  Returns after the result is in
 * `out` (the engine synchronizes on tree/list sizes). */
CSFS_B200_API int csfs_b200_csfmm_device(csfs_b200_ctx* ctx, const double* tgt_xyz, size_t nt,
                           const double* src_xyz, const double* src_w, size_t ns,
                           const csfs_b200_kernel* kernel, const csfs_b200_config* config,
                           double* out, csfs_b200_stats* stats, void* stream);

/* csfs::cstc_sum (summation.hpp:77-79, summation.cpp:308-381): the cubed-sphere
 * treecode — per-target traversal of the source tree, point-cluster MAC, PC via proxies
 * and PP direct; stats->pp / pc count the per-target interactions like the reference. */
CSFS_B200_API int csfs_b200_cstc(csfs_b200_ctx* ctx, const double* tgt_xyz, size_t nt,
                                 const double* src_xyz, const double* src_w, size_t ns,
                                 const csfs_b200_kernel* kernel, const csfs_b200_config* config,
                                 double* out, csfs_b200_stats* stats);
CSFS_B200_API int csfs_b200_cstc_device(csfs_b200_ctx* ctx, const double* tgt_xyz, size_t nt,
                                        const double* src_xyz, const double* src_w, size_t ns,
                                        const csfs_b200_kernel* kernel, const csfs_b200_config* config,
                                        double* out, csfs_b200_stats* stats, void* stream);

/* csfs::direct_sum (summation.hpp:74-75, summation.cpp:136-161): O(nt*ns) all pairs. */
CSFS_B200_API int csfs_b200_direct(csfs_b200_ctx* ctx, const double* tgt_xyz, size_t nt, const double* src_xyz,
                     const double* src_w, size_t ns, const csfs_b200_kernel* kernel, double* out);
CSFS_B200_API int csfs_b200_direct_device(csfs_b200_ctx* ctx, const double* tgt_xyz, size_t nt,
                            const double* src_xyz, const double* src_w, size_t ns,
                            const csfs_b200_kernel* kernel, double* out, void* stream);

/* --- barotropic vorticity: one RK4 step (applications.cpp:378-412, remesh off) -------------
 * Four Biot-Savart CSFMM sums with device-resident stage positions: k_i = u(pos_i, zeta_i),
 * pos = normalized(x + h k), zeta_i = zeta - 2 Omega h k.z; then x <- normalized(x + du),
 * zeta -= 2 Omega du.z, du = dt/6 (k1 + 2k2 + 2k3 + k4).  xyz (n x 3) and zeta (n) are
 * updated in place; areas (n) frozen.  stage_stats: NULL or 4 entries.  dt <= 0 -> code 1
 * "time step must be positive" (the reference's std::invalid_argument). */
CSFS_B200_API int csfs_b200_bve_step(csfs_b200_ctx* ctx, double* xyz, double* zeta, const double* areas,
                                     size_t n, double omega, double dt, const csfs_b200_config* config,
                                     csfs_b200_stats* stage_stats);
CSFS_B200_API int csfs_b200_bve_step_device(csfs_b200_ctx* ctx, double* xyz, double* zeta,
                                            const double* areas, size_t n, double omega, double dt,
                                            const csfs_b200_config* config, csfs_b200_stats* stage_stats,
                                            void* stream);

/* --- barotropic vorticity: remesh (applications.hpp:91-94, applications.cpp:329-371) ------
 * bve_remesh(state, neighbors): for every grid centre g_i, the k = min(max(neighbors, 6), n)
 * nearest particles (lat-lon buckets, rings until >= k candidates then one more ring;
 * ties by index), a Gaussian-weighted least-squares quadratic in g_i's face-local
 * (xi, eta) over the usable ones (face_plane_coords), evaluated at g_i; fewer than 6
 * usable neighbours -> the nearest particle's value.  Then xyz <- grid_xyz and zeta
 * (n) / tracer (n, NULL: no tracer) <- the fitted values.  The reference's bve_step calls
 * it after the RK4 update when BveStepOptions::remesh (default true, 12 neighbours).
 * neighbors > 64 -> code 1 (a device-side limit of this library). */
CSFS_B200_API int csfs_b200_bve_remesh(csfs_b200_ctx* ctx, double* xyz, double* zeta, double* tracer,
                                       const double* grid_xyz, size_t n, int neighbors);
CSFS_B200_API int csfs_b200_bve_remesh_device(csfs_b200_ctx* ctx, double* xyz, double* zeta, double* tracer,
                                              const double* grid_xyz, size_t n, int neighbors, void* stream);

/* --- stepwise state of the LAST csfmm call (parity / inspection) ------------------------
 * which: 0 target tree, 1 source tree.  Cluster ids are the REFERENCE's ids
 * (LIFO expansion order, cluster_tree.cpp:87-140). */
CSFS_B200_API int csfs_b200_tree_info(const csfs_b200_ctx* ctx, int which, int* n_clusters, int* depth,
                        size_t* n_particles, int* n_proxy_per_cluster);
/* perm: n (tree order -> input index); ints: ncl x 10 = face, begin, end, parent, depth,
 * child_count, children[4]; dbls: ncl x 8 = xi0, xi1, eta0, eta1, cx, cy, cz, radius;
 * proxy: ncl x (p+1)^2 x 3.  Any pointer may be NULL. */
CSFS_B200_API int csfs_b200_tree_export(csfs_b200_ctx* ctx, int which, int* perm, int* ints, double* dbls,
                          double* proxy);
/* counts[4] = |pp|,|pc|,|cp|,|cc|; lists as (t, s) int pairs in reference ids, sorted. */
CSFS_B200_API int csfs_b200_lists_export(csfs_b200_ctx* ctx, long long* counts, int* pp, int* pc, int* cp,
                           int* cc);
/* Source-tree proxy weights after the upward pass, ncl x (p+1)^2, reference id order. */
CSFS_B200_API int csfs_b200_proxy_weights_export(csfs_b200_ctx* ctx, double* pw);

/* --- the stepwise API: the pieces of csfmm_sum on trees the CALLER holds -------------------
 * The reference exposes its pipeline piece by piece (cluster_tree.hpp:52-81,
 * summation.hpp:66-102) and its tests drive the pieces on trees they modify in between
 * (acceptance.cpp:229-280).  A caller's tree — the reference's ClusterTree — is handed
 * over as plain arrays in REFERENCE cluster ids (exactly what csfs_b200_tree_export /
 * _tree_particles return for a tree this library built); every call uploads what it reads.
 * The C++ shim (host/csfs_b200_shim.cpp) marshals csfs::ClusterTree into this form. */
typedef struct {
    size_t n;              /* particles */
    int n_clusters;        /* clusters 0..5 are the face roots */
    int degree;            /* interpolation degree (proxy grid (degree+1)^2) */
    const int* perm;       /* n: tree order -> input index (ClusterTree::perm) */
    const double* xyz;     /* n x 3: positions in tree order (ClusterTree::points) */
    const double* xi;      /* n: face coordinates in tree order (ClusterTree::xi / eta) */
    const double* eta;
    const int* ints;       /* n_clusters x 10: face, begin, end, parent, depth, child_count,
                              children[4] (-1 padded) — the layout of csfs_b200_tree_export */
    const double* dbls;    /* n_clusters x 8: xi0, xi1, eta0, eta1 (bounds), cx, cy, cz, radius */
    const double* proxy;   /* n_clusters x (degree+1)^2 x 3: CellInterpolant::proxy_points */
} csfs_b200_tree_desc;

/* ClusterTree(particles, degree, n0, shrink) (cluster_tree.cpp:29-147) on the device;
 * afterwards csfs_b200_tree_info / _tree_export / _tree_particles with which = 0 return
 * it (reference ids).  The reference's std::invalid_argument messages as code 1. */
CSFS_B200_API int csfs_b200_tree_build(csfs_b200_ctx* ctx, const double* xyz, size_t n, int degree, int n0,
                                       int shrink, int* n_clusters, int* depth);
/* Tree-order positions (n x 3), xi and eta (n each) of a tree: which 0 target / 1 source
 * of the last call (or the tree_build tree).  Any pointer may be NULL. */
CSFS_B200_API int csfs_b200_tree_particles(csfs_b200_ctx* ctx, int which, double* xyz, double* xi, double* eta);
/* upward_pass(tree, weights) (cluster_tree.cpp:163-220): w in input order; pw receives
 * n_clusters x (degree+1)^2 proxy weights in reference ids. */
CSFS_B200_API int csfs_b200_upward_tree(csfs_b200_ctx* ctx, const csfs_b200_tree_desc* tree, const double* w,
                                        double* pw);
/* downward_pass(tree, out_dim, out) (cluster_tree.cpp:228-283): qphi (n_clusters x
 * (degree+1)^2 x dim, reference ids) is pushed parents -> children IN PLACE (like the
 * reference's tree) and interpolated to the particles, ADDED into out (n x dim, input
 * order). */
CSFS_B200_API int csfs_b200_downward_tree(csfs_b200_ctx* ctx, const csfs_b200_tree_desc* tree, int dim,
                                          double* qphi, double* out);
/* dual_tree_traversal(targets, sources, mac, n0) (summation.cpp:163-203): counts[4] =
 * |pp|,|pc|,|cp|,|cc|; then csfs_b200_lists_export returns the (t, s) sets in reference
 * ids, sorted (the reference emits them in its LIFO visiting order; the sets are equal). */
CSFS_B200_API int csfs_b200_traversal_tree(csfs_b200_ctx* ctx, const csfs_b200_tree_desc* targets,
                                           const csfs_b200_tree_desc* sources, double mac, int n0,
                                           long long* counts);
/* evaluate_pp / evaluate_pc / accumulate_cp_cc (summation.cpp:205-306) for the given
 * lists ((t, s) int pairs, reference ids; any count may be 0): PP and PC results are ADDED
 * into out (targets' n x dim, input order), CP and CC into qphi (targets' n_clusters x
 * (degree+1)^2 x dim).  w: sources' weights, input order (PP, CP); src_pw: sources' proxy
 * weights (n_clusters x (degree+1)^2, PC, CC).  Each target sums its list entries in the
 * (type, source id) order. */
CSFS_B200_API int csfs_b200_evaluate_tree(csfs_b200_ctx* ctx, const csfs_b200_tree_desc* targets,
                                          const csfs_b200_tree_desc* sources, const double* w, const double* src_pw,
                                          const csfs_b200_kernel* kernel, const int* pp, long long n_pp,
                                          const int* pc, long long n_pc, const int* cp, long long n_cp,
                                          const int* cc, long long n_cc, double* out, double* qphi);

/* --- multi-GPU contexts: csfs_b200_csfmm / _csfmm_device / _bve_step on them run the
 * target-partitioned CSFMM over every rank of the group, with the proxy-weight and
 * potential exchanges as NCCL all-gathers over NVLink (partition.cu).  Results are bitwise
 * identical for every rank count (and to the single-GPU engine up to the symmetric-pair
 * scope: pairs never straddle two depth-1 subtrees, so they equal a one-GPU run with
 * CSFS_B200_MUTUAL_SCOPE=unit bit for bit).  Other entry points run on rank 0's device.
 * Calls on a group are collective: every rank of a Rank group makes the same call.
 *
 *   _create_multi     ONE process drives num_gpus devices (device_ids NULL = 0..num_gpus-1,
 *                     distinct): ncclCommInitAll, one host thread + stream per device,
 *                     rank 0 = device_ids[0] is the context's device; device pointers
 *                     passed to it are on that device and the inputs are broadcast to
 *                     the others over NVLink.
 *   _create_rank      one process per GPU (e.g. torchrun): rank `rank` of `nranks`, NCCL
 *                     from the CSFS_B200_NCCL_ID_BYTES unique id rank 0 made with
 *                     csfs_b200_nccl_unique_id and shipped to the others; every rank passes
 *                     the full inputs and receives the full result.
 *   _create_emulated  nranks ranks on ONE device, run phase by phase with device copies in
 *                     place of NCCL: the partition and exchange layout, bitwise, on one
 *                     GPU (tests / per-rank cost measurement; not a speed-up).
 * A failing NCCL call returns CSFS_B200_NCCL_ERROR (3).  In a multi-device group a rank
 * that fails aborts every communicator so no rank is left waiting in an all-gather; the
 * group then returns errors until it is destroyed. */
#define CSFS_B200_NCCL_ID_BYTES 128
CSFS_B200_API int csfs_b200_create_multi(csfs_b200_ctx** out, int num_gpus, const int* device_ids);
CSFS_B200_API int csfs_b200_nccl_unique_id(unsigned char* id);
CSFS_B200_API int csfs_b200_create_rank(csfs_b200_ctx** out, int device, int nranks, int rank,
                                        const unsigned char* id);
CSFS_B200_API int csfs_b200_create_emulated(csfs_b200_ctx** out, int device, int nranks);
/* nranks / this rank / the devices of the group (nranks entries; Multi, Emulated: all,
 * Rank: this process's) and, after a partitioned call, the owned tree-order target and
 * source ranges of every rank (2 x nranks: begin, end).  Any pointer may be NULL. */
CSFS_B200_API int csfs_b200_group_info(const csfs_b200_ctx* ctx, int* nranks, int* rank, int* devices,
                                       long long* t_ranges, long long* s_ranges);

/* Per-rank phases of the last partitioned call with stats, for the ranks this process
 * runs (Multi / Emulated: all, in rank order; Rank: this one): 6 values each — plan,
 * upward + pack, interact, downward, finish (ms, CUDA events on the rank's stream) and the
 * bytes the rank broadcasts in the two all-gathers.  *n = values available; min(cap, *n)
 * are written.  In Emulated mode the phases ran alone on the device, so they are the
 * per-rank cost of an N-GPU step without the exchanges (tools/scaling_emulation.py). */
CSFS_B200_API int csfs_b200_group_phases(const csfs_b200_ctx* ctx, double* out, int cap, int* n);

/* TreeStats::leaf_size_histogram (cluster_tree.cpp:149-161) of the last call's target
 * (which 0) or source (1) tree: bucket i counts the leaves with i particles (empty face
 * roots included).  *len = max leaf size + 1; min(cap, *len) buckets are written. */
CSFS_B200_API int csfs_b200_leaf_histogram(csfs_b200_ctx* ctx, int which, int* hist, int cap, int* len);

/* --- multi-GPU building blocks: target partitioning with a caller-owned collective ----
 * The library is collective-agnostic: the CALLER owns two device buffers (sizes from
 * part_sizes) and all-reduces (sum) them between the phases (torch.distributed / NCCL
 * over NVLink in paper_2508_13550_b200/distributed.py).  Every rank, on `stream`:
 *   1. part_plan     full trees, dual traversal and work items (redundant, cheap);
 *   2. part_units    the partition units (depth-1 subtrees + unsplit roots, tree order)
 *                    with particle ranges and cost; the caller splits them into one
 *                    contiguous particle range per rank (targets: by cost, sources: count);
 *   3. part_upward   writes the owned source subtrees' proxy weights into pw, zeros
 *                    elsewhere              -> caller: all_reduce(sum, pw)
 *   4. part_eval     takes the reduced pw, computes the depth-0 proxy weights
 *                    (redundantly), the owned targets' PP/PC/CP/CC and downward pass into
 *                    the TREE-ORDER field phi, zeros elsewhere
 *                                           -> caller: all_reduce(sum, phi)
 *   5. part_finish   out[perm[t]] = phi_reduced[t] (device out, input order).
 * Each target is evaluated by exactly one rank in the single-GPU order and every reduced
 * slot has one non-zero term, so the result is bitwise identical to
 * csfs_b200_csfmm_device for any rank count. */
CSFS_B200_API int csfs_b200_part_plan(csfs_b200_ctx* ctx, const double* tgt_xyz, size_t nt,
                                      const double* src_xyz, const double* src_w, size_t ns,
                                      const csfs_b200_kernel* kernel,
                                      const csfs_b200_config* config, void* stream);
CSFS_B200_API int csfs_b200_part_units(csfs_b200_ctx* ctx, int which, int* n_units,
                                       long long* begin, long long* end, double* cost);
CSFS_B200_API int csfs_b200_part_sizes(csfs_b200_ctx* ctx, size_t* n_pw, size_t* n_phi);
CSFS_B200_API int csfs_b200_part_upward(csfs_b200_ctx* ctx, long long src_begin,
                                        long long src_end, double* pw);
CSFS_B200_API int csfs_b200_part_eval(csfs_b200_ctx* ctx, long long tgt_begin, long long tgt_end,
                                      const double* pw_reduced, double* phi);
CSFS_B200_API int csfs_b200_part_finish(csfs_b200_ctx* ctx, const double* phi_reduced,
                                        double* out);

/* --- diagnostics ------------------------------------------------------------------------ */
/* Number of engine kernels launched by this process so far (all contexts). */
CSFS_B200_API uint64_t csfs_b200_kernel_launches(void);
/* The device kernel functor on n (x_i, y_i) pairs (host arrays, n x 3 each): the
 * reference's guarded per-pair value K(x_i, y_i) (0 where the coincidence guard skips),
 * out n x out_dim — Kernel::try_eval (kernels.cpp) known-answer checks on the GPU path. */
CSFS_B200_API int csfs_b200_eval_pairs(csfs_b200_ctx* ctx, const csfs_b200_kernel* kernel,
                                       const double* x, const double* y, size_t n, double* out);
/* The device elementary functions on n host values: fn 0 log, 1 rsqrt, 2 rcp, 3 dilog. */
CSFS_B200_API int csfs_b200_eval_math(csfs_b200_ctx* ctx, int fn, const double* x, size_t n,
                                      double* out);
/* Measured FP64 FMA-pipe peak of the context's device in TFLOP/s (DFMA = 2 flops). */
CSFS_B200_API int csfs_b200_probe_fp64(csfs_b200_ctx* ctx, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* CSFS_B200_H */
