// Host-side engine structures of the B200 CSFMM: device buffers, the device-resident
// cluster tree (the GPU analogue of csfs::ClusterTree, cluster_tree.hpp:52-67), the
// interaction lists (summation.hpp:55-59) and the work items the evaluation kernel
// consumes.  One Engine per csfs_b200_ctx; one device per Engine.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "common.cuh"

namespace csfs_b200 {

// Grow-only device buffer.  grow() discards contents, grow_keep() preserves them.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void grow(size_t n) {
        if (n <= cap) return;
        if (p) CSFS_CK(cudaFree(p));
        p = nullptr;
        const size_t c = n + n / 4 + 64;
        CSFS_CK(cudaMalloc(&p, c * sizeof(T)));
        cap = c;
    }
    void grow_keep(size_t n, size_t used, cudaStream_t s) {
        if (n <= cap) return;
        const size_t c = n + n / 2 + 64;
        T* q = nullptr;
        CSFS_CK(cudaMalloc(&q, c * sizeof(T)));
        if (p && used) CSFS_CK(cudaMemcpyAsync(q, p, used * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (p) {
            CSFS_CK(cudaStreamSynchronize(s));
            CSFS_CK(cudaFree(p));
        }
        p = q;
        cap = c;
    }
    operator T*() const { return p; }
};

// Source segments / symmetric-pair lengths carry flags next to the length: the sign
// (negative = proxy points), bit 30 of the magnitude (the coincidence guard is needed
// for this entry; kernels_dev.cuh eval<G>) and bit 29 (the fused 1 - x.y is safe, eval<.., F>).
constexpr int kSegGuard = 1 << 30;
// bit 29: the entry's point sets are more than kFuseGap and less than kFuseMaxDist apart — the
// fused 1 - x.y may be used, and x.y > 0 for every pair
constexpr int kSegFused = 1 << 29;
constexpr double kFuseGap = 4.48e-3;  // chordal; 1 - x.y >= kFuseGap^2 / 2 >= 1.0e-5
constexpr double kFuseMaxDist = 1.41;  // chordal; x.y >= 1 - kFuseMaxDist^2 / 2 = 5.9e-3: one hemisphere
__host__ __device__ __forceinline__ int seg_len(int y) { return (y < 0 ? -y : y) & (kSegFused - 1); }
__host__ __device__ __forceinline__ bool seg_guard(int y) { return ((y < 0 ? -y : y) & kSegGuard) != 0; }
__host__ __device__ __forceinline__ bool seg_fused(int y) { return ((y < 0 ? -y : y) & kSegFused) != 0; }

// Raw-pointer view of a tree, passed by value into kernels.
struct TreeView {
    long long n;
    int np, npp;
    // particles, tree order
    const double *px, *py, *pz, *xi, *eta, *w;
    const int *perm, *node;
    // clusters (internal, level-major ids)
    const int *face, *depth, *begin, *end, *parent, *nchild;
    const int4* child;
    const double *xi0, *xi1, *eta0, *eta1, *cx, *cy, *cz, *rad;
    // proxies: cluster c owns [c*npp, (c+1)*npp), index k1*np+k2 (interpolation.cpp:64-67)
    const double *qx, *qy, *qz;
    const double* qrad;  // per cluster: max chordal distance from the centre to its proxy points
    const int* off_sphere;  // device flag: some particle is not a unit vector (guard everything)
};

struct DeviceTree {
    long long n = 0;
    int degree = 0, np = 0, npp = 0, n0 = 0;
    bool shrink = true, has_w = false;
    // particles (tree order) + one scratch copy for the partition scatters
    DevBuf<double> px, py, pz, xi, eta, w;
    DevBuf<int> perm, node;
    DevBuf<double> px2, py2, pz2, xi2, eta2, w2;
    DevBuf<int> perm2, node2, rank;
    // clusters
    int ncl = 0, cap = 0;
    DevBuf<int> face, depth, begin, end, parent, nchild;
    DevBuf<int4> child;
    DevBuf<double> xi0, xi1, eta0, eta1, cx, cy, cz, rad;
    DevBuf<unsigned char> split;
    DevBuf<unsigned long long> bnd;  // 4 per cluster: min xi, max xi, min eta, max eta (ordered)
    DevBuf<double2> mid;             // per cluster: the split point (midpoint of the shrunk bounds)
    std::vector<int> level_first, level_count;
    std::vector<int> root_count;  // 6
    // proxies
    DevBuf<double> qx, qy, qz, qrad;
    DevBuf<double> qw;    // proxy weights (source side), ncl*npp
    DevBuf<int> off_sphere;  // 1 flag: a particle with | |x|^2 - 1 | > 1e-12 (tree.cu k_face)
    DevBuf<double> qphi;  // proxy potentials (target side), ncl*npp*dim

    void reserve_clusters(int n_needed, cudaStream_t s);
    TreeView view() const;
    int depth_max() const { return int(level_first.size()) - 1; }
};

// Scratch shared by the build / traversal phases.
struct Scratch {
    DevBuf<int> tiles;      // scan tile totals
    DevBuf<int> grand;      // scan grand totals (device)
    DevBuf<long long> tiles64, grand64;  // the same for 64-bit counters (partial offsets)
    DevBuf<int> segP, segE, kid, koff;  // per frontier cluster x 4
    DevBuf<unsigned long long> qbnd;    // per frontier cluster x 16: quadrant bounds (local levels)
    DevBuf<int> counters;   // misc device counters
    int* host = nullptr;    // pinned host mirror for small read-backs
    DevBuf<double> fxi, feta;  // level-0 face coordinates in input order
    DevBuf<int> fface;
    // label-then-sort build (tree.cu): per-particle labels / leaves / sort keys and radix
    // scratch (input order); per (cluster, quadrant) child ids, counts and bounds; level
    // descriptors {first, cnt, nsplit, overflow}
    DevBuf<int> lab, leaf, key, kb, vb, sorted, hist, qchild, scnt, cbase;
    DevBuf<unsigned long long> sbnd;
    DevBuf<int4> lev;
    DevBuf<int> rcnt;
    int qcap = 0;  // clusters the per-quadrant arrays hold
};
// sc.host layout (pinned ints): [0, 64) small read-backs, [kHostLev, +4 * kMaxDepth + 16)
// level descriptors, [kHostRoots, +6) root counts
constexpr int kHostLev = 256;
constexpr int kHostRoots = 768;
constexpr int kHostInts = 1024;

// Interaction lists in internal cluster ids, (t, s) pairs, canonical after build.
struct Lists {
    DevBuf<int2> l[4];  // pp, pc, cp, cc
    long long n[4] = {0, 0, 0, 0};
    DevBuf<int2> front, front2;
    DevBuf<int> cnt;  // sweep counters of the host-free traversal
    bool fallback = false;  // the last traversal overflowed a buffer and re-ran synchronously
};

// Work items for the unified evaluation kernel: one item per target leaf (PP+PC
// sources, targets = leaf particles) and one per target cluster (CP+CC sources,
// targets = its proxy points).  seg = {start, len}; len < 0 marks a proxy segment.
struct Items {
    DevBuf<int> cnt, off, cur;  // per key (2*ncl_t)
    DevBuf<int> keys;           // non-empty keys, in key order
    DevBuf<long long> code;     // per entry sort code
    DevBuf<int2> seg;           // per entry source segment
    DevBuf<int4> item;          // {tgt_start, tgt_len (neg = proxy), seg_begin, seg_end}
    DevBuf<int> anchor;         // owner key: first target particle, -1 = every rank
    DevBuf<double> cost;        // pair evaluations of the item
    DevBuf<unsigned long long> pairs;  // 4 pair-eval counters (pp, pc, cp, cc)
    int n_items = 0;
    long long n_entries = 0;
    unsigned long long pair_evals[4] = {0, 0, 0, 0};
    // symmetric PP/CC pairs (build_mutual): per entry flag/pair keys; per symmetric pair its
    // {A begin, |A|, B begin, |B|}, partial offset (A block, then B block), owner anchor;
    // per leaf the partial blocks k_mutual_reduce adds to it (sorted)
    DevBuf<int> mflag, manchor, mcnt, moff, mcur;
    DevBuf<int2> epair, mleaf;
    DevBuf<int4> mpair;
    DevBuf<long long> mpoff, mlist, unit_b;
    DevBuf<double> partial;
    DevBuf<int> oitem, opair, ocnt, otiles;  // a rank's own items / pairs (interact.cu compact_owned)
    // ordering the items by cost (traverse.cu order_items_by_cost): sort scratch, permuted copies
    DevBuf<int> skey, skb, svb, sout, shist, stiles, sgrand, keys2, anchor2;
    DevBuf<int4> item2;
    DevBuf<double> cost2;
    int n_mutual = 0;
    long long n_partial = 0;  // doubles
    unsigned long long skipped_pairs = 0;
    bool mutual = false;
};

struct KernelSpec {
    int kind = 0;  // 0 laplace, 1 biharmonic, 2 biot_savart, 3 sal  (KernelKind order)
    double a1 = -2.7, b0 = -6.21196, b1 = 6.1, rho_ratio = 1025.0 / 5517.0;  // kernels.hpp:18-23
    int out_dim() const { return kind == 2 ? 3 : 1; }
};

struct FmmConfig {
    double mac = 0.7;
    int degree = 6;
    int n0 = -1;
    bool shrink = true;
    int resolved_n0() const { return n0 >= 0 ? n0 : 4 * degree * degree; }
};

struct PhaseTimes {
    double tree = 0, upward = 0, traversal = 0, lists = 0, interact = 0, downward = 0, total = 0;
};

// --- phase entry points (implemented in the .cu files) -------------------------------

// tree.cu: builds `tree` from AoS xyz (device, input order) and optional weights.
void build_tree(DeviceTree& tree, Scratch& sc, const double* xyz, const double* w, long long n,
                int degree, int n0, bool shrink, const Cheb& cheb, cudaStream_t s,
                cudaEvent_t w_ready = nullptr);
// qrad (max centre-to-proxy distance) of every cluster, for trees uploaded by the stepwise API.
void tree_proxy_radii(DeviceTree& t, cudaStream_t s);
// Device byte comparison (targets == sources detection).
bool device_equal(const void* a, const void* b, size_t bytes, Scratch& sc, cudaStream_t s);

// passes.cu
// Ownership window of one rank: clusters at depth >= 1 whose first particle lies in
// [b, e) (tree order).  The whole range is [0, n).
struct Own {
    long long b = 0, e = 0;
};
// mode: 0 all clusters; 1 owned clusters at depth >= 1 only (qw zeroed elsewhere);
//       2 depth-0 clusters only (after the proxy-weight allreduce)
void upward_pass(DeviceTree& src, const Cheb& cheb, cudaStream_t s, int mode = 0, Own own = {});
// out_perm = true: out[perm[t]] (input order); false: out[t] (tree order, owned leaves only).
void downward_pass(DeviceTree& tgt, const Cheb& cheb, int dim, const double* phi_near, double* out,
                   cudaStream_t s, Own own, bool out_perm);

// traverse.cu
void dual_traversal(const DeviceTree& tgt, const DeviceTree& src, double mac, int n0, Lists& lists,
                    Scratch& sc, cudaStream_t s);
// own_b >= 0: only items of targets whose first particle lies in [own_b, own_e), plus the
// depth-0 targets every rank evaluates (the group plan); own_b < 0: every target.
void build_items(const DeviceTree& tgt, const DeviceTree& src, const Lists& lists, Items& items,
                 Scratch& sc, cudaStream_t s, long long own_b = -1, long long own_e = -1);
// Symmetric PP marking (shared tree only); unit_begins = sorted first particles of the
// partition units (depth-1 subtrees + unsplit roots).
void build_mutual(const DeviceTree& tgt, Items& items, const std::vector<long long>& unit_begins, Scratch& sc,
                  cudaStream_t s);
// Partition units of a tree: (begin, end) particle ranges in tree order.
void partition_units(const DeviceTree& t, std::vector<long long>& b, std::vector<long long>& e, cudaStream_t s);
// Pair evaluations of the list entries of each target unit (ubeg: the units' first particles).
void list_unit_costs(const DeviceTree& tgt, const DeviceTree& src, const Lists& L, const long long* ubeg, int nu,
                     unsigned long long* ucost, cudaStream_t s);

// interact.cu
void interact(const KernelSpec& k, const DeviceTree& tgt, const DeviceTree& src, Items& items,
              double* phi_near, int* work_counter, const double2* log_tab, cudaStream_t s, Own own);
// all-pairs (direct_sum, summation.cpp:136-161): targets/sources AoS in input order.
void direct_allpairs(const KernelSpec& k, const double* txyz, long long nt, const double* sxyz,
                     const double* sw, long long ns, double* out, DevBuf<double>& soa,
                     DevBuf<int4>& items, DevBuf<int2>& segs, int* work_counter,
                     const double2* log_tab, cudaStream_t s);
// diagnostics: guarded scaled kernel values of (x_i, y_i) pairs; fastmath functions
// (fn 0 log, 1 rsqrt, 2 rcp, 3 dilog).
void eval_pairs(const KernelSpec& k, const double* x, const double* y, long long n, double* out,
                const double2* log_tab, cudaStream_t s);
void eval_math(int fn, const double* x, long long n, double* out, const double2* log_tab, cudaStream_t s);
void make_log_table(double2* tab);

// cstc.cu: the treecode (cstc_sum, summation.cpp:308-381) over a built + upward-passed
// source tree; order (nullable) = target processing order; counts[2] = n_pp, n_pc.
void cstc_eval(const KernelSpec& k, const double* txyz, long long nt, const int* order, const DeviceTree& src,
               double mac, int n0, const double2* log_tab, double* out, unsigned long long* counts,
               cudaStream_t s);

// remesh.cu: bve_remesh (applications.cpp:329-371) on the device; at most kRemeshMaxK
// neighbours per grid centre.  xyz <- grid, zeta/tracer (tracer may be null) <- the fits.
constexpr int kRemeshMaxK = 64;
void bve_remesh(double* xyz, double* zeta, double* tracer, const double* grid, long long n, int neighbors,
                DevBuf<int>& ibuf, DevBuf<double>& dbuf, cudaStream_t s);

// bve.cu: RK4 stage arithmetic of bve_step (applications.cpp:378-412)
void bve_weights(long long n, const double* zeta, const double* area, double* w, cudaStream_t s);
void bve_advance(long long n, const double* x0, const double* z0, const double* k, double h, double omega,
                 const double* area, double* pos, double* zeta, double* w, cudaStream_t s);
void bve_final(long long n, double* x, double* zeta, const double* k1, const double* k2, const double* k3,
               const double* k4, double dt, double omega, cudaStream_t s);

// passes.cu: out[perm[t]] = phi_tree[t] (multi-GPU finish).
void scatter_to_input(const DeviceTree& tgt, int dim, const double* phi_tree, double* out, cudaStream_t s);

// probe.cu: DFMA-chain FP64 peak (TFLOP/s) of the current device.
double probe_fp64_tflops(cudaStream_t s);

// reference cluster ids (LIFO expansion order, cluster_tree.cpp:87-140) for export.
std::vector<int> reference_ids(const std::vector<int>& parent, const std::vector<int>& depth,
                               const std::vector<int4>& child, const std::vector<int>& nchild);

}  // namespace csfs_b200
