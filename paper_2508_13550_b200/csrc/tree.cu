// GPU cluster-tree build: the B200 restatement of csfs::ClusterTree's constructor
// (/root/reference/proj/src/cluster_tree.cpp:29-147).
//
// The reference builds the quadtree serially with a LIFO stack.  Every split decision only
// depends on the node's own particles — their COUNT and shrunk BOUNDS (midpoint ->
// quadrant), both order independent — and the composition of its stable 4-way partitions
// is one stable sort of the particles by leaf.  So the default build (build_tree):
//   level 0 : face_project per particle, the face as its label, the six roots' counts and
//             bounds (k_face_label, k_root_geom)
//   level d : particles of splitting frontier clusters take the label "quadrant q of
//             cluster p" while per-(cluster, quadrant) counts and bounds accumulate
//             (k_label); the frontier's children are allocated on the device in parent and
//             quadrant order (k_alloc_scan, k_alloc_fill); no host round trip inside a
//             batch of levels
//   at the end: one stable radix sort of the particles by their leaf's first tree-order
//             slot (radix.cuh) -> perm; positions and face coordinates gathered once;
//             every radius in one pass (a warp per leaf over its ancestors)
// The level-synchronous build of rounds 1-2 (the particles partitioned level by level,
// CSFS_B200_TREE=levels) is kept for A/B and as the bitwise cross-check of the default.
// Internal cluster ids are level-major (BFS); reference_ids() maps them onto the
// reference's LIFO numbering for export.  Particle data stays SoA in HBM.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "engine.hpp"
#include "radix.cuh"
#include "scan.cuh"

namespace csfs_b200 {

namespace {

constexpr int kThreads = 256;
#ifndef CSFS_LOCAL_MIN
#define CSFS_LOCAL_MIN 256
#endif
constexpr int kLocalMinClusters = CSFS_LOCAL_MIN;  // frontier size from which levels split locally

// Also flags points off the unit sphere (| |x|^2 - 1 | > 1e-12): the coincidence-guard
// elision of the evaluation (traverse.cu needs_guard) assumes unit vectors, so a tree with
// such points keeps the guard on every list entry (the reference's behaviour).
__global__ void k_face(const double* __restrict__ xyz, long long n, int* fface, double* fxi,
                       double* feta, int* off_sphere) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int f;
    double a, b;
    const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    face_project(x, y, z, f, a, b);
    fface[i] = f;
    fxi[i] = a;
    feta[i] = b;
    if (!(fabs(x * x + y * y + z * z - 1.0) <= 1e-12)) atomicOr(off_sphere, 1);
}

struct ClusterPtrs {
    int *face, *depth, *begin, *end, *parent, *nchild;
    int4* child;
    double *xi0, *xi1, *eta0, *eta1, *cx, *cy, *cz, *rad;
    unsigned char* split;
    unsigned long long* bnd;
    double2* mid;
};

ClusterPtrs cluster_ptrs(DeviceTree& t) {
    return {t.face, t.depth, t.begin, t.end, t.parent, t.nchild, t.child, t.xi0, t.xi1,
            t.eta0, t.eta1, t.cx,    t.cy,    t.cz,  t.rad,    t.split,  t.bnd, t.mid};
}

__global__ void k_roots(ClusterPtrs c, const int* grand) {
    const int k = threadIdx.x;
    if (k >= 6) return;
    int b = 0;
    for (int j = 0; j < k; ++j) b += grand[j];
    c.face[k] = k;
    c.depth[k] = 0;
    c.begin[k] = b;
    c.end[k] = b + grand[k];
    c.parent[k] = -1;
    c.nchild[k] = 0;
    c.child[k] = make_int4(-1, -1, -1, -1);
    // face square (cluster_tree.cpp:72)
    c.xi0[k] = -kPi / 4.0;
    c.xi1[k] = kPi / 4.0;
    c.eta0[k] = -kPi / 4.0;
    c.eta1[k] = kPi / 4.0;
}

// --- per-level finishing (finish_cluster lambda, cluster_tree.cpp:52-70) ------------------

__global__ void k_bnd_init(int first, const int* nnew_dev, int cnt_host, ClusterPtrs c) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int cnt = nnew_dev ? *nnew_dev : cnt_host;
    if (j >= cnt) return;
    const int id = first + j;
    c.bnd[4 * id + 0] = ~0ull;
    c.bnd[4 * id + 1] = 0ull;
    c.bnd[4 * id + 2] = ~0ull;
    c.bnd[4 * id + 3] = 0ull;
    c.rad[id] = 0.0;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o < v ? o : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o > v ? o : v;
    }
    return v;
}

constexpr int kSegItems = 8;  // consecutive particles per thread in k_bounds

// Shrunk bounds: min/max of xi, eta over each new cluster's particles (:53-61).  Each thread
// first reduces kSegItems CONSECUTIVE particles in registers (a cluster change inside the
// run flushes with atomics), then the warp combines the per-thread results once; particles
// of a cluster are contiguous, so most warps see a single cluster for 256 particles.
__global__ void k_bounds(long long n, int first, const int* nnew_dev, int cnt_host,
                         const int* __restrict__ node, const double* __restrict__ xi,
                         const double* __restrict__ eta, unsigned long long* bnd) {
    const int cnt = nnew_dev ? *nnew_dev : cnt_host;
    const long long base = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kSegItems;
    constexpr int op[4] = {0, 1, 0, 1};
    int cur = -1;
    unsigned long long acc[4] = {~0ull, 0ull, ~0ull, 0ull};
    auto flush = [&]() {
        if (cur >= 0) {
            atomicMin(&bnd[4ll * cur + 0], acc[0]);
            atomicMax(&bnd[4ll * cur + 1], acc[1]);
            atomicMin(&bnd[4ll * cur + 2], acc[2]);
            atomicMax(&bnd[4ll * cur + 3], acc[3]);
        }
    };
    bool mixed = false;  // this thread's run holds more than one cluster
#pragma unroll
    for (int j = 0; j < kSegItems; ++j) {
        const long long i = base + j;
        if (i >= n) break;
        int nd = node[i];
        if (!(nd >= first && nd < first + cnt)) nd = -1;
        if (nd < 0) continue;
        const unsigned long long vx = ord_enc(xi[i]), ve = ord_enc(eta[i]);
        if (nd != cur) {
            if (cur >= 0) {
                flush();
                mixed = true;
            }
            cur = nd;
            acc[0] = acc[1] = vx;
            acc[2] = acc[3] = ve;
        } else {
            acc[0] = vx < acc[0] ? vx : acc[0];
            acc[1] = vx > acc[1] ? vx : acc[1];
            acc[2] = ve < acc[2] ? ve : acc[2];
            acc[3] = ve > acc[3] ? ve : acc[3];
        }
    }
    // warp combine when every lane ends on the same cluster and none was mixed
    const int c0 = __shfl_sync(0xffffffffu, cur, 0);
    if (__all_sync(0xffffffffu, cur == c0 && !mixed)) {
        if (c0 < 0) return;
        unsigned long long r[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) r[v] = op[v] ? warp_max_u64(acc[v]) : warp_min_u64(acc[v]);
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&bnd[4ll * c0 + 0], r[0]);
            atomicMax(&bnd[4ll * c0 + 1], r[1]);
            atomicMin(&bnd[4ll * c0 + 2], r[2]);
            atomicMax(&bnd[4ll * c0 + 3], r[3]);
        }
    } else {
        flush();
    }
}

// Bounds -> interpolant rectangle, centre (:65-66) and the split decision (:95-96).
__device__ __forceinline__ bool geom_one(const ClusterPtrs& c, int id, bool shrink, int n0) {
    const int count = c.end[id] - c.begin[id];
    double x0 = c.xi0[id], x1 = c.xi1[id], e0 = c.eta0[id], e1 = c.eta1[id];
    if (shrink && count > 0) {
        x0 = ord_dec(c.bnd[4 * id + 0]);
        x1 = ord_dec(c.bnd[4 * id + 1]);
        e0 = ord_dec(c.bnd[4 * id + 2]);
        e1 = ord_dec(c.bnd[4 * id + 3]);
        c.xi0[id] = x0;
        c.xi1[id] = x1;
        c.eta0[id] = e0;
        c.eta1[id] = e1;
    }
    const double xm = __dmul_rn(0.5, __dadd_rn(x0, x1));
    const double em = __dmul_rn(0.5, __dadd_rn(e0, e1));
    double x, y, z;
    face_unproject(c.face[id], xm, em, x, y, z);
    c.cx[id] = x;
    c.cy[id] = y;
    c.cz[id] = z;
    const double ex = __dsub_rn(x1, x0), ey = __dsub_rn(e1, e0);
    const double ext = (ex < ey) ? ey : ex;  // std::max
    const bool sp = !(count <= n0 || c.depth[id] >= kMaxDepth) && !(ext < kMinExtent);
    c.split[id] = sp ? 1 : 0;
    c.mid[id] = make_double2(xm, em);  // the split point quadrant_of derives (:98-99)
    return sp;
}

__global__ void k_geom(int first, const int* nnew_dev, int cnt_host, ClusterPtrs c, bool shrink,
                       int n0, int* nsplit) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int cnt = nnew_dev ? *nnew_dev : cnt_host;
    if (j >= cnt) return;
    const int id = first + j;
    if (geom_one(c, id, shrink, n0)) atomicAdd(nsplit, 1);
}

// Radii of every cluster once the tree is final (:67-69), by leaf: one warp per leaf computes its particles' chordal distances to the leaf's
// centre and to every ancestor's, reduces each over the warp and max-es it into the
// ancestor (integer atomics on the bit patterns of non-negative doubles: exact, order
// independent).  Positions are read once per leaf (re-reads hit L1); the same distances
// and maxima as a per-particle walk, with one atomic per (leaf, ancestor).
__global__ void k_radius_leaf(int ncl, const int* __restrict__ nchild, const int* __restrict__ begin,
                              const int* __restrict__ end, const int* __restrict__ parent,
                              const double* __restrict__ px, const double* __restrict__ py,
                              const double* __restrict__ pz, const double* __restrict__ cx,
                              const double* __restrict__ cy, const double* __restrict__ cz, double* rad) {
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (c >= ncl || nchild[c] > 0) return;  // warp-uniform
    const int b = begin[c], e = end[c];
    unsigned long long* radu = reinterpret_cast<unsigned long long*>(rad);
    for (int a = c; a >= 0; a = parent[a]) {
        const double ax = cx[a], ay = cy[a], az = cz[a];
        unsigned long long m = 0;
        for (int i = b + lane; i < e; i += 32) {
            const double dx = __dsub_rn(ax, px[i]);
            const double dy = __dsub_rn(ay, py[i]);
            const double dz = __dsub_rn(az, pz[i]);
            // the squared distance: sqrt is monotone, so sqrt(max d^2) = max sqrt(d^2) bit for bit
            // (one correctly rounded sqrt per cluster, k_rad_sqrt, instead of one per distance)
            const unsigned long long v = __double_as_longlong(dot_ref(dx, dy, dz, dx, dy, dz));
            m = v > m ? v : m;
        }
        m = warp_max_u64(m);
        if (lane == 0 && b < e) atomicMax(&radu[a], m);
    }
}

__global__ void k_rad_sqrt(int ncl, double* rad) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < ncl) rad[c] = __dsqrt_rn(rad[c]);
}

__global__ void k_gather_xyz(long long n, const int* __restrict__ perm, const double* __restrict__ xyz,
                             double* px, double* py, double* pz) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long q = perm[i];
    px[i] = xyz[3 * q];
    py[i] = xyz[3 * q + 1];
    pz[i] = xyz[3 * q + 2];
}

// --- splitting (cluster_tree.cpp:87-141) ------------------------------------------------

__device__ __forceinline__ int quadrant_of(const ClusterPtrs& c, int nd, double x, double e) {
    const double mx = __dmul_rn(0.5, __dadd_rn(c.xi0[nd], c.xi1[nd]));
    const double my = __dmul_rn(0.5, __dadd_rn(c.eta0[nd], c.eta1[nd]));
    return (x >= mx ? 1 : 0) + (e >= my ? 2 : 0);
}

// Children of splitting frontier node `id` (frontier index f), ids from `cid`, in quadrant
// order with empty quadrants pruned (:124-140); records each quadrant's destination offset
// and child id for the scatter.
__device__ __forceinline__ void emit_children(const ClusterPtrs& c, int id, int f, int cid, const int* segP,
                                              const int* segE, int* kid, int* koff) {
    int acc = c.begin[id];
    const double x0 = c.xi0[id], x1 = c.xi1[id], e0 = c.eta0[id], e1 = c.eta1[id];
    const double mx = __dmul_rn(0.5, __dadd_rn(x0, x1));
    const double my = __dmul_rn(0.5, __dadd_rn(e0, e1));
    const double rx0[4] = {x0, mx, x0, mx}, rx1[4] = {mx, x1, mx, x1};
    const double ry0[4] = {e0, e0, my, my}, ry1[4] = {my, my, e1, e1};
    int ch[4] = {-1, -1, -1, -1};
    int nch = 0;
    const int fc = c.face[id], dp = c.depth[id] + 1;
    for (int k = 0; k < 4; ++k) {
        const int cntk = segE[4 * f + k] - segP[4 * f + k];
        koff[4 * f + k] = acc;
        kid[4 * f + k] = -1;
        if (cntk > 0) {
            c.face[cid] = fc;
            c.depth[cid] = dp;
            c.begin[cid] = acc;
            c.end[cid] = acc + cntk;
            c.parent[cid] = id;
            c.nchild[cid] = 0;
            c.child[cid] = make_int4(-1, -1, -1, -1);
            c.xi0[cid] = rx0[k];
            c.xi1[cid] = rx1[k];
            c.eta0[cid] = ry0[k];
            c.eta1[cid] = ry1[k];
            kid[4 * f + k] = cid;
            ch[nch++] = cid;
            ++cid;
        }
        acc += cntk;
    }
    c.child[id] = make_int4(ch[0], ch[1], ch[2], ch[3]);
    c.nchild[id] = nch;
}

struct PartArrays {
    const double *px, *py, *pz, *xi, *eta, *w;
    const int *perm, *node;
    double *px2, *py2, *pz2, *xi2, *eta2, *w2;
    int *perm2, *node2;
};

// Stable scatter: moving particles go to koff + rank-within-(node, quadrant), others stay.
__global__ void k_scatter(long long n, int first, int cnt, ClusterPtrs c, PartArrays a,
                          const int* __restrict__ rank, const int* __restrict__ segP,
                          const int* __restrict__ kid, const int* __restrict__ koff) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nd = a.node[i];
    long long pos = i;
    int newnode = nd;
    const double x = a.xi[i], e = a.eta[i];
    if (nd >= first && nd < first + cnt && c.split[nd]) {
        const int q = quadrant_of(c, nd, x, e);
        const int f = nd - first;
        pos = koff[4 * f + q] + (rank[i] - segP[4 * f + q]);
        newnode = kid[4 * f + q];
    }
    if (a.px) {
        a.px2[pos] = a.px[i];
        a.py2[pos] = a.py[i];
        a.pz2[pos] = a.pz[i];
    }
    a.xi2[pos] = x;
    a.eta2[pos] = e;
    a.perm2[pos] = a.perm[i];
    a.node2[pos] = newnode;
    if (a.w) a.w2[pos] = a.w[i];
}

// --- local levels: one CTA per frontier cluster ----------------------------------------
// Once the frontier holds enough clusters to fill the GPU, a level is split cluster by
// cluster instead of with whole-array scans: k_part sizes and bounds every quadrant of a
// splitting cluster and writes its particles into the other buffer, stably partitioned by
// quadrant (a block-wide 4-counter scan per tile of 1024; the second read of the cluster
// mostly hits L2); the frontier allocator (emit_children) then assigns the children.
// Clusters that stop splitting copy their range across once, so both buffers keep every
// finished leaf and the buffers can still be swapped per level.  Same result as the global
// path (stable partition, exact min/max), ~56 instead of ~112 B/particle per level and
// 5 launches instead of 10.

__global__ void __launch_bounds__(kScanThreads) k_part(int first, int cnt, ClusterPtrs c,
                                                       const double* __restrict__ xi, const double* __restrict__ eta,
                                                       const int* __restrict__ perm, double* xi2, double* eta2,
                                                       int* perm2, int* segP, int* segE, unsigned long long* qbnd) {
    const int f = blockIdx.x;
    const int nd = first + f;
    if (f >= cnt) return;
    const int b = c.begin[nd], e = c.end[nd];
    if (!c.split[nd]) {  // finishes here: copy across once (see above)
        for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
            xi2[i] = xi[i];
            eta2[i] = eta[i];
            perm2[i] = perm[i];
        }
        return;
    }
    int n4[4] = {0, 0, 0, 0};
    unsigned long long lo[4][2], hi[4][2];  // [q][xi, eta]
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        lo[q][0] = lo[q][1] = ~0ull;
        hi[q][0] = hi[q][1] = 0ull;
    }
    for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
        const double x = xi[i], y = eta[i];
        const int q = quadrant_of(c, nd, x, y);
        const unsigned long long ux = ord_enc(x), uy = ord_enc(y);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k == q) {
                ++n4[k];
                lo[k][0] = ux < lo[k][0] ? ux : lo[k][0];
                hi[k][0] = ux > hi[k][0] ? ux : hi[k][0];
                lo[k][1] = uy < lo[k][1] ? uy : lo[k][1];
                hi[k][1] = uy > hi[k][1] ? uy : hi[k][1];
            }
    }
    __shared__ unsigned long long sh[kScanThreads / 32][4][5];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        unsigned long long v[5] = {(unsigned long long)n4[q], lo[q][0], hi[q][0], lo[q][1], hi[q][1]};
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], d);
            unsigned long long o;
            o = __shfl_xor_sync(0xffffffffu, v[1], d);
            v[1] = o < v[1] ? o : v[1];
            o = __shfl_xor_sync(0xffffffffu, v[2], d);
            v[2] = o > v[2] ? o : v[2];
            o = __shfl_xor_sync(0xffffffffu, v[3], d);
            v[3] = o < v[3] ? o : v[3];
            o = __shfl_xor_sync(0xffffffffu, v[4], d);
            v[4] = o > v[4] ? o : v[4];
        }
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 5; ++k) sh[w][q][k] = v[k];
    }
    __syncthreads();
    __shared__ int qn[4];
    if (threadIdx.x < 4) {
        const int q = threadIdx.x;
        unsigned long long v[5] = {0, ~0ull, 0, ~0ull, 0};
        for (int ww = 0; ww < kScanThreads / 32; ++ww) {
            v[0] += sh[ww][q][0];
            v[1] = sh[ww][q][1] < v[1] ? sh[ww][q][1] : v[1];
            v[2] = sh[ww][q][2] > v[2] ? sh[ww][q][2] : v[2];
            v[3] = sh[ww][q][3] < v[3] ? sh[ww][q][3] : v[3];
            v[4] = sh[ww][q][4] > v[4] ? sh[ww][q][4] : v[4];
        }
        qn[q] = int(v[0]);
        segP[4 * f + q] = 0;
        segE[4 * f + q] = int(v[0]);
        // min xi, max xi, min eta, max eta (the k_bounds layout)
        qbnd[16 * f + 4 * q + 0] = v[1];
        qbnd[16 * f + 4 * q + 1] = v[2];
        qbnd[16 * f + 4 * q + 2] = v[3];
        qbnd[16 * f + 4 * q + 3] = v[4];
    }
    __syncthreads();
    // stable scatter by quadrant into the other buffer: the children's ranges follow in
    // quadrant order from the parent's begin (emit_children's offsets), so no allocator
    // result is needed here; a block-wide 4-counter scan per tile of kScanTile particles
    int base[4];
    base[0] = b;
#pragma unroll
    for (int q = 1; q < 4; ++q) base[q] = base[q - 1] + qn[q - 1];
    for (int t0 = b; t0 < e; t0 += kScanTile) {
        const int i0 = t0 + threadIdx.x * kScanItems;
        int qq[kScanItems];
        int cc[4] = {0, 0, 0, 0};
        double xv[kScanItems], ev[kScanItems];
        int pv[kScanItems];
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const int i = i0 + j;
            qq[j] = -1;
            if (i < e) {
                xv[j] = xi[i];
                ev[j] = eta[i];
                pv[j] = perm[i];
                qq[j] = quadrant_of(c, nd, xv[j], ev[j]);
#pragma unroll
                for (int k = 0; k < 4; ++k) cc[k] += (qq[j] == k);
            }
        }
        int tot[4];
        block_exclusive_scan<4>(cc, tot);
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            if (qq[j] < 0) continue;
            int pos = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (qq[j] == k) pos = base[k] + cc[k]++;
            xi2[pos] = xv[j];
            eta2[pos] = ev[j];
            perm2[pos] = pv[j];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) base[k] += tot[k];
    }
}

// Children's bounds from the quadrant bounds (what k_bnd_init + k_bounds produce globally).
__global__ void k_part_bnd(int first, int cnt, ClusterPtrs c, const int* __restrict__ kid,
                           const unsigned long long* __restrict__ qbnd) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= 4 * cnt) return;
    const int f = j >> 2, q = j & 3;
    if (!c.split[first + f]) return;
    const int id = kid[4 * f + q];
    if (id < 0) return;
#pragma unroll
    for (int v = 0; v < 4; ++v) c.bnd[4 * id + v] = qbnd[16 * f + 4 * q + v];
    c.rad[id] = 0.0;
}

// node[] (particle -> leaf) after local levels, which do not maintain it per particle.
__global__ void k_fill_node(int ncl, const int* __restrict__ begin, const int* __restrict__ end,
                            const int* __restrict__ nchild, int* node) {
    const int c = blockIdx.x;
    if (c >= ncl || nchild[c] > 0) return;
    for (int i = begin[c] + threadIdx.x; i < end[c]; i += blockDim.x) node[i] = c;
}

// --- label-then-sort build (the default) --------------------------------------------------
// Particles never move while the levels are decided.  Each particle keeps a label in input
// order: a cluster id (>= 0), or -(4 p + q + 1) = "quadrant q of splitting cluster p", which
// resolves through qchild[4 p + q] once the next level is allocated.  Per level:
//   k_label : particles of splitting frontier clusters take their quadrant label; per
//             (cluster, quadrant) the count and the shrunk bounds accumulate with atomics
//             (integer min/max on order-preserving encodings: exact and order independent),
//             aggregated over the lanes of a warp that share a quadrant (match_any + redux);
//   k_alloc : one CTA allocates the children of the whole frontier in parent and quadrant
//             order (empties pruned: cluster_tree.cpp:124-140), sets their ranges from the
//             quadrant counts, bounds, centres and split decisions, and writes the next
//             level's descriptor — so no level needs the host.
// After the last level ONE stable sort of the particles by their leaf's begin yields the
// reference's order: the composition of its stable 4-way partitions keeps every leaf's
// particles in input order.
struct LevelDesc {
    int first, cnt, nsplit, ovf;
};

__device__ __forceinline__ unsigned long long redux_min_u64(unsigned m, unsigned long long v) {
    const unsigned hi = unsigned(v >> 32);
    const unsigned mh = __reduce_min_sync(m, hi);
    const unsigned ml = __reduce_min_sync(m, hi == mh ? unsigned(v) : 0xffffffffu);
    return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned long long redux_max_u64(unsigned m, unsigned long long v) {
    const unsigned hi = unsigned(v >> 32);
    const unsigned mh = __reduce_max_sync(m, hi);
    const unsigned ml = __reduce_max_sync(m, hi == mh ? unsigned(v) : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

// Per-(cluster, quadrant) counts and bounds over a tile of kTile consecutive particles.
// The particles' slots and face coordinates are first staged in shared memory with
// coalesced loads (phase A, one particle per thread per step); then each thread walks kRun
// CONSECUTIVE staged particles, keeping count and bounds in registers while the slot stays
// the same (a change flushes the finished run with atomics: integer min/max on
// order-preserving encodings, exact and order independent).  A tile whose particles all
// share one slot (the top levels on coherent inputs) is reduced over the CTA and issues one
// set of atomics; otherwise the lanes whose last runs share a slot combine them
// (match_any + redux) and one of them issues the atomics.
#ifndef CSFS_TREE_RUN
#define CSFS_TREE_RUN 8
#endif
constexpr int kRun = CSFS_TREE_RUN;
constexpr int kRunThreads = 256;
constexpr int kTile = kRun * kRunThreads;
constexpr int kTilePad = kTile + kTile / kRun;
__device__ __forceinline__ int tpad(int e) { return e + e / kRun; }  // conflict-free per-thread runs

struct RunAcc {
    int key = -1, cnt = 0;
    unsigned long long lo_x = 0, hi_x = 0, lo_e = 0, hi_e = 0;
};

__device__ __forceinline__ void run_flush(const RunAcc& r, int* cnt, unsigned long long* bnd) {
    atomicAdd(&cnt[r.key], r.cnt);
    atomicMin(&bnd[4ll * r.key + 0], r.lo_x);
    atomicMax(&bnd[4ll * r.key + 1], r.hi_x);
    atomicMin(&bnd[4ll * r.key + 2], r.lo_e);
    atomicMax(&bnd[4ll * r.key + 3], r.hi_e);
}

struct TileStage {
    int key[kTilePad];
    double x[kTilePad], e[kTilePad];
};

__device__ __forceinline__ void tile_accumulate(const TileStage& st, int* cnt, unsigned long long* bnd) {
    RunAcc r;
    bool flushed = false;
#pragma unroll
    for (int j = 0; j < kRun; ++j) {
        const int p = tpad(threadIdx.x * kRun + j);
        const int key = st.key[p];
        if (key < 0) continue;
        const unsigned long long ux = ord_enc(st.x[p]), ue = ord_enc(st.e[p]);
        if (key != r.key) {
            if (r.key >= 0) {
                run_flush(r, cnt, bnd);
                flushed = true;
            }
            r.key = key;
            r.cnt = 1;
            r.lo_x = r.hi_x = ux;
            r.lo_e = r.hi_e = ue;
        } else {
            ++r.cnt;
            r.lo_x = ux < r.lo_x ? ux : r.lo_x;
            r.hi_x = ux > r.hi_x ? ux : r.hi_x;
            r.lo_e = ue < r.lo_e ? ue : r.lo_e;
            r.hi_e = ue > r.hi_e ? ue : r.hi_e;
        }
    }
    const int key0 = st.key[0];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (__syncthreads_and(key0 >= 0 && !flushed && (r.key == key0 || r.key < 0))) {
        // one slot for the whole tile: CTA reduction, one set of atomics
        __shared__ unsigned long long red[kRunThreads / 32][5];
        const unsigned long long v[5] = {(unsigned long long)(r.key < 0 ? 0 : r.cnt), r.key < 0 ? ~0ull : r.lo_x,
                                         r.key < 0 ? 0ull : r.hi_x, r.key < 0 ? ~0ull : r.lo_e,
                                         r.key < 0 ? 0ull : r.hi_e};
        const unsigned long long c = __reduce_add_sync(0xffffffffu, unsigned(v[0]));
        const unsigned long long a0 = redux_min_u64(0xffffffffu, v[1]), a1 = redux_max_u64(0xffffffffu, v[2]);
        const unsigned long long a2 = redux_min_u64(0xffffffffu, v[3]), a3 = redux_max_u64(0xffffffffu, v[4]);
        if (lane == 0) {
            red[w][0] = c;
            red[w][1] = a0;
            red[w][2] = a1;
            red[w][3] = a2;
            red[w][4] = a3;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            RunAcc t;
            t.key = key0;
            unsigned long long cc = 0;
            t.lo_x = t.lo_e = ~0ull;
            for (int k = 0; k < kRunThreads / 32; ++k) {
                cc += red[k][0];
                t.lo_x = red[k][1] < t.lo_x ? red[k][1] : t.lo_x;
                t.hi_x = red[k][2] > t.hi_x ? red[k][2] : t.hi_x;
                t.lo_e = red[k][3] < t.lo_e ? red[k][3] : t.lo_e;
                t.hi_e = red[k][4] > t.hi_e ? red[k][4] : t.hi_e;
            }
            t.cnt = int(cc);
            run_flush(t, cnt, bnd);
        }
        return;
    }
    // The lanes hold consecutive runs of the tile, so the runs of one slot sit in ADJACENT
    // lanes: a segmented reduction over the runs of equal-key adjacent lanes, five
    // full-mask shuffle steps whatever the number of slots in the warp.  (match_any +
    // redux.sync over each slot's lanes compiles to a loop over the distinct masks: at the
    // deep levels of a grid, 16 slots per warp, that loop was 36% of the kernel's
    // instructions and half of its stall samples — ncu, round 2.)  Equal keys in
    // non-adjacent lanes (incoherent inputs) simply flush separately: the atomics combine
    // them, exact and order independent either way.
    constexpr unsigned kFull = 0xffffffffu;
    const int kprev = __shfl_up_sync(kFull, r.key, 1);
    const bool head = lane == 0 || kprev != r.key;
    const unsigned heads = __ballot_sync(kFull, head);
    RunAcc t = r;
    if (r.key < 0) {
        t.cnt = 0;
        t.lo_x = t.lo_e = ~0ull;
        t.hi_x = t.hi_e = 0ull;
    }
    if (heads == 1u) {  // one slot for the whole warp: plain warp reductions
        t.cnt = int(__reduce_add_sync(kFull, unsigned(t.cnt)));
        t.lo_x = redux_min_u64(kFull, t.lo_x);
        t.hi_x = redux_max_u64(kFull, t.hi_x);
        t.lo_e = redux_min_u64(kFull, t.lo_e);
        t.hi_e = redux_max_u64(kFull, t.hi_e);
    } else {
        const unsigned above = heads & ~((2u << lane) - 1u);  // heads past this lane
        const int last = above ? __ffs(above) - 2 : 31;       // the last lane of this lane's run
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int c = __shfl_down_sync(kFull, t.cnt, d);
            const unsigned long long a0 = __shfl_down_sync(kFull, t.lo_x, d), a1 = __shfl_down_sync(kFull, t.hi_x, d);
            const unsigned long long a2 = __shfl_down_sync(kFull, t.lo_e, d), a3 = __shfl_down_sync(kFull, t.hi_e, d);
            if (lane + d <= last) {
                t.cnt += c;
                t.lo_x = a0 < t.lo_x ? a0 : t.lo_x;
                t.hi_x = a1 > t.hi_x ? a1 : t.hi_x;
                t.lo_e = a2 < t.lo_e ? a2 : t.lo_e;
                t.hi_e = a3 > t.hi_e ? a3 : t.hi_e;
            }
        }
    }
    if (head && r.key >= 0) run_flush(t, cnt, bnd);
}

__global__ void k_root_init(ClusterPtrs c, int* rcnt) {
    const int k = threadIdx.x;
    if (k == 6) rcnt[6] = 0;  // OR of every cluster's first slot (the sort key's common zero bits)
    if (k < 6) {
        rcnt[k] = 0;
        c.bnd[4 * k + 0] = ~0ull;
        c.bnd[4 * k + 1] = 0ull;
        c.bnd[4 * k + 2] = ~0ull;
        c.bnd[4 * k + 3] = 0ull;
    }
}

// Level 0 (cluster_tree.cpp:35-50): face coordinates, the face label, and the six roots'
// counts and bounds.  Also flags points off the unit sphere (see k_face).
__global__ void __launch_bounds__(kRunThreads)
    k_face_label(const double* __restrict__ xyz, long long n, double* fxi, double* feta, int* lab, int* off_sphere,
                 int* rcnt, unsigned long long* rbnd) {
    __shared__ TileStage st;
    const long long base = (long long)blockIdx.x * kTile;
    bool off = false;
#pragma unroll 2
    for (int j = 0; j < kRun; ++j) {
        const int el = j * kRunThreads + threadIdx.x;
        const long long i = base + el;
        int f = -1;
        double a = 0.0, b = 0.0;
        if (i < n) {
            const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
            face_project(x, y, z, f, a, b);
            fxi[i] = a;
            feta[i] = b;
            lab[i] = f;
            off = off || !(fabs(x * x + y * y + z * z - 1.0) <= 1e-12);
        }
        const int p = tpad(el);
        st.key[p] = f;
        st.x[p] = a;
        st.e[p] = b;
    }
    if (off) atomicOr(off_sphere, 1);
    __syncthreads();
    tile_accumulate(st, rcnt, rbnd);
}

// The six roots (:71-82): ranges in face order, face squares, shrunk bounds, centres and
// split decisions; level 0's descriptor; the roots' quadrant accumulators.
__global__ void k_root_geom(ClusterPtrs c, int* rcnt, bool shrink, int n0, LevelDesc* lev, int* scnt,
                            unsigned long long* sbnd) {
    __shared__ int nsp;
    const int k = threadIdx.x;
    if (k == 0) nsp = 0;
    __syncthreads();
    if (k < 6) {
        int b = 0;
        for (int j = 0; j < k; ++j) b += rcnt[j];
        c.face[k] = k;
        c.depth[k] = 0;
        c.begin[k] = b;
        c.end[k] = b + rcnt[k];
        if (rcnt[k] > 0) atomicOr(&rcnt[6], b);
        c.parent[k] = -1;
        c.nchild[k] = 0;
        c.child[k] = make_int4(-1, -1, -1, -1);
        c.xi0[k] = -kPi / 4.0;
        c.xi1[k] = kPi / 4.0;
        c.eta0[k] = -kPi / 4.0;
        c.eta1[k] = kPi / 4.0;
        c.rad[k] = 0.0;
        if (geom_one(c, k, shrink, n0)) atomicAdd(&nsp, 1);
        for (int q = 0; q < 4; ++q) {
            scnt[4 * k + q] = 0;
            sbnd[16 * k + 4 * q + 0] = ~0ull;
            sbnd[16 * k + 4 * q + 1] = 0ull;
            sbnd[16 * k + 4 * q + 2] = ~0ull;
            sbnd[16 * k + 4 * q + 3] = 0ull;
        }
    }
    __syncthreads();
    if (k == 0) lev[0] = LevelDesc{0, 6, nsp, 0};
}

// Level d: quadrant labels of the particles of splitting frontier clusters (:97-100).
// Phase A is written as three independent sweeps over the thread's kRun particles (labels
// and face coordinates, then label resolution, then the quadrant test) so that each
// sweep's loads are all in flight together.
__global__ void __launch_bounds__(kRunThreads)
    k_label(long long n, int d, const LevelDesc* __restrict__ lev, ClusterPtrs c, const double* __restrict__ fxi,
            const double* __restrict__ feta, int* lab, const int* __restrict__ qchild, int* scnt,
            unsigned long long* sbnd) {
    const LevelDesc L = lev[d];
    if (L.nsplit == 0) return;
    __shared__ TileStage st;
    const long long base = (long long)blockIdx.x * kTile + threadIdx.x;
    int v[kRun], nd[kRun];
    double x[kRun], e[kRun];
#pragma unroll
    for (int j = 0; j < kRun; ++j) {
        const long long i = base + j * kRunThreads;
        const bool in = i < n;
        v[j] = in ? lab[i] : INT_MAX;
        x[j] = in ? fxi[i] : 0.0;
        e[j] = in ? feta[i] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kRun; ++j) nd[j] = v[j] < 0 ? qchild[-v[j] - 1] : v[j];
    int cur = -1;  // the thread's particles often share a cluster: its split flag and point once
    bool csp = false;
    double2 cm = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < kRun; ++j) {
        const long long i = base + j * kRunThreads;
        int key = -1;
        if (nd[j] != cur) {
            cur = nd[j];
            csp = cur >= L.first && cur < L.first + L.cnt && c.split[cur];
            if (csp) cm = c.mid[cur];
        }
        if (csp) {
            key = 4 * nd[j] + (x[j] >= cm.x ? 1 : 0) + (e[j] >= cm.y ? 2 : 0);  // quadrant_of
            lab[i] = -(key + 1);
        } else if (v[j] < 0) {
            lab[i] = nd[j];
        }
        const int p = tpad(j * kRunThreads + threadIdx.x);
        st.key[p] = key;
        st.x[p] = x[j];
        st.e[p] = e[j];
    }
    __syncthreads();
    tile_accumulate(st, scnt, sbnd);
}

// Level d's children (:124-140) in two launches: one CTA scans the frontier's non-empty
// quadrant counts into first child ids (parent order, empties pruned); then one thread per
// (frontier cluster, quadrant) creates its child.
constexpr int kAllocThreads = 1024;
constexpr int kAllocItems = 4;

__global__ void __launch_bounds__(kAllocThreads)
    k_alloc_scan(int d, LevelDesc* lev, ClusterPtrs c, const int* __restrict__ scnt, int* cbase, int cap) {
    const LevelDesc L = lev[d];
    const int next = L.first + L.cnt;
    if (L.nsplit == 0) {
        if (threadIdx.x == 0) lev[d + 1] = LevelDesc{next, 0, 0, 0};
        return;
    }
    int carry = 0;
    for (int f0 = 0; f0 < L.cnt; f0 += kAllocThreads * kAllocItems) {
        int m[kAllocItems], tot = 0;
#pragma unroll
        for (int j = 0; j < kAllocItems; ++j) {
            const int f = f0 + threadIdx.x * kAllocItems + j;
            m[j] = 0;
            if (f < L.cnt && c.split[L.first + f]) {
                const int4 q = reinterpret_cast<const int4*>(scnt)[L.first + f];
                m[j] = (q.x > 0) + (q.y > 0) + (q.z > 0) + (q.w > 0);
            }
            tot += m[j];
        }
        int v[1] = {tot}, all[1];
        block_exclusive_scan<1, kAllocThreads>(v, all);
        int b = next + carry + v[0];
#pragma unroll
        for (int j = 0; j < kAllocItems; ++j) {
            const int f = f0 + threadIdx.x * kAllocItems + j;
            if (f < L.cnt) cbase[f] = b;
            b += m[j];
        }
        carry += all[0];
    }
    if (threadIdx.x == 0) {
        const bool ovf = (long long)next + carry > cap;
        lev[d + 1] = LevelDesc{next, ovf ? 0 : carry, 0, ovf ? 1 : 0};
    }
}

__global__ void k_alloc_fill(int d, LevelDesc* lev, ClusterPtrs c, const int* __restrict__ scnt, int* scnt_w,
                             unsigned long long* sbnd, const int* __restrict__ cbase, int* qchild, bool shrink,
                             int n0, int* orb) {
    const LevelDesc L = lev[d];
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    bool sp = false;
    int ob = 0;  // this child's first slot, for the OR of all of them
    if (L.nsplit > 0 && !lev[d + 1].ovf && g < 4 * L.cnt) {
        const int f = g >> 2, q = g & 3, id = L.first + f;
        if (c.split[id]) {
            const int4 cq4 = reinterpret_cast<const int4*>(scnt)[id];
            const int cq[4] = {cq4.x, cq4.y, cq4.z, cq4.w};
            int acc = c.begin[id], k = 0;
            for (int p = 0; p < q; ++p) {
                acc += cq[p];
                k += cq[p] > 0;
            }
            const int cid = cbase[f] + k;
            const int slot = 4 * id + q;
            qchild[slot] = cq[q] > 0 ? cid : -1;
            if (q == 0) {  // the parent's child list (quadrant order, empties pruned)
                int ch[4] = {-1, -1, -1, -1}, m = 0;
                for (int p = 0; p < 4; ++p)
                    if (cq[p] > 0) {
                        ch[m] = cbase[f] + m;
                        ++m;
                    }
                c.child[id] = make_int4(ch[0], ch[1], ch[2], ch[3]);
                c.nchild[id] = m;
            }
            if (cq[q] > 0) {
                const double x0 = c.xi0[id], x1 = c.xi1[id], e0 = c.eta0[id], e1 = c.eta1[id];
                const double mx = __dmul_rn(0.5, __dadd_rn(x0, x1));
                const double my = __dmul_rn(0.5, __dadd_rn(e0, e1));
                c.face[cid] = c.face[id];
                c.depth[cid] = c.depth[id] + 1;
                c.begin[cid] = acc;
                c.end[cid] = acc + cq[q];
                ob = acc;
                c.parent[cid] = id;
                c.nchild[cid] = 0;
                c.child[cid] = make_int4(-1, -1, -1, -1);
                c.xi0[cid] = (q & 1) ? mx : x0;
                c.xi1[cid] = (q & 1) ? x1 : mx;
                c.eta0[cid] = (q & 2) ? my : e0;
                c.eta1[cid] = (q & 2) ? e1 : my;
                c.rad[cid] = 0.0;
#pragma unroll
                for (int v = 0; v < 4; ++v) c.bnd[4ll * cid + v] = sbnd[4ll * slot + v];
                sp = geom_one(c, cid, shrink, n0);
#pragma unroll
                for (int v = 0; v < 4; ++v) {  // the child's own quadrant accumulators
                    scnt_w[4 * cid + v] = 0;
                    sbnd[16ll * cid + 4 * v + 0] = ~0ull;
                    sbnd[16ll * cid + 4 * v + 1] = 0ull;
                    sbnd[16ll * cid + 4 * v + 2] = ~0ull;
                    sbnd[16ll * cid + 4 * v + 3] = 0ull;
                }
            }
        }
    }
    const unsigned b = __ballot_sync(0xffffffffu, sp);
    if (b && (threadIdx.x & 31) == 0) atomicAdd(&lev[d + 1].nsplit, __popc(b));
    const unsigned o = __reduce_or_sync(0xffffffffu, unsigned(ob));
    if (o && (threadIdx.x & 31) == 0) atomicOr(orb, int(o));
}

// Final labels -> sort keys (the leaf's first tree-order slot).
__global__ void k_leaf_key(long long n, const int* __restrict__ lab, const int* __restrict__ qchild,
                           const int* __restrict__ begin, int* key) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int v = lab[i];
    key[i] = begin[v < 0 ? qchild[-v - 1] : v];
}

// Tree order: perm, face coordinates and positions through the sorted positions.  (The
// per-particle leaf, DeviceTree::node, is only kept by the level build, which needs it.)
__global__ void k_gather_tree(long long n, const int* __restrict__ sorted, const double* __restrict__ fxi,
                              const double* __restrict__ feta, const double* __restrict__ xyz, int* perm,
                              double* xi, double* eta, double* px, double* py, double* pz) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int i = sorted[t];
    perm[t] = i;
    xi[t] = fxi[i];
    eta[t] = feta[i];
    px[t] = xyz[3ll * i];
    py[t] = xyz[3ll * i + 1];
    pz[t] = xyz[3ll * i + 2];
}

// Proxy points (interpolation.cpp:51-68): mapped nodes mid + half*s_k, pushed to the sphere.
__global__ void k_proxy(int ncl, int np, Cheb cheb, const int* __restrict__ face,
                        const double* __restrict__ xi0, const double* __restrict__ xi1,
                        const double* __restrict__ eta0, const double* __restrict__ eta1,
                        double* qx, double* qy, double* qz) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int npp = np * np;
    if (g >= (long long)ncl * npp) return;
    const int c = int(g / npp), k = int(g % npp);
    const int k1 = k / np, k2 = k % np;
    const double xm = __dmul_rn(0.5, __dadd_rn(xi0[c], xi1[c]));
    const double xh = __dmul_rn(0.5, __dsub_rn(xi1[c], xi0[c]));
    const double em = __dmul_rn(0.5, __dadd_rn(eta0[c], eta1[c]));
    const double eh = __dmul_rn(0.5, __dsub_rn(eta1[c], eta0[c]));
    const double xn = __dadd_rn(xm, __dmul_rn(xh, cheb.nodes[k1]));
    const double en = __dadd_rn(em, __dmul_rn(eh, cheb.nodes[k2]));
    double x, y, z;
    face_unproject(face[c], xn, en, x, y, z);
    qx[g] = x;
    qy[g] = y;
    qz[g] = z;
}

// Proxy radius: the farthest proxy point from the cluster centre (chordal).  The
// evaluation kernels use it, with the particle radius, to prove a list entry free of
// coincident pairs (kernels_dev.cuh needs_guard).
__global__ void k_qrad(int ncl, int npp, const double* __restrict__ cx, const double* __restrict__ cy,
                       const double* __restrict__ cz, const double* __restrict__ qx, const double* __restrict__ qy,
                       const double* __restrict__ qz, double* qrad) {
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;  // a warp per cluster
    if (c >= ncl) return;  // warp-uniform
    const double ox = cx[c], oy = cy[c], oz = cz[c];
    double r2 = 0.0;
    for (int k = lane; k < npp; k += 32) {  // consecutive proxies: coalesced
        const long long g = (long long)c * npp + k;
        const double dx = qx[g] - ox, dy = qy[g] - oy, dz = qz[g] - oz;
        r2 = fmax(r2, dx * dx + dy * dy + dz * dz);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, d));  // max: order-free
    if (lane == 0) qrad[c] = sqrt(r2);
}

__global__ void k_gather(long long n, const int* __restrict__ perm, const double* __restrict__ src,
                         double* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

__global__ void k_equal(const unsigned long long* a, const unsigned long long* b, long long n,
                        int* diff) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (a[i] != b[i]) {
            *diff = 1;
            return;
        }
}

void finish_level(DeviceTree& t, Scratch& sc, int first, const int* nnew_dev, int cnt_bound,
                  cudaStream_t s) {
    ClusterPtrs c = cluster_ptrs(t);
    const int gb = ceil_div(std::max(cnt_bound, 1), kThreads);
    const int gp = ceil_div(t.n, kThreads);
    const int gs = ceil_div(t.n, kThreads * kSegItems);
    k_bnd_init<<<gb, kThreads, 0, s>>>(first, nnew_dev, cnt_bound, c);
    CSFS_LAUNCH_CHECK();
    k_bounds<<<gs, kThreads, 0, s>>>(t.n, first, nnew_dev, cnt_bound, t.node, t.xi, t.eta, t.bnd);
    CSFS_LAUNCH_CHECK();
    CSFS_CK(cudaMemsetAsync(sc.counters.p + 1, 0, sizeof(int), s));
    k_geom<<<gb, kThreads, 0, s>>>(first, nnew_dev, cnt_bound, c, t.shrink, t.n0, sc.counters.p + 1);
    CSFS_LAUNCH_CHECK();
// radii: once for all levels after the build (k_radius_leaf)
}

template <class T>
void swap_buf(DevBuf<T>& a, DevBuf<T>& b) {
    std::swap(a.p, b.p);
    std::swap(a.cap, b.cap);
}

}  // namespace

void DeviceTree::reserve_clusters(int n_needed, cudaStream_t s) {
    if (n_needed <= cap) return;
    const size_t c = size_t(n_needed) + n_needed / 2 + 64;
    const size_t u = size_t(ncl);
    face.grow_keep(c, u, s);
    depth.grow_keep(c, u, s);
    begin.grow_keep(c, u, s);
    end.grow_keep(c, u, s);
    parent.grow_keep(c, u, s);
    nchild.grow_keep(c, u, s);
    child.grow_keep(c, u, s);
    xi0.grow_keep(c, u, s);
    xi1.grow_keep(c, u, s);
    eta0.grow_keep(c, u, s);
    eta1.grow_keep(c, u, s);
    cx.grow_keep(c, u, s);
    cy.grow_keep(c, u, s);
    cz.grow_keep(c, u, s);
    rad.grow_keep(c, u, s);
    split.grow_keep(c, u, s);
    bnd.grow_keep(4 * c, 4 * u, s);
    mid.grow_keep(c, u, s);
    cap = int(c);
}

TreeView DeviceTree::view() const {
    TreeView v;
    v.n = n;
    v.np = np;
    v.npp = npp;
    v.px = px;
    v.py = py;
    v.pz = pz;
    v.xi = xi;
    v.eta = eta;
    v.w = has_w ? w.p : nullptr;
    v.perm = perm;
    v.node = node;
    v.face = face;
    v.depth = depth;
    v.begin = begin;
    v.end = end;
    v.parent = parent;
    v.nchild = nchild;
    v.child = child;
    v.xi0 = xi0;
    v.xi1 = xi1;
    v.eta0 = eta0;
    v.eta1 = eta1;
    v.cx = cx;
    v.cy = cy;
    v.cz = cz;
    v.rad = rad;
    v.qx = qx;
    v.qrad = qrad;
    v.off_sphere = off_sphere;
    v.qy = qy;
    v.qz = qz;
    return v;
}

static void finish_tree(DeviceTree& t, const double* w_in, long long n, const Cheb& cheb, cudaStream_t s,
                        cudaEvent_t w_ready);

// The level-synchronous build of rounds 1-2 (particles partitioned level by level, one host
// read-back per level); CSFS_B200_TREE=levels selects it (A/B and cross-check of the default).
static void build_tree_levels(DeviceTree& t, Scratch& sc, const double* xyz, const double* w_in, long long n,
                              int degree, int n0, bool shrink, const Cheb& cheb, cudaStream_t s,
                              cudaEvent_t w_ready) {
    t.n = n;
    t.degree = degree;
    t.np = degree + 1;
    t.npp = t.np * t.np;
    t.n0 = n0;
    t.shrink = shrink;
    t.has_w = w_in != nullptr;
    t.ncl = 0;
    t.level_first.clear();
    t.level_count.clear();

    for (DevBuf<double>* b : {&t.px, &t.py, &t.pz, &t.xi, &t.eta, &t.px2, &t.py2, &t.pz2, &t.xi2,
                              &t.eta2, &sc.fxi, &sc.feta})
        b->grow(n);
    for (DevBuf<int>* b : {&t.perm, &t.node, &t.perm2, &t.node2, &t.rank, &sc.fface}) b->grow(n);
    if (t.has_w) {
        t.w.grow(n);
    }
    sc.tiles.grow(scan_tile_ints(n, 6));
    sc.grand.grow(8);
    sc.counters.grow(8);
    t.reserve_clusters(64, s);

    const int gp = ceil_div(n, kThreads);

    // ---- level 0: faces (cluster_tree.cpp:35-50) ------------------------------------------
    t.off_sphere.grow(1);
    CSFS_CK(cudaMemsetAsync(t.off_sphere.p, 0, sizeof(int), s));
    k_face<<<gp, kThreads, 0, s>>>(xyz, n, sc.fface, sc.fxi, sc.feta, t.off_sphere);
    CSFS_LAUNCH_CHECK();
    {
        const int* fface = sc.fface;
        const double* fxi = sc.fxi;
        const double* feta = sc.feta;
        const int* grand = sc.grand;
        double *px = t.px, *py = t.py, *pz = t.pz, *xi = t.xi, *eta = t.eta, *w = t.w;
        int *perm = t.perm, *node = t.node;
        const bool hw = t.has_w;
        auto f = [=] __device__(long long i, int* c) { c[fface[i]] = 1; };
        auto e = [=] __device__(long long i, const int* c, const int* pre) {
            const int k = fface[i];
            int base = 0;
            for (int j = 0; j < k; ++j) base += grand[j];
            const long long p = base + pre[k];
            xi[p] = fxi[i];
            eta[p] = feta[i];
            perm[p] = int(i);
            node[p] = k;
        };
        (void)w;
        (void)hw;
        run_scan<6>(n, f, e, sc.tiles, sc.grand, s);
    }
    k_roots<<<1, 32, 0, s>>>(cluster_ptrs(t), sc.grand);
    CSFS_LAUNCH_CHECK();
    t.ncl = 6;
    t.level_first.push_back(0);
    t.level_count.push_back(6);
    finish_level(t, sc, 0, nullptr, 6, s);
    CSFS_CK(cudaMemcpyAsync(sc.host, sc.counters.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaMemcpyAsync(sc.host + 2, sc.grand.p, 6 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaStreamSynchronize(s));
    int nsplit = sc.host[1];
    t.root_count.assign(sc.host + 2, sc.host + 8);

    // ---- levels 1.. (cluster_tree.cpp:87-141) ----------------------------------------------
    bool local = false;  // once on, stays on (node[] is rebuilt at the end)
    while (nsplit > 0) {
        const int first = t.level_first.back();
        const int cnt = t.level_count.back();
        const int next_id = t.ncl;
        t.reserve_clusters(t.ncl + 4 * nsplit, s);
        sc.segP.grow(4 * size_t(cnt));
        sc.segE.grow(4 * size_t(cnt));
        sc.kid.grow(4 * size_t(cnt));
        sc.koff.grow(4 * size_t(cnt));
        ClusterPtrs c = cluster_ptrs(t);
        local = local || cnt >= kLocalMinClusters;
        if (local) {
            sc.qbnd.grow(16 * size_t(cnt));
            k_part<<<cnt, kScanThreads, 0, s>>>(first, cnt, c, t.xi, t.eta, t.perm, t.xi2, t.eta2, t.perm2, sc.segP,
                                                sc.segE, sc.qbnd);
            CSFS_LAUNCH_CHECK();
            {  // child allocation over the frontier (as below)
                const int* segP = sc.segP;
                const int* segE = sc.segE;
                int* kid = sc.kid;
                int* koff = sc.koff;
                auto f = [=] __device__(long long fi, int* cc) {
                    if (!c.split[first + fi]) return;
                    int m = 0;
                    for (int k = 0; k < 4; ++k) m += (segE[4 * fi + k] - segP[4 * fi + k]) > 0;
                    cc[0] = m;
                };
                auto e = [=] __device__(long long fi, const int* cc, const int* pre) {
                    if (c.split[first + fi])
                        emit_children(c, first + int(fi), int(fi), next_id + pre[0], segP, segE, kid, koff);
                };
                run_scan<1>(cnt, f, e, sc.tiles, sc.grand, s);
                CSFS_CK(cudaMemcpyAsync(sc.counters.p, sc.grand.p, sizeof(int), cudaMemcpyDeviceToDevice, s));
            }
            swap_buf(t.xi, t.xi2);
            swap_buf(t.eta, t.eta2);
            swap_buf(t.perm, t.perm2);
            k_part_bnd<<<ceil_div(4 * cnt, kThreads), kThreads, 0, s>>>(first, cnt, c, sc.kid, sc.qbnd);
            CSFS_LAUNCH_CHECK();
            CSFS_CK(cudaMemsetAsync(sc.counters.p + 1, 0, sizeof(int), s));
            k_geom<<<ceil_div(4 * nsplit, kThreads), kThreads, 0, s>>>(next_id, sc.counters.p, 4 * nsplit, c,
                                                                        t.shrink, t.n0, sc.counters.p + 1);
            CSFS_LAUNCH_CHECK();
            CSFS_CK(cudaMemcpyAsync(sc.host, sc.counters.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
            CSFS_CK(cudaStreamSynchronize(s));
            const int nnew = sc.host[0];
            nsplit = sc.host[1];
            t.ncl += nnew;
            t.level_first.push_back(next_id);
            t.level_count.push_back(nnew);
            continue;
        }
        {
            const int* node = t.node;
            const double* xi = t.xi;
            const double* eta = t.eta;
            int* rank = t.rank;
            int* segP = sc.segP;
            int* segE = sc.segE;
            auto f = [=] __device__(long long i, int* cc) {
                const int nd = node[i];
                if (nd >= first && nd < first + cnt && c.split[nd])
                    cc[quadrant_of(c, nd, xi[i], eta[i])] = 1;
            };
            auto e = [=] __device__(long long i, const int* cc, const int* pre) {
                const int nd = node[i];
                if (!(nd >= first && nd < first + cnt && c.split[nd])) return;
                const int q = cc[0] ? 0 : cc[1] ? 1 : cc[2] ? 2 : 3;
                rank[i] = pre[q];
                const int fi = nd - first;
                if (i == c.begin[nd])
                    for (int k = 0; k < 4; ++k) segP[4 * fi + k] = pre[k];
                if (i == c.end[nd] - 1)
                    for (int k = 0; k < 4; ++k) segE[4 * fi + k] = pre[k] + cc[k];
            };
            run_scan<4>(n, f, e, sc.tiles, sc.grand, s);
        }
        {  // child allocation: a scan over the frontier of non-empty quadrant counts
            const int* segP = sc.segP;
            const int* segE = sc.segE;
            int* kid = sc.kid;
            int* koff = sc.koff;
            auto f = [=] __device__(long long fi, int* cc) {
                if (!c.split[first + fi]) return;
                int m = 0;
                for (int k = 0; k < 4; ++k) m += (segE[4 * fi + k] - segP[4 * fi + k]) > 0;
                cc[0] = m;
            };
            auto e = [=] __device__(long long fi, const int* cc, const int* pre) {
                if (c.split[first + fi]) emit_children(c, first + int(fi), int(fi), next_id + pre[0], segP, segE, kid, koff);
            };
            run_scan<1>(cnt, f, e, sc.tiles, sc.grand, s);
            CSFS_CK(cudaMemcpyAsync(sc.counters.p, sc.grand.p, sizeof(int), cudaMemcpyDeviceToDevice, s));
        }
        // weights are not carried through the levels: gathered once via perm at the end
        // positions and weights are not carried through the levels: gathered once via perm
        PartArrays a{nullptr, nullptr, nullptr, t.xi, t.eta, nullptr, t.perm, t.node, nullptr, nullptr, nullptr,
                     t.xi2, t.eta2, nullptr, t.perm2, t.node2};
        k_scatter<<<gp, kThreads, 0, s>>>(n, first, cnt, c, a, t.rank, sc.segP, sc.kid, sc.koff);
        CSFS_LAUNCH_CHECK();
        swap_buf(t.xi, t.xi2);
        swap_buf(t.eta, t.eta2);
        swap_buf(t.perm, t.perm2);
        swap_buf(t.node, t.node2);

        finish_level(t, sc, next_id, sc.counters.p, 4 * nsplit, s);
        CSFS_CK(cudaMemcpyAsync(sc.host, sc.counters.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
        const int nnew = sc.host[0];
        nsplit = sc.host[1];
        t.ncl += nnew;
        t.level_first.push_back(next_id);
        t.level_count.push_back(nnew);
    }

    if (local) {
        k_fill_node<<<t.ncl, kThreads, 0, s>>>(t.ncl, t.begin, t.end, t.nchild, t.node);
        CSFS_LAUNCH_CHECK();
    }
    // ---- positions in tree order, then every cluster's radius ------------------------------
    k_gather_xyz<<<gp, kThreads, 0, s>>>(n, t.perm, xyz, t.px, t.py, t.pz);
    CSFS_LAUNCH_CHECK();
    finish_tree(t, w_in, n, cheb, s, w_ready);
}

// Radii, weights in tree order and proxy points of a tree whose particles are in tree order.
static void finish_tree(DeviceTree& t, const double* w_in, long long n, const Cheb& cheb, cudaStream_t s,
                        cudaEvent_t w_ready) {
    const int gp = ceil_div(n, kThreads);
    k_radius_leaf<<<ceil_div((long long)t.ncl * 32, 128), 128, 0, s>>>(t.ncl, t.nchild, t.begin, t.end, t.parent,
                                                                      t.px, t.py, t.pz, t.cx, t.cy, t.cz, t.rad);
    CSFS_LAUNCH_CHECK();
    k_rad_sqrt<<<ceil_div(t.ncl, kThreads), kThreads, 0, s>>>(t.ncl, t.rad);
    CSFS_LAUNCH_CHECK();

    // ---- weights in tree order (permute_weights, summation.cpp:98-104) ---------------------
    if (t.has_w) {
        // w_ready: the weights' host->device copy, overlapped with the levels above
        if (w_ready) CSFS_CK(cudaStreamWaitEvent(s, w_ready, 0));
        k_gather<<<gp, kThreads, 0, s>>>(n, t.perm, w_in, t.w);
        CSFS_LAUNCH_CHECK();
    }

    // ---- proxy points --------------------------------------------------------------------
    const long long nq = (long long)t.ncl * t.npp;
    t.qx.grow(nq);
    t.qy.grow(nq);
    t.qz.grow(nq);
    k_proxy<<<ceil_div(nq, kThreads), kThreads, 0, s>>>(t.ncl, t.np, cheb, t.face, t.xi0, t.xi1,
                                                          t.eta0, t.eta1, t.qx, t.qy, t.qz);
    CSFS_LAUNCH_CHECK();
    t.qrad.grow(std::max(t.ncl, 1));
    k_qrad<<<ceil_div((long long)t.ncl * 32, kThreads), kThreads, 0, s>>>(t.ncl, t.npp, t.cx, t.cy, t.cz, t.qx, t.qy,
                                                                          t.qz, t.qrad);
    CSFS_LAUNCH_CHECK();
}

// Grows the per-(cluster, quadrant) arrays with the cluster arrays, keeping `used` clusters.
static void reserve_quadrants(Scratch& sc, int cap, int used, cudaStream_t s) {
    if (cap <= sc.qcap) return;
    sc.qchild.grow_keep(4 * size_t(cap), 4 * size_t(used), s);
    sc.scnt.grow_keep(4 * size_t(cap), 4 * size_t(used), s);
    sc.sbnd.grow_keep(16 * size_t(cap), 16 * size_t(used), s);
    sc.qcap = cap;
}

void build_tree(DeviceTree& t, Scratch& sc, const double* xyz, const double* w_in, long long n, int degree,
                int n0, bool shrink, const Cheb& cheb, cudaStream_t s, cudaEvent_t w_ready) {
    {
        const char* e = std::getenv("CSFS_B200_TREE");  // read per call: tests flip it
        if (e && std::string(e) == "levels") {
            build_tree_levels(t, sc, xyz, w_in, n, degree, n0, shrink, cheb, s, w_ready);
            return;
        }
    }
    t.n = n;
    t.degree = degree;
    t.np = degree + 1;
    t.npp = t.np * t.np;
    t.n0 = n0;
    t.shrink = shrink;
    t.has_w = w_in != nullptr;
    t.ncl = 0;
    t.level_first.clear();
    t.level_count.clear();
    for (DevBuf<double>* b : {&t.px, &t.py, &t.pz, &t.xi, &t.eta, &sc.fxi, &sc.feta}) b->grow(n);
    for (DevBuf<int>* b : {&t.perm, &sc.lab, &sc.key, &sc.kb, &sc.vb, &sc.sorted}) b->grow(n);
    if (t.has_w) t.w.grow(n);
    const int ntiles = ceil_div(n, kRadixTile);
    sc.hist.grow(size_t(kRadixBins) * ntiles);
    sc.tiles.grow(scan_tile_ints((long long)kRadixBins * ntiles, 1));
    sc.grand.grow(8);
    sc.lev.grow(kMaxDepth + 4);
    sc.rcnt.grow(8);
    t.off_sphere.grow(1);
    // Cluster capacity per batch of speculatively enqueued levels: a level has at most 4x the
    // clusters of the one above and at most 4 floor(n / (n0 + 1)) (splitting clusters hold
    // > n0 particles each, disjointly); the batch stops at the depth a uniform distribution
    // reaches (+1) or when the bound would pass `budget`.
    const long long per_level = 4 * (n / (n0 + 1));
    const long long budget = 6 + 2 * per_level + 4096;
    int d_est = 0;
    while (d_est < kMaxDepth && 6.0 * std::pow(4.0, d_est) * std::max(n0, 1) < double(n)) ++d_est;

    LevelDesc* lev = reinterpret_cast<LevelDesc*>(sc.lev.p);
    t.reserve_clusters(64, s);
    reserve_quadrants(sc, t.cap, 0, s);
    ClusterPtrs c = cluster_ptrs(t);
    CSFS_CK(cudaMemsetAsync(t.off_sphere.p, 0, sizeof(int), s));
    k_root_init<<<1, 32, 0, s>>>(c, sc.rcnt);
    CSFS_LAUNCH_CHECK();
    const int grun = std::max(1, ceil_div(n, (long long)kTile));
    k_face_label<<<grun, kRunThreads, 0, s>>>(xyz, n, sc.fxi, sc.feta, sc.lab, t.off_sphere, sc.rcnt, t.bnd);
    CSFS_LAUNCH_CHECK();
    k_root_geom<<<1, 32, 0, s>>>(c, sc.rcnt, shrink, n0, lev, sc.scnt, sc.sbnd);
    CSFS_LAUNCH_CHECK();
    CSFS_CK(cudaMemcpyAsync(sc.host + kHostRoots, sc.rcnt.p, 6 * sizeof(int), cudaMemcpyDeviceToHost, s));

    // ---- levels (cluster_tree.cpp:87-141), no host round trip inside a batch -------------
    int d = 0;
    long long frontier = 6, used = 6;  // exact at the start of a batch
    const LevelDesc* hl = reinterpret_cast<const LevelDesc*>(sc.host + kHostLev);
    for (;;) {
        long long cap = used, fb = frontier;
        int d_end = d;
        std::vector<long long> fbound;  // frontier-size bound of each level of the batch
        for (;;) {  // levels d .. d_end allocate children at depths d+1 .. d_end+1
            const long long kids = std::min(4 * fb, per_level);
            if (d_end > d && (cap + kids > budget || d_end > d_est)) {
                --d_end;
                break;
            }
            fbound.push_back(fb);
            cap += kids;
            fb = kids;
            if (d_end + 1 >= kMaxDepth) break;
            ++d_end;
        }
        if (d_end < d) d_end = d;
        if (cap > INT_MAX / 16) throw std::invalid_argument("cluster tree too large");
        t.ncl = int(used);  // reserve_clusters keeps the first t.ncl clusters
        t.reserve_clusters(int(cap), s);
        reserve_quadrants(sc, t.cap, int(used), s);
        c = cluster_ptrs(t);
        sc.cbase.grow(size_t(*std::max_element(fbound.begin(), fbound.end())));
        for (int k = d; k <= d_end; ++k) {
            k_label<<<grun, kRunThreads, 0, s>>>(n, k, lev, c, sc.fxi, sc.feta, sc.lab, sc.qchild, sc.scnt, sc.sbnd);
            CSFS_LAUNCH_CHECK();
            k_alloc_scan<<<1, kAllocThreads, 0, s>>>(k, lev, c, sc.scnt, sc.cbase, t.cap);
            CSFS_LAUNCH_CHECK();
            k_alloc_fill<<<ceil_div(4 * fbound[k - d], kThreads), kThreads, 0, s>>>(k, lev, c, sc.scnt, sc.scnt,
                                                                                 sc.sbnd, sc.cbase, sc.qchild,
                                                                                 shrink, n0, sc.rcnt.p + 6);
            CSFS_LAUNCH_CHECK();
        }
        CSFS_CK(cudaMemcpyAsync(sc.host + kHostLev, sc.lev.p, (d_end + 2) * sizeof(LevelDesc),
                                cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaMemcpyAsync(sc.host + kHostRoots + 6, sc.rcnt.p + 6, sizeof(int), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
        for (int k = d; k <= d_end + 1; ++k)
            if (hl[k].ovf) throw std::runtime_error("cluster tree build: capacity bound violated");
        const LevelDesc nx = hl[d_end + 1];
        if (nx.nsplit == 0 || d_end + 1 >= kMaxDepth) {
            for (int k = 0; k <= d_end + 1 && hl[k].cnt > 0; ++k) {
                t.level_first.push_back(hl[k].first);
                t.level_count.push_back(hl[k].cnt);
                t.ncl = hl[k].first + hl[k].cnt;
            }
            break;
        }
        d = d_end + 1;
        frontier = nx.cnt;
        used = (long long)nx.first + nx.cnt;
    }
    t.root_count.assign(sc.host + kHostRoots, sc.host + kHostRoots + 6);

    // ---- one stable sort by leaf: the reference's order ----------------------------------
    const int gp = ceil_div(n, kThreads);
    k_leaf_key<<<gp, kThreads, 0, s>>>(n, sc.lab, sc.qchild, t.begin, sc.key);
    CSFS_LAUNCH_CHECK();
    int bits = 1;
    while (bits < 31 && (1LL << bits) < n) ++bits;
    // the keys are clusters' first slots: the low bits that are zero in every one of them
    // (8 on the L10 grid with 256-particle leaves) need no radix pass
    const unsigned orb = unsigned(sc.host[kHostRoots + 6]);
    const int low = orb ? std::min(__builtin_ctz(orb), bits - 1) : 0;
    const int* sorted = radix_sort_positions(n, bits, sc.key, sc.kb, sc.vb, sc.sorted, sc.hist, sc.tiles, sc.grand, s, low);
    k_gather_tree<<<gp, kThreads, 0, s>>>(n, sorted, sc.fxi, sc.feta, xyz, t.perm, t.xi, t.eta, t.px, t.py, t.pz);
    CSFS_LAUNCH_CHECK();
    finish_tree(t, w_in, n, cheb, s, w_ready);
}

void tree_proxy_radii(DeviceTree& t, cudaStream_t s) {
    t.qrad.grow(std::max(t.ncl, 1));
    if (t.ncl == 0) return;
    k_qrad<<<ceil_div((long long)t.ncl * 32, kThreads), kThreads, 0, s>>>(t.ncl, t.npp, t.cx, t.cy, t.cz, t.qx, t.qy,
                                                                          t.qz, t.qrad);
    CSFS_LAUNCH_CHECK();
}

bool device_equal(const void* a, const void* b, size_t bytes, Scratch& sc, cudaStream_t s) {
    if (a == b) return true;
    sc.counters.grow(8);
    CSFS_CK(cudaMemsetAsync(sc.counters.p + 4, 0, sizeof(int), s));
    const long long n = (long long)(bytes / 8);
    k_equal<<<592, 256, 0, s>>>(static_cast<const unsigned long long*>(a),
                                 static_cast<const unsigned long long*>(b), n, sc.counters.p + 4);
    CSFS_LAUNCH_CHECK();
    CSFS_CK(cudaMemcpyAsync(sc.host + 4, sc.counters.p + 4, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaStreamSynchronize(s));
    return sc.host[4] == 0;
}

// LIFO expansion order of the reference (cluster_tree.cpp:87-140): the stack starts as
// roots 0..5 (5 on top); popping a node that splits appends its children (ids =
// clusters.size() in quadrant order) and pushes them, so the last child is expanded next.
// Replaying that order over the GPU topology reproduces the reference ids exactly.
std::vector<int> reference_ids(const std::vector<int>& parent, const std::vector<int>& depth,
                               const std::vector<int4>& child, const std::vector<int>& nchild) {
    (void)parent;
    (void)depth;
    const int ncl = int(nchild.size());
    std::vector<int> ref(ncl, -1);
    for (int r = 0; r < 6 && r < ncl; ++r) ref[r] = r;
    int next = 6;
    std::vector<int> stack = {0, 1, 2, 3, 4, 5};
    while (!stack.empty()) {
        const int id = stack.back();
        stack.pop_back();
        const int4 ch = child[id];
        const int cs[4] = {ch.x, ch.y, ch.z, ch.w};
        for (int q = 0; q < nchild[id]; ++q) {
            ref[cs[q]] = next++;
            stack.push_back(cs[q]);
        }
    }
    return ref;
}

}  // namespace csfs_b200
