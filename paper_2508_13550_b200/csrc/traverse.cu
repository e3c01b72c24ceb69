// Dual tree traversal and work-item construction: the B200 restatement of
// dual_tree_traversal, well_separated* and group_by_target
// (/root/reference/proj/src/summation.cpp:89-96, 123-134, 163-203).
//
// Each (target, source) decision of the reference depends only on the pair itself, so
// the LIFO stack is replaced by frontier-synchronous expansion: classify every frontier
// pair, one 5-counter scan compacts the PP/PC/CP/CC emissions and the child pairs (K6).
// The resulting list SETS equal the reference's; only the emission
// order differs, and build_items() puts every target's sources into a canonical
// (list type, source id) order so results are deterministic run to run.
#include <algorithm>

#include <cstdio>
#include <cstdlib>

#include "engine.hpp"
#include "radix.cuh"
#include "scan.cuh"

namespace csfs_b200 {

namespace {

constexpr int kThreads = 256;

// well_separated (summation.cpp:123-126): R = |c0 - c1|, R > 0 && r0 + r1 < mac*R.
__device__ __forceinline__ bool well_separated(double x0, double y0, double z0, double r0, double x1,
                                               double y1, double z1, double r1, double mac) {
    const double dx = __dsub_rn(x0, x1), dy = __dsub_rn(y0, y1), dz = __dsub_rn(z0, z1);
    const double R = __dsqrt_rn(dot_ref(dx, dy, dz, dx, dy, dz));
    return R > 0.0 && __dadd_rn(r0, r1) < __dmul_rn(mac, R);
}

// 0 PP, 1 PC, 2 CP, 3 CC, 4 split source, 5 split target  (summation.cpp:177-200)
__device__ __forceinline__ int classify(const TreeView& T, const TreeView& S, int t, int s,
                                        double mac, int n0) {
    const int ct = T.end[t] - T.begin[t], cs = S.end[s] - S.begin[s];
    const bool big_t = ct > n0, big_s = cs > n0;
    const bool sep = well_separated(T.cx[t], T.cy[t], T.cz[t], T.rad[t], S.cx[s], S.cy[s], S.cz[s],
                                    S.rad[s], mac);
    if (sep && (big_t || big_s)) {
        if (!big_t && big_s) return 1;
        if (big_t && !big_s) return 2;
        return 3;
    }
    if (!sep && (big_t || big_s)) {
        const bool prefer_source = cs >= ct;
        const bool can_s = S.nchild[s] > 0, can_t = T.nchild[t] > 0;
        if (can_s && (prefer_source || !can_t)) return 4;
        if (can_t) return 5;
    }
    return 0;
}

// Can a list entry contain a pair with 1 - x.y < 1e-14 (the kernels' coincidence guard)?
// t / s: target / source cluster; *_prox: that side is the cluster's proxy points (else
// its particles).  Proven free (false) when the two point sets are separated by more than
// 1e-6 (chordal; the guard triggers below ~1.4e-7), either by the bounding spheres
// (centre distance minus particle / proxy radii) or, for particle sets on one cube face,
// by a gap of more than 1e-4 rad between their shrunk (xi, eta) boxes (the equiangular map
// shrinks distances by at most a small constant factor).  Same cluster of the same tree, or
// a tree holding points off the unit sphere (k_face flags it): always guarded.
__device__ __forceinline__ bool needs_guard(const TreeView& T, const TreeView& S, int t, bool t_prox, int s,
                                            bool s_prox) {
    if (T.px == S.px && t == s && !t_prox && !s_prox) return true;
    if (*T.off_sphere || *S.off_sphere) return true;  // the bounds below assume |x| = 1
    const double dx = T.cx[t] - S.cx[s], dy = T.cy[t] - S.cy[s], dz = T.cz[t] - S.cz[s];
    const double R = sqrt(dx * dx + dy * dy + dz * dz);
    const double rt = t_prox ? T.qrad[t] : T.rad[t], rs = s_prox ? S.qrad[s] : S.rad[s];
    if (R - rt - rs > 1e-6) return false;
    if (!t_prox && !s_prox && T.face[t] == S.face[s]) {
        const double gx = fmax(S.xi0[s] - T.xi1[t], T.xi0[t] - S.xi1[s]);
        const double ge = fmax(S.eta0[s] - T.eta1[t], T.eta0[t] - S.eta1[s]);
        if (fmax(gx, ge) > 1e-4) return false;
    }
    return true;
}

// Can the entry use the fused 1 - x.y (kernels_dev.cuh one_minus_dot<true>)?  Only when
// every pair of its point sets is more than kFuseGap apart (chordal, bounding spheres with
// the particle / proxy radii): then 1 - x.y >= kFuseGap^2/2 = 1e-5 and the fused form
// differs from the reference's unfused one by < 8e-11 relatively per pair (worst case).
// Unit vectors only (the distance bound uses |x| = 1).  The entry must also lie within one
// hemisphere — every pair less than kFuseMaxDist = 1.41 apart, so x.y >= 1 - 1.41^2/2 =
// 5.9e-3 > 0: the biharmonic functor's far form then knows u = (1 + x.y)/2 > 1/2 and runs
// the dilogarithm's reflection region without a select (kernels_dev.cuh dilog_far).  Only
// the few top-level CC entries between opposite faces fail it (0.1% of C5's evaluations).
__device__ __forceinline__ bool can_fuse(const TreeView& T, const TreeView& S, int t, bool t_prox, int s,
                                         bool s_prox) {
    if (*T.off_sphere || *S.off_sphere) return false;
    const double dx = T.cx[t] - S.cx[s], dy = T.cy[t] - S.cy[s], dz = T.cz[t] - S.cz[s];
    const double R = sqrt(dx * dx + dy * dy + dz * dz);
    const double rt = t_prox ? T.qrad[t] : T.rad[t], rs = s_prox ? S.qrad[s] : S.rad[s];
    return R - rt - rs > kFuseGap && R + rt + rs < kFuseMaxDist;
}

// A target cluster is ours when the range is everything, it is at depth 0 (every rank
// evaluates those), or its first particle lies in [own_b, own_e).
__device__ __forceinline__ bool owned_target(const TreeView& T, int t, long long own_b, long long own_e) {
    return own_b < 0 || T.depth[t] == 0 || (T.begin[t] >= own_b && T.begin[t] < own_e);
}

__global__ void k_count(const int2* __restrict__ l, long long n, int key_off, int* cnt,
                        const TreeView T, const TreeView S, int type, unsigned long long* pairs, long long own_b,
                        long long own_e) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long pe = 0;
    if (i < n) {
        const int2 ts = l[i];
        if (owned_target(T, ts.x, own_b, own_e)) atomicAdd(&cnt[key_off + ts.x], 1);
        const long long nt = (type <= 1) ? (T.end[ts.x] - T.begin[ts.x]) : T.npp;
        const long long ns = (type == 0 || type == 2) ? (S.end[ts.y] - S.begin[ts.y]) : S.npp;
        pe = (unsigned long long)(nt * ns);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) pe += __shfl_xor_sync(0xffffffffu, pe, d);
    if ((threadIdx.x & 31) == 0 && pe) atomicAdd(&pairs[type], pe);
}

__global__ void k_fill(const int2* __restrict__ l, long long n, int key_off, int type,
                       const int* __restrict__ off, int* cur, long long* code, const TreeView T, long long own_b,
                       long long own_e) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int2 ts = l[i];
    if (!owned_target(T, ts.x, own_b, own_e)) return;
    const int key = key_off + ts.x;
    const int slot = off[key] + atomicAdd(&cur[key], 1);
    code[slot] = ((long long)type << 32) | (unsigned)ts.y;
}

// Sorts the `n` unique 64-bit codes at c[0, n) ascending with the 32 lanes of a warp: a
// rank sort (every lane ranks its entries against all, then scatters) for n <= 128, else
// lane 0 insertion-sorts.  Ends with __syncwarp (the sorted codes are visible warp-wide).
__device__ __forceinline__ void warp_sort_unique(long long* c, int n, int lane) {
    constexpr unsigned kFull = 0xffffffffu;
    if (n <= 128) {
        long long my[4];
        int rank[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            my[q] = (lane + 32 * q < n) ? c[lane + 32 * q] : 0;
            rank[q] = 0;
        }
        for (int e = 0; e < n; ++e) {
            long long v = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const long long vq = __shfl_sync(kFull, my[q], e & 31);
                if ((e >> 5) == q) v = vq;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) rank[q] += (v < my[q]);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (lane + 32 * q < n) c[rank[q]] = my[q];
    } else if (lane == 0) {
        for (int a = 1; a < n; ++a) {
            const long long v = c[a];
            int j = a - 1;
            while (j >= 0 && c[j] > v) {
                c[j + 1] = c[j];
                --j;
            }
            c[j + 1] = v;
        }
    }
    __syncwarp();
}

// Per work item (one warp): canonical order of its sources, then segment descriptors.
// anchor = first target particle of the item's cluster (owner test for the multi-GPU
// partition), or -1 for depth-0 targets, which every rank evaluates redundantly.
__global__ void k_items(int n_items, int ncl_t, const int* __restrict__ keys,
                        const int* __restrict__ cnt, const int* __restrict__ off, long long* code,
                        int2* seg, int4* item, int* anchor, double* cost, const TreeView T,
                        const TreeView S) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= n_items) return;  // warp-uniform
    const int key = keys[i];
    const int b = off[key], n = cnt[key];
    long long* c = code + b;
    warp_sort_unique(c, n, lane);
    long long src_pts = 0;
    const int t = key < ncl_t ? key : key - ncl_t;
    const bool t_prox = key >= ncl_t;
    for (int a = lane; a < n; a += 32) {
        const int type = int(c[a] >> 32);
        const int s = int(c[a] & 0xffffffffll);
        const bool s_prox = !(type == 0 || type == 2);
        const int g = needs_guard(T, S, t, t_prox, s, s_prox) ? kSegGuard
                      : can_fuse(T, S, t, t_prox, s, s_prox)   ? kSegFused
                                                                : 0;
        if (!s_prox) {
            seg[b + a] = make_int2(S.begin[s], (S.end[s] - S.begin[s]) | g);
            src_pts += S.end[s] - S.begin[s];
        } else {
            seg[b + a] = make_int2(s * S.npp, -(S.npp | g));
            src_pts += S.npp;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) src_pts += __shfl_xor_sync(0xffffffffu, src_pts, d);
    if (lane == 0) {
        const int tl = key < ncl_t ? T.end[t] - T.begin[t] : T.npp;
        if (key < ncl_t) item[i] = make_int4(T.begin[t], tl, b, b + n);
        else item[i] = make_int4(t * T.npp, -T.npp, b, b + n);
        anchor[i] = T.depth[t] == 0 ? -1 : T.begin[t];
        cost[i] = double(tl) * double(src_pts);
    }
}

__device__ __forceinline__ int unit_of(const long long* ub, int nu, long long b) {
    int lo = 0, hi = nu;  // last unit with begin <= b
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (ub[mid] <= b) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Symmetric pairs (targets == sources, scalar kernels): K(t, s) = kSym K(s, t)
// bit-for-bit, so an interaction listed in BOTH directions is evaluated once by the tile
// kernel k_mutual (both segments are dropped from the list items):
//   * PP leaf pairs {A, B} (|A|, |B| <= 256): A's particles x B's particles;
//   * CC cluster pairs {A, B}: A's (p+1)^2 proxy points x B's, weighted by the proxy
//     weights; the partial sums land in the proxy potentials (the M2L-like far field).
// Only targets at depth >= 1 and pairs inside one partition unit qualify (unit_b: one unit
// = every pair), so the choice — and the summation order — is the same for every rank
// count of the partitioned path.  Pair ids: PP = (leaf t, leaf s), CC = (ncl + t, ncl + s)
// (the work-item keys), t < s.
__device__ __forceinline__ bool listed(const long long* code, const int* off, const int* cnt, int key,
                                       long long want) {
    int lo = off[key], hi = off[key] + cnt[key];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (code[mid] < want) lo = mid + 1;
        else hi = mid;
    }
    return lo < off[key] + cnt[key] && code[lo] == want;
}

__global__ void k_mutual_mark(int n_items, int ncl_t, const int* __restrict__ keys,
                              const int* __restrict__ cnt, const int* __restrict__ off,
                              const long long* __restrict__ code, int2* seg, int* mflag, int2* epair,
                              const long long* __restrict__ unit_b, int n_units, const TreeView T,
                              unsigned long long* saved) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;  // one warp per item
    unsigned long long sv = 0;
    if (i < n_items) {
        const int key = keys[i];
        const int b = off[key], n = cnt[key];
        for (int a = lane; a < n; a += 32) mflag[b + a] = 0;
        const bool leaf_item = key < ncl_t;
        const int t = leaf_item ? key : key - ncl_t;
        const int nt = leaf_item ? T.end[t] - T.begin[t] : T.npp;
        if (T.depth[t] >= 1 && (!leaf_item || nt <= 256)) {
            const int ut = unit_of(unit_b, n_units, T.begin[t]);
            const long long type = leaf_item ? 0 : 3;  // PP entries of leaf items, CC of cluster items
            for (int a = lane; a < n; a += 32) {
                const long long c = code[b + a];
                if ((c >> 32) != type) continue;  // sorted by (type, source)
                const int s = int(c & 0xffffffffll);
                const int ns = leaf_item ? T.end[s] - T.begin[s] : T.npp;
                if (s == t || ns > 256 || T.depth[s] < 1 || unit_of(unit_b, n_units, T.begin[s]) != ut) continue;
                const int key_s = leaf_item ? s : ncl_t + s;
                if (listed(code, off, cnt, key_s, (type << 32) | (long long)(unsigned)t)) {
                    seg[b + a].y = 0;  // both directions leave the list items
                    if (t < s) {
                        mflag[b + a] = 1;
                        epair[b + a] = make_int2(key, key_s);
                        sv += (unsigned long long)ns * nt;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, d);
    if ((threadIdx.x & 31) == 0 && sv) atomicAdd(saved, sv);
}

__global__ void k_mutual_count(int n_pairs, const int4* __restrict__ pair, const int* __restrict__ leaf_of_begin_unused,
                               int* mcnt, const int2* __restrict__ pl) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_pairs) return;
    atomicAdd(&mcnt[pl[p].x], 1);  // pair ids are the work-item keys (leaf or ncl + cluster)
    atomicAdd(&mcnt[pl[p].y], 1);
}

__global__ void k_mutual_fill(int n_pairs, const int4* __restrict__ pair, const long long* __restrict__ poff,
                              const int2* __restrict__ pl, const int* __restrict__ moff, int* mcur, long long* mlist) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_pairs) return;
    const int A = pl[p].x, B = pl[p].y;
    mlist[moff[A] + atomicAdd(&mcur[A], 1)] = poff[p];
    mlist[moff[B] + atomicAdd(&mcur[B], 1)] = poff[p] + seg_len(pair[p].y);
}

__global__ void k_mutual_sort(int ncl, const int* __restrict__ mcnt, const int* __restrict__ moff, long long* mlist) {
    const int X = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;  // one warp per key
    if (X >= ncl) return;
    warp_sort_unique(mlist + moff[X], mcnt[X], lane);
}

// One sweep of the dual traversal without a host round trip: every frontier pair is
// classified (classify = the reference's decision, summation.cpp:177-200); list entries and
// the split pairs' children are appended with warp-aggregated atomics (one atomic per warp
// and category).  The order of the entries is therefore arbitrary, but nothing depends on
// it: build_items sorts every work item's entries by (type, source) — the reference's
// accumulation order — and the lists are compared as sets.  Counters that pass a buffer's
// capacity raise *overflow (the caller then re-runs the synchronous sweep loop).
__global__ void __launch_bounds__(256) k_traverse_step(const TreeView T, const TreeView S, double mac, int n0,
                                                       const int2* __restrict__ fin, const int* __restrict__ fcnt,
                                                       int2* fout, int* fcnt_next, long long fcap, int2* l0, int2* l1,
                                                       int2* l2, int2* l3, int* lcnt, long long lcap, int* overflow) {
    // after an overflow the counts no longer describe the buffers: drain (the caller re-runs)
    const int F = *overflow ? 0 : int(min((long long)*fcnt, fcap));
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < F; base += stride) {
        const long long i = base + lane;
        int cat = -1;
        int2 p = make_int2(0, 0);
        if (i < F) {
            p = fin[i];
            cat = classify(T, S, p.x, p.y, mac, n0);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, cat == k);
            if (m == 0u) continue;
            const int leader = __ffs(m) - 1;
            int at = 0;
            if (lane == leader) at = atomicAdd(&lcnt[k], __popc(m));
            at = __shfl_sync(0xffffffffu, at, leader);
            if (cat == k) {
                const long long pos = (long long)at + __popc(m & ((1u << lane) - 1u));
                int2* l = k == 0 ? l0 : k == 1 ? l1 : k == 2 ? l2 : l3;
                if (pos < lcap) l[pos] = p;
                else *overflow = 1;
            }
        }
        const int nc = cat == 4 ? S.nchild[p.y] : cat == 5 ? T.nchild[p.x] : 0;
        int incl = nc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int at = 0;
        if (lane == 31) at = atomicAdd(fcnt_next, tot);
        at = __shfl_sync(0xffffffffu, at, 31);
        if (nc) {
            const long long pos = (long long)at + incl - nc;
            if (pos + nc > fcap) {
                *overflow = 1;
            } else {
                const int4 ch = cat == 4 ? S.child[p.y] : T.child[p.x];
                const int cs[4] = {ch.x, ch.y, ch.z, ch.w};
                for (int q = 0; q < nc; ++q) fout[pos + q] = cat == 4 ? make_int2(p.x, cs[q]) : make_int2(cs[q], p.y);
            }
        }
    }
}

}  // namespace

namespace {
// Each list entry's pair evaluations into its target's unit (depth-0 targets excluded:
// every rank evaluates them); lanes that share a unit combine first (per-entry costs are
// below 2^16, so 32 of them fit the 32-bit reduction), then one u64 atomic: exact.
__global__ void k_list_unit_costs(const int2* __restrict__ l, long long n, int type, const TreeView T,
                                  const TreeView S, const long long* __restrict__ ubeg, int nu,
                                  unsigned long long* ucost) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int u = -1;
    unsigned v = 0;
    if (i < n) {
        const int2 ts = l[i];
        if (T.depth[ts.x] > 0) {
            const long long a = T.begin[ts.x];
            int lo = 0, hi = nu;  // first unit beginning after a
            while (lo < hi) {
                const int m = (lo + hi) >> 1;
                if (ubeg[m] <= a) lo = m + 1;
                else hi = m;
            }
            u = lo - 1;
            const long long nt = (type <= 1) ? (T.end[ts.x] - T.begin[ts.x]) : T.npp;
            const long long ns = (type == 0 || type == 2) ? (S.end[ts.y] - S.begin[ts.y]) : S.npp;
            v = unsigned(nt * ns);
        }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, u);
    if (u < 0) return;
    const unsigned long long sum = __reduce_add_sync(peers, v);
    if ((peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&ucost[u], sum);
}
}  // namespace

void list_unit_costs(const DeviceTree& tgt, const DeviceTree& src, const Lists& L, const long long* ubeg, int nu,
                     unsigned long long* ucost, cudaStream_t s) {
    const TreeView T = tgt.view(), S = src.view();
    for (int k = 0; k < 4; ++k) {
        if (L.n[k] == 0 || nu <= 0) continue;
        k_list_unit_costs<<<ceil_div(L.n[k], 256), 256, 0, s>>>(L.l[k], L.n[k], k, T, S, ubeg, nu, ucost);
        CSFS_LAUNCH_CHECK();
    }
}

void partition_units(const DeviceTree& t, std::vector<long long>& ub, std::vector<long long>& ue, cudaStream_t s) {
    const int nfirst = t.depth_max() >= 1 ? t.level_first[1] + t.level_count[1] : 6;
    std::vector<int> b(nfirst), e(nfirst), nch(nfirst), dep(nfirst);
    // on the stream that built the tree (the legacy default stream does not order with it)
    CSFS_CK(cudaMemcpyAsync(b.data(), t.begin.p, nfirst * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaMemcpyAsync(e.data(), t.end.p, nfirst * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaMemcpyAsync(nch.data(), t.nchild.p, nfirst * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaMemcpyAsync(dep.data(), t.depth.p, nfirst * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaStreamSynchronize(s));
    std::vector<std::pair<long long, long long>> u;
    for (int i = 0; i < nfirst; ++i)
        if (e[i] > b[i] && (dep[i] == 1 || nch[i] == 0)) u.push_back({b[i], e[i]});
    std::sort(u.begin(), u.end());
    ub.clear();
    ue.clear();
    for (auto& p : u) {
        ub.push_back(p.first);
        ue.push_back(p.second);
    }
}

void build_mutual(const DeviceTree& tgt, Items& it, const std::vector<long long>& unit_begins, Scratch& sc,
                  cudaStream_t s) {
    const TreeView T = tgt.view();
    const int ncl = tgt.ncl;
    const long long ne = std::max<long long>(it.n_entries, 1);
    it.mflag.grow(ne);
    it.epair.grow(ne);
    it.mcnt.grow(2 * ncl);  // per work-item key: leaves [0, ncl), clusters' proxies [ncl, 2 ncl)
    it.moff.grow(2 * ncl);
    it.mcur.grow(2 * ncl);
    it.unit_b.grow(std::max<size_t>(unit_begins.size(), 1));
    it.n_mutual = 0;
    it.n_partial = 0;
    it.skipped_pairs = 0;
    if (it.n_items == 0) return;
    CSFS_CK(cudaMemcpyAsync(it.unit_b.p, unit_begins.data(), unit_begins.size() * sizeof(long long),
                            cudaMemcpyHostToDevice, s));
    CSFS_CK(cudaMemsetAsync(it.pairs.p + 4, 0, sizeof(unsigned long long), s));
    CSFS_CK(cudaMemsetAsync(it.mcnt.p, 0, 2 * ncl * sizeof(int), s));
    CSFS_CK(cudaMemsetAsync(it.mcur.p, 0, 2 * ncl * sizeof(int), s));
    const int nb = ceil_div((long long)it.n_items * 32, 128);
    k_mutual_mark<<<nb, 128, 0, s>>>(it.n_items, ncl, it.keys, it.cnt, it.off, it.code, it.seg, it.mflag, it.epair,
                                     it.unit_b, int(unit_begins.size()), T, it.pairs.p + 4);
    CSFS_LAUNCH_CHECK();
    // pair index and partial offset: 2-counter scan over entries, in 64 bits (the partial
    // buffer passes 2^31 doubles above ~45M points)
    sc.tiles64.grow(scan_tile_ints(it.n_entries, 2));
    sc.grand64.grow(2);
    {
        const int* mflag = it.mflag;
        const int2* ep = it.epair;
        auto f = [=] __device__(long long e, long long* c) {
            if (mflag[e]) {
                const int2 q = ep[e];
                c[0] = 1;
                c[1] = q.x >= ncl ? 2 * T.npp : (T.end[q.x] - T.begin[q.x]) + (T.end[q.y] - T.begin[q.y]);
            }
        };
        auto count_only = [=] __device__(long long, const long long*, const long long*) {};
        run_scan<2, long long>(it.n_entries, f, count_only, sc.tiles64.p, sc.grand64.p, s);
        long long tot[2] = {0, 0};
        CSFS_CK(cudaMemcpyAsync(tot, sc.grand64.p, 2 * sizeof(long long), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaMemcpyAsync(&it.skipped_pairs, it.pairs.p + 4, sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
        it.n_mutual = int(tot[0]);
        it.n_partial = tot[1];
        const int np = std::max(it.n_mutual, 1);
        it.mpair.grow(np);
        it.mpoff.grow(np);
        it.manchor.grow(np);
        it.mleaf.grow(np);
        it.mlist.grow(2 * size_t(np));
        int4* pair = it.mpair;
        long long* poff = it.mpoff;
        int* manchor = it.manchor;
        int2* leaf = it.mleaf;
        auto e = [=] __device__(long long i, const long long* c, const long long* pre) {
            if (!c[0]) return;
            const int p = int(pre[0]);
            const int2 q = ep[i];
            if (q.x >= ncl) {  // CC: proxy sets, negative lengths
                const int a = q.x - ncl, b = q.y - ncl;
                const int g = needs_guard(T, T, a, true, b, true) ? kSegGuard : 0;
                const int fz = !g && can_fuse(T, T, a, true, b, true) ? kSegFused : 0;
                pair[p] = make_int4(a * T.npp, -(T.npp | g), b * T.npp, -(T.npp | fz));
                manchor[p] = T.begin[a];
            } else {
                const int g = needs_guard(T, T, q.x, false, q.y, false) ? kSegGuard : 0;
                const int fz = !g && can_fuse(T, T, q.x, false, q.y, false) ? kSegFused : 0;
                pair[p] = make_int4(T.begin[q.x], (T.end[q.x] - T.begin[q.x]) | g, T.begin[q.y],
                                    (T.end[q.y] - T.begin[q.y]) | fz);
                manchor[p] = T.begin[q.x];
            }
            poff[p] = pre[1];
            leaf[p] = q;
        };
        if (it.n_mutual) run_scan<2, long long>(it.n_entries, f, e, sc.tiles64.p, sc.grand64.p, s);
    }
    if (it.n_mutual == 0) return;
    const int pb = ceil_div(it.n_mutual, 256);
    k_mutual_count<<<pb, 256, 0, s>>>(it.n_mutual, it.mpair, nullptr, it.mcnt, it.mleaf);
    CSFS_LAUNCH_CHECK();
    {
        const int* mcnt = it.mcnt;
        int* moff = it.moff;
        sc.tiles.grow(scan_tile_ints(2 * ncl, 1));
        auto f = [=] __device__(long long i, int* c) { c[0] = mcnt[i]; };
        auto e = [=] __device__(long long i, const int* c, const int* pre) { moff[i] = pre[0]; };
        run_scan<1>(2 * ncl, f, e, sc.tiles, sc.grand, s);
    }
    k_mutual_fill<<<pb, 256, 0, s>>>(it.n_mutual, it.mpair, it.mpoff, it.mleaf, it.moff, it.mcur, it.mlist);
    CSFS_LAUNCH_CHECK();
    k_mutual_sort<<<ceil_div((long long)2 * ncl * 32, 128), 128, 0, s>>>(2 * ncl, it.mcnt, it.moff, it.mlist);
    CSFS_LAUNCH_CHECK();
}

// The sweeps without host round trips: a pair (t, s) of the frontier at sweep k has
// depth(t) + depth(s) = k (every split deepens one side), so depth_t + depth_s + 1 sweeps
// drain it; all of them are enqueued at once and the counts are read back once.  Buffers
// are sized from their current capacity (grown by earlier calls) or a first guess; if a
// sweep overflows one, the caller falls back to the synchronous loop, which grows them.
static bool dual_traversal_async(const TreeView& T, const TreeView& S, int depth_sum, double mac, int n0,
                                 const std::vector<int2>& seeds, long long guess, Lists& L, Scratch& sc,
                                 cudaStream_t s) {
    const int K = depth_sum + 1;
    long long lcap = guess;
    for (int k = 0; k < 4; ++k) lcap = std::max<long long>(lcap, (long long)L.l[k].cap);
    for (int k = 0; k < 4; ++k) L.l[k].grow(size_t(lcap));
    for (int k = 0; k < 4; ++k) lcap = std::min<long long>(lcap, (long long)L.l[k].cap);
    long long fcap = std::max<long long>(2 * guess, (long long)std::max(L.front.cap, L.front2.cap));
    L.front.grow(size_t(fcap));
    L.front2.grow(size_t(fcap));
    fcap = std::min<long long>((long long)L.front.cap, (long long)L.front2.cap);
    L.cnt.grow(size_t(K + 8));
    int* fc = L.cnt.p;            // [0, K]: frontier sizes per sweep
    int* lc = L.cnt.p + K + 1;    // 4 list counts
    int* ovf = L.cnt.p + K + 5;   // overflow flag
    CSFS_CK(cudaMemsetAsync(L.cnt.p, 0, (K + 8) * sizeof(int), s));
    sc.host[32] = int(seeds.size());
    CSFS_CK(cudaMemcpyAsync(fc, sc.host + 32, sizeof(int), cudaMemcpyHostToDevice, s));
    CSFS_CK(cudaMemcpyAsync(L.front.p, seeds.data(), seeds.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
    int dev = 0, sms = 0;
    CSFS_CK(cudaGetDevice(&dev));
    CSFS_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    for (int k = 0; k < K; ++k) {
        const int2* fin = (k & 1) ? L.front2.p : L.front.p;
        int2* fout = (k & 1) ? L.front.p : L.front2.p;
        k_traverse_step<<<4 * sms, 256, 0, s>>>(T, S, mac, n0, fin, fc + k, fout, fc + k + 1, fcap, L.l[0], L.l[1],
                                                L.l[2], L.l[3], lc, lcap, ovf);
        CSFS_LAUNCH_CHECK();
    }
    CSFS_CK(cudaMemcpyAsync(sc.host, fc + K, 6 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaStreamSynchronize(s));
    if (sc.host[5] != 0 || sc.host[0] != 0) return false;  // overflow, or pairs left (cannot happen)
    for (int k = 0; k < 4; ++k) L.n[k] = sc.host[1 + k];
    return true;
}

void dual_traversal(const DeviceTree& tgt, const DeviceTree& src, double mac, int n0, Lists& L,
                    Scratch& sc, cudaStream_t s) {
    const TreeView T = tgt.view(), S = src.view();
    std::vector<int2> seeds;
    for (int t = 0; t < 6; ++t)
        for (int q = 0; q < 6; ++q)
            if (tgt.root_count[t] > 0 && src.root_count[q] > 0) seeds.push_back(make_int2(t, q));
    for (int k = 0; k < 4; ++k) L.n[k] = 0;
    if (seeds.empty()) return;
    // first-guess buffer size; CSFS_B200_TRAVERSAL_GUESS overrides it (the tests force the
    // overflow fallback with a tiny one)
    static const long long guess_env = [] {
        const char* e = std::getenv("CSFS_B200_TRAVERSAL_GUESS");
        return e ? std::atoll(e) : 0LL;
    }();
    const long long guess = guess_env > 0 ? guess_env : 16LL * (tgt.ncl + src.ncl) + 4096;
    L.fallback = false;
    if (dual_traversal_async(T, S, tgt.depth_max() + src.depth_max(), mac, n0, seeds, guess, L, sc, s)) return;
    L.fallback = true;
    for (int k = 0; k < 4; ++k) L.n[k] = 0;
    long long F = (long long)seeds.size();
    L.front.grow(std::max<long long>(F, 64));
    if (F) CSFS_CK(cudaMemcpyAsync(L.front.p, seeds.data(), F * sizeof(int2), cudaMemcpyHostToDevice, s));
    sc.grand.grow(8);
    while (F > 0) {
        for (int k = 0; k < 4; ++k) L.l[k].grow_keep(size_t(L.n[k] + F), size_t(L.n[k]), s);
        L.front2.grow(size_t(4 * F));
        sc.tiles.grow(scan_tile_ints(F, 5));
        const int2* fin = L.front;
        int2* fout = L.front2;
        int2* l0 = L.l[0];
        int2* l1 = L.l[1];
        int2* l2 = L.l[2];
        int2* l3 = L.l[3];
        const long long b0 = L.n[0], b1 = L.n[1], b2 = L.n[2], b3 = L.n[3];
        auto f = [=] __device__(long long i, int* c) {
            const int2 p = fin[i];
            const int cat = classify(T, S, p.x, p.y, mac, n0);
            if (cat < 4) c[cat] = 1;
            else c[4] = (cat == 4) ? S.nchild[p.y] : T.nchild[p.x];
        };
        auto e = [=] __device__(long long i, const int* c, const int* pre) {
            const int2 p = fin[i];
            const int cat = classify(T, S, p.x, p.y, mac, n0);
            switch (cat) {
                case 0: l0[b0 + pre[0]] = p; break;
                case 1: l1[b1 + pre[1]] = p; break;
                case 2: l2[b2 + pre[2]] = p; break;
                case 3: l3[b3 + pre[3]] = p; break;
                case 4: {
                    const int4 ch = S.child[p.y];
                    const int cs[4] = {ch.x, ch.y, ch.z, ch.w};
                    for (int q = 0; q < c[4]; ++q) fout[pre[4] + q] = make_int2(p.x, cs[q]);
                    break;
                }
                default: {
                    const int4 ch = T.child[p.x];
                    const int cs[4] = {ch.x, ch.y, ch.z, ch.w};
                    for (int q = 0; q < c[4]; ++q) fout[pre[4] + q] = make_int2(cs[q], p.y);
                    break;
                }
            }
        };
        run_scan<5>(F, f, e, sc.tiles, sc.grand, s);
        CSFS_CK(cudaMemcpyAsync(sc.host, sc.grand.p, 5 * sizeof(int), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
        for (int k = 0; k < 4; ++k) L.n[k] += sc.host[k];
        F = sc.host[4];
        std::swap(L.front.p, L.front2.p);
        std::swap(L.front.cap, L.front2.cap);
    }
}

namespace {
// Item sort key: the cost's double bit pattern (monotone for non-negative doubles) cut to
// the exponent + kCostMant mantissa bits.  Coarse buckets (2 bits: costs to within 25%)
// keep the items of a bucket in key (tree) order, so neighbouring items still run close
// in time and share their sources in L2: C5 k_interact DRAM reads 3.37 -> 2.65 GB at 8 -> 2
// bits, same time; 7 key bits, one radix pass.
#ifndef CSFS_COST_KEY_BITS
#define CSFS_COST_KEY_BITS 2
#endif
constexpr int kCostMant = CSFS_COST_KEY_BITS;  // mantissa bits kept: cost buckets of 2^-kCostMant
__global__ void k_cost_key(int n, const double* __restrict__ cost, int* key) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long b = (long long)(__double_as_longlong(cost[i]) >> (52 - kCostMant)) - (1023ll << kCostMant);
    const long long top = (32ll << kCostMant) - 1;
    key[i] = int(b < 0 ? 0 : (b > top ? top : b));
}

__global__ void k_permute_items(int n, const int* __restrict__ order, const int* __restrict__ keys,
                                const int4* __restrict__ item, const int* __restrict__ anchor,
                                const double* __restrict__ cost, int* keys2, int4* item2, int* anchor2,
                                double* cost2) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int i = order[j];
    keys2[j] = keys[i];
    item2[j] = item[i];
    anchor2[j] = anchor[i];
    cost2[j] = cost[i];
}
}  // namespace

// Items in ascending cost (stable: key order among equal costs).  k_interact hands them out
// back to front, so the most expensive go first and the kernel's tail is made of the
// cheapest (longest-processing-time-first); nothing else depends on the item order — every
// item owns its outputs and sums them in a fixed order.
void order_items_by_cost(Items& it, cudaStream_t s) {
    const int n = it.n_items;
    if (n <= 1) return;
    for (DevBuf<int>* b : {&it.skey, &it.skb, &it.svb, &it.sout, &it.keys2, &it.anchor2}) b->grow(n);
    it.item2.grow(n);
    it.cost2.grow(n);
    const int ntiles = ceil_div(n, kRadixTile);
    it.shist.grow(size_t(kRadixBins) * ntiles);
    it.stiles.grow(scan_tile_ints((long long)kRadixBins * ntiles, 1));
    it.sgrand.grow(8);
    k_cost_key<<<ceil_div(n, 256), 256, 0, s>>>(n, it.cost, it.skey);
    CSFS_LAUNCH_CHECK();
    const int* order = radix_sort_positions(n, 5 + kCostMant, it.skey, it.skb, it.svb, it.sout, it.shist, it.stiles, it.sgrand, s);
    k_permute_items<<<ceil_div(n, 256), 256, 0, s>>>(n, order, it.keys, it.item, it.anchor, it.cost, it.keys2,
                                                     it.item2, it.anchor2, it.cost2);
    CSFS_LAUNCH_CHECK();
    std::swap(it.keys.p, it.keys2.p);
    std::swap(it.keys.cap, it.keys2.cap);
    std::swap(it.item.p, it.item2.p);
    std::swap(it.item.cap, it.item2.cap);
    std::swap(it.anchor.p, it.anchor2.p);
    std::swap(it.anchor.cap, it.anchor2.cap);
    std::swap(it.cost.p, it.cost2.p);
    std::swap(it.cost.cap, it.cost2.cap);
}

void build_items(const DeviceTree& tgt, const DeviceTree& src, const Lists& L, Items& it, Scratch& sc,
                 cudaStream_t s, long long own_b, long long own_e) {
    const TreeView T = tgt.view(), S = src.view();
    const int ncl_t = tgt.ncl;
    const int nkeys = 2 * ncl_t;
    it.cnt.grow(nkeys);
    it.off.grow(nkeys);
    it.cur.grow(nkeys);
    it.keys.grow(nkeys);
    it.pairs.grow(8);
    CSFS_CK(cudaMemsetAsync(it.cnt.p, 0, nkeys * sizeof(int), s));
    CSFS_CK(cudaMemsetAsync(it.cur.p, 0, nkeys * sizeof(int), s));
    CSFS_CK(cudaMemsetAsync(it.pairs.p, 0, 4 * sizeof(unsigned long long), s));
    for (int k = 0; k < 4; ++k) {
        if (L.n[k] == 0) continue;
        k_count<<<ceil_div(L.n[k], kThreads), kThreads, 0, s>>>(L.l[k], L.n[k], k <= 1 ? 0 : ncl_t,
                                                                 it.cnt, T, S, k, it.pairs, own_b, own_e);
        CSFS_LAUNCH_CHECK();
    }
    sc.tiles.grow(scan_tile_ints(nkeys, 2));
    {
        const int* cnt = it.cnt;
        int* off = it.off;
        int* keys = it.keys;
        auto f = [=] __device__(long long i, int* c) {
            c[0] = cnt[i];
            c[1] = cnt[i] > 0;
        };
        auto e = [=] __device__(long long i, const int* c, const int* pre) {
            off[i] = pre[0];
            if (c[1]) keys[pre[1]] = int(i);
        };
        run_scan<2>(nkeys, f, e, sc.tiles, sc.grand, s);
    }
    CSFS_CK(cudaMemcpyAsync(sc.host, sc.grand.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaMemcpyAsync(it.pair_evals, it.pairs.p, 4 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaStreamSynchronize(s));
    it.n_entries = sc.host[0];
    it.n_items = sc.host[1];
    it.code.grow(std::max<long long>(it.n_entries, 1));
    it.seg.grow(std::max<long long>(it.n_entries, 1));
    it.item.grow(std::max(it.n_items, 1));
    it.anchor.grow(std::max(it.n_items, 1));
    it.cost.grow(std::max(it.n_items, 1));
    for (int k = 0; k < 4; ++k) {
        if (L.n[k] == 0) continue;
        k_fill<<<ceil_div(L.n[k], kThreads), kThreads, 0, s>>>(L.l[k], L.n[k], k <= 1 ? 0 : ncl_t, k,
                                                                it.off, it.cur, it.code, T, own_b, own_e);
        CSFS_LAUNCH_CHECK();
    }
    if (it.n_items) {
        k_items<<<ceil_div((long long)it.n_items * 32, 128), 128, 0, s>>>(it.n_items, ncl_t, it.keys, it.cnt, it.off,
                                                         it.code, it.seg, it.item, it.anchor, it.cost,
                                                         T, S);
        CSFS_LAUNCH_CHECK();
        order_items_by_cost(it, s);
    }
}

}  // namespace csfs_b200
