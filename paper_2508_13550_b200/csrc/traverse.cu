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

#include "engine.hpp"
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

__global__ void k_count(const int2* __restrict__ l, long long n, int key_off, int* cnt,
                        const TreeView T, const TreeView S, int type, unsigned long long* pairs) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long pe = 0;
    if (i < n) {
        const int2 ts = l[i];
        atomicAdd(&cnt[key_off + ts.x], 1);
        const long long nt = (type <= 1) ? (T.end[ts.x] - T.begin[ts.x]) : T.npp;
        const long long ns = (type == 0 || type == 2) ? (S.end[ts.y] - S.begin[ts.y]) : S.npp;
        pe = (unsigned long long)(nt * ns);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) pe += __shfl_xor_sync(0xffffffffu, pe, d);
    if ((threadIdx.x & 31) == 0 && pe) atomicAdd(&pairs[type], pe);
}

__global__ void k_fill(const int2* __restrict__ l, long long n, int key_off, int type,
                       const int* __restrict__ off, int* cur, long long* code) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int2 ts = l[i];
    const int key = key_off + ts.x;
    const int slot = off[key] + atomicAdd(&cur[key], 1);
    code[slot] = ((long long)type << 32) | (unsigned)ts.y;
}

// Per work item: canonical order of its sources, then segment descriptors.
// anchor = first target particle of the item's cluster (owner test for the multi-GPU
// partition), or -1 for depth-0 targets, which every rank evaluates redundantly.
__global__ void k_items(int n_items, int ncl_t, const int* __restrict__ keys,
                        const int* __restrict__ cnt, const int* __restrict__ off, long long* code,
                        int2* seg, int4* item, int* anchor, double* cost, const TreeView T,
                        const TreeView S) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    const int key = keys[i];
    const int b = off[key], n = cnt[key];
    long long* c = code + b;
    for (int a = 1; a < n; ++a) {  // insertion sort (lists per target are short)
        const long long v = c[a];
        int j = a - 1;
        while (j >= 0 && c[j] > v) {
            c[j + 1] = c[j];
            --j;
        }
        c[j + 1] = v;
    }
    long long src_pts = 0;
    for (int a = 0; a < n; ++a) {
        const int type = int(c[a] >> 32);
        const int s = int(c[a] & 0xffffffffll);
        if (type == 0 || type == 2) {
            seg[b + a] = make_int2(S.begin[s], S.end[s] - S.begin[s]);
            src_pts += S.end[s] - S.begin[s];
        } else {
            seg[b + a] = make_int2(s * S.npp, -S.npp);
            src_pts += S.npp;
        }
    }
    const int t = key < ncl_t ? key : key - ncl_t;
    const int tl = key < ncl_t ? T.end[t] - T.begin[t] : T.npp;
    if (key < ncl_t) item[i] = make_int4(T.begin[t], tl, b, b + n);
    else item[i] = make_int4(t * T.npp, -T.npp, b, b + n);
    anchor[i] = T.depth[t] == 0 ? -1 : T.begin[t];
    cost[i] = double(tl) * double(src_pts);
}

}  // namespace

void dual_traversal(const DeviceTree& tgt, const DeviceTree& src, double mac, int n0, Lists& L,
                    Scratch& sc, cudaStream_t s) {
    const TreeView T = tgt.view(), S = src.view();
    std::vector<int2> seeds;
    for (int t = 0; t < 6; ++t)
        for (int q = 0; q < 6; ++q)
            if (tgt.root_count[t] > 0 && src.root_count[q] > 0) seeds.push_back(make_int2(t, q));
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

void build_items(const DeviceTree& tgt, const DeviceTree& src, const Lists& L, Items& it, Scratch& sc,
                 cudaStream_t s) {
    const TreeView T = tgt.view(), S = src.view();
    const int ncl_t = tgt.ncl;
    const int nkeys = 2 * ncl_t;
    it.cnt.grow(nkeys);
    it.off.grow(nkeys);
    it.cur.grow(nkeys);
    it.keys.grow(nkeys);
    it.pairs.grow(4);
    CSFS_CK(cudaMemsetAsync(it.cnt.p, 0, nkeys * sizeof(int), s));
    CSFS_CK(cudaMemsetAsync(it.cur.p, 0, nkeys * sizeof(int), s));
    CSFS_CK(cudaMemsetAsync(it.pairs.p, 0, 4 * sizeof(unsigned long long), s));
    for (int k = 0; k < 4; ++k) {
        if (L.n[k] == 0) continue;
        k_count<<<ceil_div(L.n[k], kThreads), kThreads, 0, s>>>(L.l[k], L.n[k], k <= 1 ? 0 : ncl_t,
                                                                 it.cnt, T, S, k, it.pairs);
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
                                                                it.off, it.cur, it.code);
        CSFS_LAUNCH_CHECK();
    }
    if (it.n_items) {
        k_items<<<ceil_div(it.n_items, 128), 128, 0, s>>>(it.n_items, ncl_t, it.keys, it.cnt, it.off,
                                                         it.code, it.seg, it.item, it.anchor, it.cost,
                                                         T, S);
        CSFS_LAUNCH_CHECK();
    }
}

}  // namespace csfs_b200
