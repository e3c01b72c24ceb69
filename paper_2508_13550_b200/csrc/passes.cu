// Upward (P2M + M2M) and downward (L2L + L2P) passes: the B200 restatement of
// upward_pass / downward_pass (/root/reference/proj/src/cluster_tree.cpp:163-220, 228-283)
// and transfer_matrix (:16-25).
//
// These are HBM/latency-bound tensor-product barycentric contractions over (p+1)^2
// Chebyshev-2 proxy grids (K7, K8, K12, K13 in SURVEY.md §2.3).  One CTA per cluster;
// the per-particle 1-D bases live in shared memory, every output coefficient is owned by
// exactly one thread (deterministic, no atomics).  The leaf P2M forms a = w*Lx[k1] like
// the reference and accumulates a*Ly[k2] with FMAs into four interleaved partial sums per
// coefficient (fixed order; roundoff-level difference from the reference's serial sum,
// within the 1e-12 proxy-weight bar); L2L is done separably.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "engine.hpp"
#include "fastmath.cuh"

namespace csfs_b200 {

namespace {

constexpr int kPassThreads = 128;
constexpr int kP2mChunk = kPassThreads;  // particles per P2M chunk: one per thread

// Leaf P2M (cluster_tree.cpp:180-191).  Internal clusters are written by k_m2m.
// Which clusters a pass touches: mode 0 all, 1 owned at depth >= 1, 2 depth 0 only.
__device__ __forceinline__ bool selected(const TreeView& t, int c, int mode, Own own) {
    if (mode == 0) return true;
    if (mode == 2) return t.depth[c] == 0;
    return t.depth[c] >= 1 && t.begin[c] >= own.b && t.begin[c] < own.e;
}

template <int NP>
__global__ void __launch_bounds__(kPassThreads)
    k_p2m(TreeView t, Cheb cheb, const double* __restrict__ w, double* __restrict__ qw, int mode,
          Own own) {
    extern __shared__ double sm[];
    const int c = blockIdx.x;
    if (t.nchild[c] > 0 || !selected(t, c, mode, own)) return;
    const int np = NP > 0 ? NP : cheb.np, npp = np * np;
    double* WL = sm;                    // kP2mChunk x np   (w * Lx)
    double* LY = sm + kP2mChunk * np;   // kP2mChunk x np
    const int b = t.begin[c], e = t.end[c];
    const double x0 = t.xi0[c], x1 = t.xi1[c], e0 = t.eta0[c], e1 = t.eta1[c];
    const double xm = __dmul_rn(0.5, __dadd_rn(x0, x1)), xh = __dmul_rn(0.5, __dsub_rn(x1, x0));
    const double em = __dmul_rn(0.5, __dadd_rn(e0, e1)), eh = __dmul_rn(0.5, __dsub_rn(e1, e0));
    constexpr int M = NP > 0 ? NP : kMaxNp;
    constexpr int kOut = (M * M + kPassThreads - 1) / kPassThreads;  // outputs per thread
    double acc[kOut][4];  // 4 interleaved partial sums per output (ILP on the add chain)
#pragma unroll
    for (int q = 0; q < kOut; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[q][r] = 0.0;
    for (int base = b; base < e; base += kP2mChunk) {
        const int m = min(kP2mChunk, e - base);
        for (int j = threadIdx.x; j < m; j += kPassThreads) {  // one particle per thread
            double lx[M], ly[M];
            bary1d_fast<NP>(cheb, ref_coord(t.xi[base + j], xm, xh), lx);
            bary1d_fast<NP>(cheb, ref_coord(t.eta[base + j], em, eh), ly);
            const double wt = w[base + j];
#pragma unroll
            for (int k = 0; k < M; ++k)
                if (k < np) {
                    WL[j * np + k] = __dmul_rn(wt, lx[k]);
                    LY[j * np + k] = ly[k];
                }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kOut; ++q) {
            const int o = threadIdx.x + q * kPassThreads;
            if (o < npp) {
                const int k1 = o / np, k2 = o % np;
                int j = 0;
                for (; j + 4 <= m; j += 4)
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        acc[q][r] = fma(WL[(j + r) * np + k1], LY[(j + r) * np + k2], acc[q][r]);
                for (; j < m; ++j) acc[q][j & 3] = fma(WL[j * np + k1], LY[j * np + k2], acc[q][j & 3]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < kOut; ++q) {
        const int o = threadIdx.x + q * kPassThreads;
        if (o < npp) qw[(long long)c * npp + o] = (acc[q][0] + acc[q][1]) + (acc[q][2] + acc[q][3]);
    }
}

// Leaf P2M with register blocking (the default for compile-time degrees): the bases of a
// chunk of 128 particles are staged as above; then thread (s, k1) — S particle subsets x
// NP rows — accumulates the whole row k1 (NP outputs in registers) over the particles
// j = s, s + S, ...: per particle one shared load of w Lx[k1] and NP/2 two-wide loads of
// the particle's Ly row (shared by the NP threads of subset s) for NP FMAs, instead of two
// shared loads per FMA.  The S partial rows are added in fixed subset order at the end
// (deterministic; roundoff-level difference from the reference's serial sum, within the
// 1e-12 proxy-weight bar).
template <int NP>
__global__ void __launch_bounds__(kPassThreads)
    k_p2m_rb(TreeView t, Cheb cheb, const double* __restrict__ w, double* __restrict__ qw, int mode, Own own) {
    constexpr int S = kPassThreads / NP;  // particle subsets
    constexpr int LDY = NP + 1;           // Ly row stride: 16-byte aligned pairs
    constexpr int NPP = NP * NP;
    __shared__ double WL[kP2mChunk * NP];
    __shared__ __align__(16) double LY[kP2mChunk * LDY];
    __shared__ double red[S * NPP];
    const int c = blockIdx.x;
    if (t.nchild[c] > 0 || !selected(t, c, mode, own)) return;
    const int b = t.begin[c], e = t.end[c];
    const double x0 = t.xi0[c], x1 = t.xi1[c], e0 = t.eta0[c], e1 = t.eta1[c];
    const double xm = __dmul_rn(0.5, __dadd_rn(x0, x1)), xh = __dmul_rn(0.5, __dsub_rn(x1, x0));
    const double em = __dmul_rn(0.5, __dadd_rn(e0, e1)), eh = __dmul_rn(0.5, __dsub_rn(e1, e0));
    const int sub = threadIdx.x / NP, k1 = threadIdx.x - sub * NP;
    const bool row = sub < S;
    double acc[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) acc[k] = 0.0;
    for (int base = b; base < e; base += kP2mChunk) {
        const int m = min(kP2mChunk, e - base);
        for (int j = threadIdx.x; j < m; j += kPassThreads) {  // one particle per thread
            double lx[NP], ly[NP];
            bary1d_fast<NP>(cheb, ref_coord(t.xi[base + j], xm, xh), lx);
            bary1d_fast<NP>(cheb, ref_coord(t.eta[base + j], em, eh), ly);
            const double wt = w[base + j];
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                WL[j * NP + k] = __dmul_rn(wt, lx[k]);
                LY[j * LDY + k] = ly[k];
            }
        }
        __syncthreads();
        if (row)
            for (int j = sub; j < m; j += S) {
                const double a = WL[j * NP + k1];
                const double2* y2 = reinterpret_cast<const double2*>(LY + j * LDY);
#pragma unroll
                for (int k = 0; k + 1 < NP; k += 2) {
                    const double2 v = y2[k >> 1];
                    acc[k] = fma(a, v.x, acc[k]);
                    acc[k + 1] = fma(a, v.y, acc[k + 1]);
                }
                if (NP & 1) acc[NP - 1] = fma(a, LY[j * LDY + NP - 1], acc[NP - 1]);
            }
        __syncthreads();
    }
    if (row)
#pragma unroll
        for (int k = 0; k < NP; ++k) red[sub * NPP + k1 * NP + k] = acc[k];
    __syncthreads();
    for (int o = threadIdx.x; o < NPP; o += kPassThreads) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < S; ++q) v += red[q * NPP + o];
        qw[(long long)c * NPP + o] = v;
    }
}

// The same leaf P2M on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64): per leaf the
// proxy weights are the GEMM  pw = (w Lx)^T Ly  over its particles, (np x m) (m x np),
// padded to 8 x 8 output tiles (np <= 8: one tile; np <= 16: 2 x 2, one warp each), K in
// steps of 4 particles.  The bases are staged per 128-particle chunk exactly as above
// (zero-padded to the tile edge); each lane feeds one A and one B element per MMA.
// Products are accumulated in the MMA's fused order (roundoff-level difference).
// Selected with CSFS_B200_P2M=dmma — the A/B of DESIGN.md §3 (profiles/r02_p2m_dmma_vs_fma).
template <int NP>
__global__ void __launch_bounds__(kPassThreads)
    k_p2m_dmma(TreeView t, Cheb cheb, const double* __restrict__ w, double* __restrict__ qw, int mode,
               Own own) {
    static_assert(NP > 0 && NP <= 16, "tile-padded degrees only");
    constexpr int NPAD = NP <= 8 ? 8 : 16;
    constexpr int TILES = NPAD / 8;  // per axis
    // row stride: a fragment load touches 4 particle rows x 8 coefficients; rows 24 doubles
    // apart fall in alternate bank halves (2 wavefronts, the minimum for 32 doubles)
    constexpr int LDW = NPAD == 16 ? 24 : 8;
    __shared__ double WL[kP2mChunk * LDW];  // [particle][k1], zero-padded
    __shared__ double LY[kP2mChunk * LDW];  // [particle][k2]
    const int c = blockIdx.x;
    if (t.nchild[c] > 0 || !selected(t, c, mode, own)) return;
    const int b = t.begin[c], e = t.end[c];
    const double x0 = t.xi0[c], x1 = t.xi1[c], e0 = t.eta0[c], e1 = t.eta1[c];
    const double xm = __dmul_rn(0.5, __dadd_rn(x0, x1)), xh = __dmul_rn(0.5, __dsub_rn(x1, x0));
    const double em = __dmul_rn(0.5, __dadd_rn(e0, e1)), eh = __dmul_rn(0.5, __dsub_rn(e1, e0));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool mma_warp = warp < TILES * TILES;
    const int r0 = (warp / TILES) * 8, c0 = (warp % TILES) * 8;  // output tile origin (k1, k2)
    const int arow = lane >> 2, acol = lane & 3;                 // fragment coordinates
    // C/D fragments (row arow, cols 2 acol, +1): 4 independent accumulator chains over the
    // K steps (the MMA latency, not its issue, bounds one chain), summed in fixed order
    double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
    for (int base = b; base < e; base += kP2mChunk) {
        const int m = min(kP2mChunk, e - base);
        for (int j = threadIdx.x; j < kP2mChunk; j += kPassThreads) {
            double lx[NP], ly[NP];
            double wt = 0.0;
            if (j < m) {
                bary1d_fast<NP>(cheb, ref_coord(t.xi[base + j], xm, xh), lx);
                bary1d_fast<NP>(cheb, ref_coord(t.eta[base + j], em, eh), ly);
                wt = w[base + j];
            }
#pragma unroll
            for (int k = 0; k < NPAD; ++k) {
                WL[j * LDW + k] = (j < m && k < NP) ? __dmul_rn(wt, lx[k < NP ? k : 0]) : 0.0;
                LY[j * LDW + k] = (j < m && k < NP) ? ly[k < NP ? k : 0] : 0.0;
            }
        }
        __syncthreads();
        if (mma_warp) {
            const int steps = (m + 15) >> 4;  // 4 K-steps of 4 particles per iteration (zero-padded rows)
            for (int s = 0; s < steps; ++s) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int tp = 16 * s + 4 * u + acol;  // particle of this lane's A row / B column
                    const double a = WL[tp * LDW + r0 + arow];
                    const double bb = LY[tp * LDW + c0 + arow];
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                 : "+d"(d0[u]), "+d"(d1[u]) : "d"(a), "d"(bb));
                }
            }
        }
        __syncthreads();
    }
    if (mma_warp) {
        const int k1 = r0 + arow, k2 = c0 + 2 * acol;
        const double s0 = (d0[0] + d0[1]) + (d0[2] + d0[3]), s1 = (d1[0] + d1[1]) + (d1[2] + d1[3]);
        if (k1 < NP && k2 < NP) qw[(long long)c * NP * NP + k1 * NP + k2] = s0;
        if (k1 < NP && k2 + 1 < NP) qw[(long long)c * NP * NP + k1 * NP + k2 + 1] = s1;
    }
}

// Transfer matrix columns: At[m*np + k] = L^parent_k(child node m)  (transfer_matrix, :16-25).
__device__ void transfer_cols(const Cheb& cheb, double pmid, double phalf, double cmid,
                              double chalf, int m, double* At) {
    const double node = __dadd_rn(cmid, __dmul_rn(chalf, cheb.nodes[m]));
    const double xhat = phalf > 0.0 ? __ddiv_rn(__dsub_rn(node, pmid), phalf) : 0.0;
    bary1d(cheb, xhat, At + m * cheb.np);
}

__device__ __forceinline__ void mid_half(double a0, double a1, double& mid, double& half) {
    mid = __dmul_rn(0.5, __dadd_rn(a0, a1));
    half = __dmul_rn(0.5, __dsub_rn(a1, a0));
}

// Both transfer matrices of one (parent, child) pair with a whole thread group at work:
// At[r*np + k] = L^parent_k(child node r) for the xi axis (rows r < np: Ax) and the eta axis
// (rows np .. 2np-1: Ae = At + np*np).  The same operations as transfer_cols / bary1d, bit for
// bit — one division per entry in parallel, each row's denominator summed in node order by
// one thread — instead of 2np threads each walking a row of np divisions while the others
// wait (the barrier stalls of k_l2l / k_m2m4, ncu round 2).  EVERY thread of the CTA calls it
// (four CTA barriers); `active`: the thread's group has a pair; lt, nthr: the thread's index
// in its group and the group size; aux: 2np doubles, hit: 2np ints of shared memory per group.
__device__ __forceinline__ void transfer_pair(const Cheb& cheb, bool active, int lt, int nthr, double pxm, double pxh,
                                              double pem, double peh, double cxm, double cxh, double cem, double ceh,
                                              double* At, double* aux, int* hit) {
    const int np = cheb.np;
    if (active && lt < 2 * np) {  // the child nodes in the parent's reference interval
        const bool xa = lt < np;
        const int m = xa ? lt : lt - np;
        const double node = __dadd_rn(xa ? cxm : cem, __dmul_rn(xa ? cxh : ceh, cheb.nodes[m]));
        const double ph = xa ? pxh : peh;
        aux[lt] = ph > 0.0 ? __ddiv_rn(__dsub_rn(node, xa ? pxm : pem), ph) : 0.0;
        hit[lt] = np;
    }
    __syncthreads();
    if (active)
        for (int o = lt; o < 2 * np * np; o += nthr) {
            const int r = o / np, k = o - r * np;
            const double d = __dsub_rn(aux[r], cheb.nodes[k]);
            if (fabs(d) < kNodeTol) atomicMin(&hit[r], k);  // the first node hit (interpolation.cpp:28-33)
            At[o] = __ddiv_rn(cheb.weights[k], d);
        }
    __syncthreads();
    if (active && lt < 2 * np && hit[lt] == np) {
        double denom = 0.0;
        for (int k = 0; k < np; ++k) denom = __dadd_rn(denom, At[lt * np + k]);
        aux[lt] = __ddiv_rn(1.0, denom);
    }
    __syncthreads();
    if (active)
        for (int o = lt; o < 2 * np * np; o += nthr) {
            const int r = o / np, k = o - r * np, h = hit[r];
            At[o] = h < np ? (k == h ? 1.0 : 0.0) : __dmul_rn(At[o], aux[r]);
        }
    __syncthreads();
}

// M2M (cluster_tree.cpp:192-216): pw = sum_children Axi * cw * Aeta^T, for one level.
__global__ void __launch_bounds__(kPassThreads)
    k_m2m(TreeView t, Cheb cheb, int first, double* __restrict__ qw, int mode, Own own) {
    extern __shared__ double sm[];
    const int c = first + blockIdx.x;
    const int nch = t.nchild[c];
    if (nch == 0 || !selected(t, c, mode, own)) return;
    const int np = cheb.np, npp = np * np;
    double* Ax = sm;             // At layout
    double* Ae = sm + npp;
    double* tmp = sm + 2 * npp;  // tmp[k1*np + m2]
    double pxm, pxh, pem, peh;
    mid_half(t.xi0[c], t.xi1[c], pxm, pxh);
    mid_half(t.eta0[c], t.eta1[c], pem, peh);
    double acc[(kMaxNp * kMaxNp + kPassThreads - 1) / kPassThreads];
#pragma unroll
    for (int i = 0; i < (kMaxNp * kMaxNp + kPassThreads - 1) / kPassThreads; ++i) acc[i] = 0.0;
    const int4 ch4 = t.child[c];
    const int chs[4] = {ch4.x, ch4.y, ch4.z, ch4.w};
    for (int q = 0; q < nch; ++q) {
        const int ch = chs[q];
        double cxm, cxh, cem, ceh;
        mid_half(t.xi0[ch], t.xi1[ch], cxm, cxh);
        mid_half(t.eta0[ch], t.eta1[ch], cem, ceh);
        if (threadIdx.x < np) transfer_cols(cheb, pxm, pxh, cxm, cxh, threadIdx.x, Ax);
        else if (threadIdx.x < 2 * np) transfer_cols(cheb, pem, peh, cem, ceh, threadIdx.x - np, Ae);
        __syncthreads();
        const double* cw = qw + (long long)ch * npp;
        for (int o = threadIdx.x; o < npp; o += kPassThreads) {
            const int k1 = o / np, m2 = o % np;
            double s = 0.0;
            for (int m1 = 0; m1 < np; ++m1) s = __dadd_rn(s, __dmul_rn(Ax[m1 * np + k1], cw[m1 * np + m2]));
            tmp[o] = s;
        }
        __syncthreads();
        int idx = 0;
        for (int o = threadIdx.x; o < npp; o += kPassThreads, ++idx) {
            const int k1 = o / np, k2 = o % np;
            double s = 0.0;
            for (int m2 = 0; m2 < np; ++m2) s = __dadd_rn(s, __dmul_rn(tmp[k1 * np + m2], Ae[m2 * np + k2]));
            acc[idx] = __dadd_rn(acc[idx], s);
        }
        __syncthreads();
    }
    int idx = 0;
    for (int o = threadIdx.x; o < npp; o += kPassThreads, ++idx) qw[(long long)c * npp + o] = acc[idx];
}

// The same M2M with the (up to) four children in parallel: thread group q (kPassThreads
// threads) builds child q's transfer matrices and its contribution Axi cw Aeta^T into
// shared memory; the contributions are then added in child order — the same operations
// and order as k_m2m, bit for bit, with 6 barriers per cluster instead of 12 and the
// transfer matrices built by the whole group (transfer_pair).  Used while 16 (p+1)^2 +
// 16 (p+1) doubles fit the 48 KB static window (degree <= 17).
constexpr int kM2mGroups = 4;
__global__ void __launch_bounds__(kM2mGroups * kPassThreads)
    k_m2m4(TreeView t, Cheb cheb, int first, double* __restrict__ qw, int mode, Own own) {
    extern __shared__ double sm[];
    const int c = first + blockIdx.x;
    const int nch = t.nchild[c];
    if (nch == 0 || !selected(t, c, mode, own)) return;
    const int np = cheb.np, npp = np * np;
    const int q = threadIdx.x / kPassThreads, lt = threadIdx.x - q * kPassThreads;
    double* Ax = sm + q * 3 * npp;  // At layout
    double* Ae = Ax + npp;
    double* tmp = Ae + npp;  // tmp[k1*np + m2]
    double* contrib = sm + kM2mGroups * 3 * npp;
    double* aux = sm + kM2mGroups * 4 * npp + q * 4 * np;  // 2np doubles + 2np ints per group
    double pxm, pxh, pem, peh;
    mid_half(t.xi0[c], t.xi1[c], pxm, pxh);
    mid_half(t.eta0[c], t.eta1[c], pem, peh);
    const int4 ch4 = t.child[c];
    const int chs[4] = {ch4.x, ch4.y, ch4.z, ch4.w};
    const bool mine = q < nch;
    const int ch = mine ? chs[q] : 0;
    double cxm = 0.0, cxh = 0.0, cem = 0.0, ceh = 0.0;
    if (mine) {
        mid_half(t.xi0[ch], t.xi1[ch], cxm, cxh);
        mid_half(t.eta0[ch], t.eta1[ch], cem, ceh);
    }
    transfer_pair(cheb, mine, lt, kPassThreads, pxm, pxh, pem, peh, cxm, cxh, cem, ceh, Ax, aux,
                  reinterpret_cast<int*>(aux + 2 * np));
    if (mine) {
        const double* cw = qw + (long long)ch * npp;
        for (int o = lt; o < npp; o += kPassThreads) {
            const int k1 = o / np, m2 = o % np;
            double s = 0.0;
            for (int m1 = 0; m1 < np; ++m1) s = __dadd_rn(s, __dmul_rn(Ax[m1 * np + k1], cw[m1 * np + m2]));
            tmp[o] = s;
        }
    }
    __syncthreads();
    if (mine)
        for (int o = lt; o < npp; o += kPassThreads) {
            const int k1 = o / np, k2 = o % np;
            double s = 0.0;
            for (int m2 = 0; m2 < np; ++m2) s = __dadd_rn(s, __dmul_rn(tmp[k1 * np + m2], Ae[m2 * np + k2]));
            contrib[q * npp + o] = s;
        }
    __syncthreads();
    for (int o = threadIdx.x; o < npp; o += kM2mGroups * kPassThreads) {
        double acc = 0.0;
        for (int k = 0; k < nch; ++k) acc = __dadd_rn(acc, contrib[k * npp + o]);
        qw[(long long)c * npp + o] = acc;
    }
}

// L2L (cluster_tree.cpp:256-279), one CTA per child at level `first..`:
// child[n1,n2,d] += sum_{m1,m2} Axi[m1,n1] Aeta[m2,n2] P[m1,m2,d], done separably.
__global__ void __launch_bounds__(kPassThreads)
    k_l2l(TreeView t, Cheb cheb, int first, int dim, double* __restrict__ qphi, Own own) {
    extern __shared__ double sm[];
    const int ch = first + blockIdx.x;
    const int c = t.parent[ch];
    if (c < 0 || t.begin[ch] < own.b || t.begin[ch] >= own.e) return;
    const int np = cheb.np, npp = np * np;
    double* Ax = sm;
    double* Ae = sm + npp;
    double* tmp = sm + 2 * npp;  // tmp[(n1*np + m2)*dim + d]
    double pxm, pxh, pem, peh, cxm, cxh, cem, ceh;
    mid_half(t.xi0[c], t.xi1[c], pxm, pxh);
    mid_half(t.eta0[c], t.eta1[c], pem, peh);
    mid_half(t.xi0[ch], t.xi1[ch], cxm, cxh);
    mid_half(t.eta0[ch], t.eta1[ch], cem, ceh);
    double* aux = tmp + npp * dim;  // 2np doubles + 2np ints
    transfer_pair(cheb, true, threadIdx.x, kPassThreads, pxm, pxh, pem, peh, cxm, cxh, cem, ceh, Ax, aux,
                  reinterpret_cast<int*>(aux + 2 * np));
    const double* P = qphi + (long long)c * npp * dim;
    for (int o = threadIdx.x; o < npp * dim; o += kPassThreads) {
        const int d = o % dim, r = o / dim, n1 = r / np, m2 = r % np;
        double s = 0.0;
        // Axi[m1][n1] = L^parent_{m1}(child node n1) = At[n1*np + m1]
        for (int m1 = 0; m1 < np; ++m1) s += Ax[n1 * np + m1] * P[(m1 * np + m2) * dim + d];
        tmp[o] = s;
    }
    __syncthreads();
    double* C = qphi + (long long)ch * npp * dim;
    for (int o = threadIdx.x; o < npp * dim; o += kPassThreads) {
        const int d = o % dim, r = o / dim, n1 = r / np, n2 = r % np;
        double s = 0.0;
        for (int m2 = 0; m2 < np; ++m2) s += Ae[n2 * np + m2] * tmp[(n1 * np + m2) * dim + d];
        C[o] += s;
    }
}

// L2P (cluster_tree.cpp:241-255) fused with the final scatter to input order:
// out[perm[t]] = near[t] + sum_k Lx[k1] Ly[k2] P[k].  NP > 0: compile-time (p+1), bases in
// registers; NP = 0: any degree.
#ifndef CSFS_L2P_MINB
#define CSFS_L2P_MINB 8
#endif
template <int NP, int D>
__global__ void __launch_bounds__(kPassThreads, CSFS_L2P_MINB)
    k_l2p(TreeView t, Cheb cheb, const double* __restrict__ qphi, const double* __restrict__ near,
          double* __restrict__ out, Own own, bool out_perm) {
    extern __shared__ double sm[];
    const int c = blockIdx.x;
    if (t.nchild[c] > 0) return;
    const int b = t.begin[c], e = t.end[c];
    if (b == e || b < own.b || b >= own.e) return;
    const int np = NP > 0 ? NP : cheb.np, npp = np * np;
    for (int o = threadIdx.x; o < npp * D; o += kPassThreads) sm[o] = qphi[(long long)c * npp * D + o];
    __syncthreads();
    double xm, xh, em, eh;
    mid_half(t.xi0[c], t.xi1[c], xm, xh);
    mid_half(t.eta0[c], t.eta1[c], em, eh);
    constexpr int M = NP > 0 ? NP : kMaxNp;
    for (int p = b + threadIdx.x; p < e; p += kPassThreads) {
        double lx[M], ly[M];
        bary1d_fast<NP>(cheb, ref_coord(t.xi[p], xm, xh), lx);
        bary1d_fast<NP>(cheb, ref_coord(t.eta[p], em, eh), ly);
        double f[D];
#pragma unroll
        for (int d = 0; d < D; ++d) f[d] = 0.0;
        // separably: f = sum_k1 Lx[k1] (sum_k2 Ly[k2] P[k1][k2])  (np^2 + np FMAs per output
        // component instead of 2 np^2; roundoff-level difference from the reference's order)
#pragma unroll
        for (int k1 = 0; k1 < M; ++k1) {
            if (k1 >= np) break;
            const double* row = sm + k1 * np * D;
            double g[D];
#pragma unroll
            for (int d = 0; d < D; ++d) g[d] = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < M; ++k2) {
                if (k2 >= np) break;
#pragma unroll
                for (int d = 0; d < D; ++d) g[d] = fma(ly[k2], row[k2 * D + d], g[d]);
            }
#pragma unroll
            for (int d = 0; d < D; ++d) f[d] = fma(lx[k1], g[d], f[d]);
        }
        const long long dst = (long long)(out_perm ? t.perm[p] : p) * D;
#pragma unroll
        for (int d = 0; d < D; ++d) out[dst + d] = near[(long long)p * D + d] + f[d];
    }
}

__global__ void k_scatter_out(long long n, int dim, const int* __restrict__ perm,
                              const double* __restrict__ phi, double* __restrict__ out) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n * dim) return;
    const long long t = g / dim;
    const int d = int(g - t * dim);
    out[(long long)perm[t] * dim + d] = phi[g];
}

}  // namespace

void scatter_to_input(const DeviceTree& tgt, int dim, const double* phi_tree, double* out, cudaStream_t s) {
    const long long n = tgt.n * dim;
    k_scatter_out<<<ceil_div(n, 256), 256, 0, s>>>(tgt.n, dim, tgt.perm, phi_tree, out);
    CSFS_LAUNCH_CHECK();
}

void upward_pass(DeviceTree& src, const Cheb& cheb, cudaStream_t s, int mode, Own own) {
    const TreeView v = src.view();
    const int np = cheb.np, npp = np * np;
    if (mode != 2) {
        src.qw.grow((size_t)src.ncl * npp);
        if (mode == 1) CSFS_CK(cudaMemsetAsync(src.qw.p, 0, (size_t)src.ncl * npp * sizeof(double), s));
    }
    const size_t sm_p2m = size_t(2) * kP2mChunk * np * sizeof(double);
    const int n_p2m = mode == 2 ? src.level_count[0] : src.ncl;  // depth 0 = ids 0..5
    auto p2m = [&](auto kern) { kern<<<n_p2m, kPassThreads, sm_p2m, s>>>(v, cheb, src.w, src.qw, mode, own); };
    auto p2m_tc = [&](auto kern) { kern<<<n_p2m, kPassThreads, 0, s>>>(v, cheb, src.w, src.qw, mode, own); };
    // CSFS_B200_P2M: unset = register-blocked FMA kernel, "fma" = the round-1/2 FMA kernel
    // (two shared loads per FMA), "dmma" = FP64 tensor cores (DESIGN.md §3 A/B)
    const char* pe = std::getenv("CSFS_B200_P2M");
    const std::string pv = pe ? pe : "";
    const bool dmma = pv == "dmma", plain = pv == "fma";
    switch (np) {
        case 7: dmma ? p2m_tc(k_p2m_dmma<7>) : plain ? p2m(k_p2m<7>) : p2m_tc(k_p2m_rb<7>); break;
        case 9: dmma ? p2m_tc(k_p2m_dmma<9>) : plain ? p2m(k_p2m<9>) : p2m_tc(k_p2m_rb<9>); break;
        case 11: dmma ? p2m_tc(k_p2m_dmma<11>) : plain ? p2m(k_p2m<11>) : p2m_tc(k_p2m_rb<11>); break;
        default: p2m(k_p2m<0>);
    }
    CSFS_LAUNCH_CHECK();
    const size_t sm_m2m = size_t(3) * npp * sizeof(double);
    const size_t sm_m2m4 = size_t(4 * kM2mGroups) * (npp + np) * sizeof(double);
    const int lo = mode == 1 ? 1 : 0;
    const int hi = mode == 2 ? 0 : src.depth_max() - 1;
    for (int L = hi; L >= lo; --L) {
        if (src.level_count[L] == 0) continue;
        if (sm_m2m4 <= 48 * 1024)
            k_m2m4<<<src.level_count[L], kM2mGroups * kPassThreads, sm_m2m4, s>>>(v, cheb, src.level_first[L], src.qw,
                                                                                mode, own);
        else
            k_m2m<<<src.level_count[L], kPassThreads, sm_m2m, s>>>(v, cheb, src.level_first[L], src.qw, mode, own);
        CSFS_LAUNCH_CHECK();
    }
}

void downward_pass(DeviceTree& tgt, const Cheb& cheb, int dim, const double* phi_near, double* out,
                   cudaStream_t s, Own own, bool out_perm) {
    const TreeView v = tgt.view();
    const int np = cheb.np, npp = np * np;
    const size_t sm_l2l = size_t(2 * npp + npp * dim + 4 * np) * sizeof(double);
    for (int L = 1; L <= tgt.depth_max(); ++L) {
        if (tgt.level_count[L] == 0) continue;
        k_l2l<<<tgt.level_count[L], kPassThreads, sm_l2l, s>>>(v, cheb, tgt.level_first[L], dim, tgt.qphi, own);
        CSFS_LAUNCH_CHECK();
    }
    const size_t sm_l2p = size_t(npp) * dim * sizeof(double);
    auto go = [&](auto kern) {
        kern<<<tgt.ncl, kPassThreads, sm_l2p, s>>>(v, cheb, tgt.qphi, phi_near, out, own, out_perm);
    };
    if (dim == 1) {
        switch (np) {
            case 7: go(k_l2p<7, 1>); break;
            case 9: go(k_l2p<9, 1>); break;
            case 11: go(k_l2p<11, 1>); break;
            default: go(k_l2p<0, 1>);
        }
    } else {
        switch (np) {
            case 7: go(k_l2p<7, 3>); break;
            case 9: go(k_l2p<9, 3>); break;
            case 11: go(k_l2p<11, 3>); break;
            default: go(k_l2p<0, 3>);
        }
    }
    CSFS_LAUNCH_CHECK();
}

}  // namespace csfs_b200
