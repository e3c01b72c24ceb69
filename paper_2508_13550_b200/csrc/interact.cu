// Unified near/far-field evaluation kernel: evaluate_pp, evaluate_pc and
// accumulate_cp_cc of the reference (/root/reference/proj/src/summation.cpp:205-306) are
// all "targets x source point set, weighted" direct sums, so one
// persistent kernel evaluates every list:
//   * a work item = one target leaf (targets: its particles; sources: PP leaves' particles
//     and PC clusters' proxy points) or one target cluster (targets: its (p+1)^2 proxy
//     points; sources: CP leaves' particles and CC clusters' proxy points);
//   * CTAs pull items from an atomic queue (dynamic, like the reference's
//     schedule(dynamic,4)); every output slot is owned by exactly one item and summed in
//     a fixed order, so results are deterministic;
//   * source points + weights stream through shared memory in chunks ({x,y},{z,w} pairs:
//     two broadcast LDS.128 per source per thread); each thread keeps TPT targets in
//     registers, so every shared-memory source is reused TPT times and the TPT
//     evaluations are independent FP64 chains (ILP for the DFMA pipe);
//   * small target sets (49/64/81/121) are packed G groups per CTA that split the source
//     range and are combined in a fixed order at the end.
// This is FP64-pipe bound: the inner loop is the kernel functor.
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "engine.hpp"
#include "kernels_dev.cuh"
#include "scan.cuh"

namespace csfs_b200 {

// fastmath.cuh table: {r_i, L_i} from tools/gen_log_table.c (verified by
// tests/test_host.py::test_log_table).
void make_log_table(double2* tab) {
    static const double kTab[kLogTab][2] = {
#include "log_table.inc"
    };
    for (int i = 0; i < kLogTab; ++i) tab[i] = make_double2(kTab[i][0], kTab[i][1]);
}

namespace {

#ifndef CSFS_IB
#define CSFS_IB 256
#endif
// fused 1 - x.y on list entries whose point sets are > kFuseGap apart (engine.hpp)
#ifndef CSFS_FUSED_DOT
#define CSFS_FUSED_DOT 1
#endif
#ifndef CSFS_TPT
#define CSFS_TPT 2
#endif
#ifndef CSFS_MINB
#define CSFS_MINB 2
#endif
#ifndef CSFS_UNROLL
#define CSFS_UNROLL 8
#endif
constexpr int kIB = CSFS_IB;    // threads per CTA
constexpr int kTPT = CSFS_TPT;  // targets per thread
constexpr int kICH = 256;       // source points per shared-memory chunk
constexpr int kUnroll = CSFS_UNROLL;
// source-loop unroll of k_interact per functor (measured: the log/rsqrt functors gain from
// deeper unrolling, the larger dilog functor loses): Op::kUnroll, else CSFS_UNROLL
template <class Op, class = void>
struct UnrollOf {
    static constexpr int value = kUnroll;
};
template <class Op>
struct UnrollOf<Op, std::void_t<decltype(Op::kUnroll)>> {
    static constexpr int value = Op::kUnroll;
};
// resident CTAs per SM k_interact is compiled for, per functor (Op::kMinBlocks, else
// CSFS_MINB): three (80 registers, 3 x 73 KB of shared memory) for Laplace and the
// biharmonic kernel — C2 -4.7%, C3 -4.3% — two (124 registers) for SAL, whose deeper
// unrolled loop loses 1% at 80 registers, and for Biot-Savart (its 3-component reduction
// buffer leaves no room for a third CTA)
template <class Op, class = void>
struct MinBlocksOf {
    static constexpr int value = CSFS_MINB;
};
template <class Op>
struct MinBlocksOf<Op, std::void_t<decltype(Op::kMinBlocks)>> {
    static constexpr int value = Op::kMinBlocks;
};
// Ops whose far-field sum factors through the source positions (Biot-Savart:
// sum_s a_s (t x s) = t x sum_s a_s s): Op::kFarFactored, eval_far, far_finish
template <class Op, class = void>
struct FarOf {
    static constexpr bool value = false;
};
template <class Op>
struct FarOf<Op, std::void_t<decltype(Op::kFarFactored)>> {
    static constexpr bool value = Op::kFarFactored;
};

#ifndef CSFS_MTPT
#define CSFS_MTPT 2
#endif
constexpr int kMTPT = CSFS_MTPT;  // targets per thread in the symmetric kernel

struct InteractParams {
    const int4* item;
    int n_items;
    const int2* seg;
    int* counter;
    const double *tpx, *tpy, *tpz;  // targets: particles (tree order)
    const double *tqx, *tqy, *tqz;  // targets: proxy points
    const double *spx, *spy, *spz, *spw;  // sources: particles + weights
    const double *sqx, *sqy, *sqz, *sqw;  // sources: proxy points + proxy weights
    double* out_p;  // phi_near (N_t x dim)
    double* out_q;  // proxy potentials (ncl_t x npp x dim)
    const int* anchor;  // per item owner key (nullptr: every item is ours)
    long long own_b, own_e;
    // a rank's own items, compacted (interact(): partitioned calls): item idx[0 .. *n_own)
    const int* idx;
    const int* n_own;
    const double2* log_tab;  // kLogTabWords entries (fastmath.cuh)
    // symmetric-pair partial blocks of each item's key (k_mutual ran first), added to the
    // item's outputs in ascending block order; mcnt == nullptr: none
    const int* keys;
    const int *mcnt, *moff;
    const long long* mlist;
    const double* partial;
};

template <class Op>
__global__ void __launch_bounds__(kIB, MinBlocksOf<Op>::value) k_interact(InteractParams P, Op op) {
    constexpr int D = Op::dim;
    constexpr int kU = UnrollOf<Op>::value;
    // the group reduction after the source loop reuses the source buffers for scalar kernels
    // (D == 1: 4 KB of 8), so three CTAs (3 x (64 KB table + 8 KB)) fit one SM's 228 KB
    __shared__ double2 sbuf[2 * kICH];
    __shared__ double red_own[D == 1 ? 1 : kIB * kTPT * D];
    double2* const sxy = sbuf;
    double2* const szw = sbuf + kICH;
    double* const red = D == 1 ? reinterpret_cast<double*>(sbuf) : red_own;
    static_assert(D != 1 || kIB * kTPT * sizeof(double) <= sizeof(double2) * 2 * kICH, "red fits the source buffers");
    extern __shared__ double2 tab_sm[];  // kLogTabBytes (dynamic)
    __shared__ int item_sh[2];
    const int tid = threadIdx.x;
    const LogTable tab = stage_log_table(tab_sm, P.log_tab);  // synced by the loop's first barrier
    // The queue ticket of the NEXT item is fetched while this one is evaluated (the atomic's
    // round trip sat at the head of every item: 16% of the stall samples of the small-leaf
    // configs, ncu round 2).  Two slots: thread 0 publishes ticket i + 1 into the slot that
    // nobody reads until the next barrier, so one barrier per item is enough.
    int ticket = 0, slot = 0;
    if (tid == 0) ticket = atomicAdd(P.counter, 1);
    for (;;) {
        if (tid == 0) item_sh[slot] = ticket;
        __syncthreads();  // also: the previous item's shared-memory reads are done
        const int q = item_sh[slot];
        slot ^= 1;
        const int n_items = P.n_own ? *P.n_own : P.n_items;
        if (q >= n_items) break;
        if (tid == 0) ticket = atomicAdd(P.counter, 1);
#ifndef CSFS_ITEM_ORDER_REVERSED
#define CSFS_ITEM_ORDER_REVERSED 1
#endif
        // the queue hands out the items back to front: build_items sorted them by cost
        // (traverse.cu order_items_by_cost), so the most expensive go first and the
        // kernel's tail is made of the cheapest (longest-processing-time first)
        const int iq = CSFS_ITEM_ORDER_REVERSED ? n_items - 1 - q : q;
        const int it = P.idx ? P.idx[iq] : iq;
        if (P.anchor) {
            const int a = P.anchor[it];
            if (a >= 0 && (a < P.own_b || a >= P.own_e)) continue;  // another rank's target
        }
        const int4 d = P.item[it];
        const bool tproxy = d.y < 0;
        const int tlen = tproxy ? -d.y : d.y;
        // group size: threads that together hold the (up to) kIB*kTPT targets of one pass
        const int per = (tlen + kTPT - 1) / kTPT;
        const int gs = min(kIB, (per + 31) & ~31);
        const int G = kIB / gs;
        const int g = tid / gs, r = tid - g * gs;
        const double* TX = tproxy ? P.tqx : P.tpx;
        const double* TY = tproxy ? P.tqy : P.tpy;
        const double* TZ = tproxy ? P.tqz : P.tpz;
        double* OUT = tproxy ? P.out_q : P.out_p;
        for (int t0 = 0; t0 < tlen; t0 += gs * kTPT) {
            const bool grp = g < G;
            double tx[kTPT], ty[kTPT], tz[kTPT], acc[kTPT][D];
            constexpr bool kFar = FarOf<Op>::value;
            double far[kFar ? kTPT : 1][3];  // far-field source moments (FarOf ops)
            if constexpr (kFar)
#pragma unroll
                for (int k = 0; k < kTPT; ++k) far[k][0] = far[k][1] = far[k][2] = 0.0;
            bool act[kTPT];
#pragma unroll
            for (int k = 0; k < kTPT; ++k) {
                const int t = t0 + r + k * gs;
                act[k] = grp && t < tlen;
                tx[k] = 0.0;
                ty[k] = 0.0;
                tz[k] = 1.0;
                if (act[k]) {
                    tx[k] = op.tgt(TX[d.x + t]);
                    ty[k] = op.tgt(TY[d.x + t]);
                    tz[k] = op.tgt(TZ[d.x + t]);
                }
#pragma unroll
                for (int c = 0; c < D; ++c) acc[k][c] = 0.0;
            }
            const bool any = act[0];  // slot 0 is filled first
            // guarded: the chunk holds a segment that may contain coincident pairs
            // group g takes a contiguous share of the chunk: unit stride, so the unrolled
            // loop addresses shared memory with immediate offsets (no per-source pointer math)
            auto compute = [&](int n, bool guarded, bool fused) {
                if (!any) return;
                const int share = (n + G - 1) / G;
                const int jb = g * share, je = min(n, jb + share);
                if (guarded) {
#pragma unroll kU
                    for (int j = jb; j < je; ++j) {
                        const double2 a = sxy[j], b = szw[j];
#pragma unroll
                        for (int k = 0; k < kTPT; ++k)
                            op.template eval<true>(tx[k], ty[k], tz[k], a.x, a.y, b.x, b.y, acc[k], tab);
                    }
                } else if (fused) {
#pragma unroll kU
                    for (int j = jb; j < je; ++j) {
                        const double2 a = sxy[j], b = szw[j];
#pragma unroll
                        for (int k = 0; k < kTPT; ++k) {
                            if constexpr (kFar)
                                op.eval_far(tx[k], ty[k], tz[k], a.x, a.y, b.x, b.y, far[k], tab);
                            else
                                op.template eval<false, true>(tx[k], ty[k], tz[k], a.x, a.y, b.x, b.y, acc[k], tab);
                        }
                    }
                } else {
#pragma unroll kU
                    for (int j = jb; j < je; ++j) {
                        const double2 a = sxy[j], b = szw[j];
#pragma unroll
                        for (int k = 0; k < kTPT; ++k)
                            op.template eval<false>(tx[k], ty[k], tz[k], a.x, a.y, b.x, b.y, acc[k], tab);
                    }
                }
            };
            // Source chunks of kICH points walk the item's segments; the next chunk's global
            // loads (one point per thread) are issued before the current chunk is evaluated,
            // so their latency hides behind the FP64 work.
            static_assert(kICH == kIB, "one source slot per thread");
            int ce = d.z, cpos = 0;  // cursor into the segment list (CTA-uniform)
            double rx = 0.0, ry = 0.0, rz = 0.0, rw = 0.0;
            bool fguard = false;  // guard flag of the chunk being fetched (CTA-uniform)
            bool ffused = true;   // every segment of the chunk may use the fused 1 - x.y
            auto fetch = [&]() {
                int filled = 0;
                fguard = false;
                ffused = true;
                while (filled < kICH && ce < d.w) {
                    const int2 sg = P.seg[ce];
                    const bool sproxy = sg.y < 0;
                    const int len = seg_len(sg.y);  // 0: evaluated by the symmetric kernel
                    fguard = fguard || (len > 0 && seg_guard(sg.y));
                    ffused = ffused && (len == 0 || seg_fused(sg.y));
                    const int take = min(len - cpos, kICH - filled);
                    if (tid >= filled && tid < filled + take) {
                        const long long src = (long long)sg.x + cpos + (tid - filled);
                        rx = (sproxy ? P.sqx : P.spx)[src];
                        ry = (sproxy ? P.sqy : P.spy)[src];
                        rz = (sproxy ? P.sqz : P.spz)[src];
                        rw = (sproxy ? P.sqw : P.spw)[src];
                    }
                    filled += take;
                    cpos += take;
                    if (cpos == len) {
                        ++ce;
                        cpos = 0;
                    }
                }
                return filled;
            };
            int n = fetch();
            bool guarded = fguard, fused = ffused;
            while (n > 0) {
                if (tid < n) {
                    sxy[tid] = make_double2(rx, ry);
                    szw[tid] = make_double2(rz, rw);
                }
                __syncthreads();
                const int next = fetch();  // loads in flight during compute
#ifdef CSFS_FORCE_GUARD
                guarded = CSFS_FORCE_GUARD;
#endif
                compute(n, guarded, CSFS_FUSED_DOT && Op::kFusable && fused);
                __syncthreads();
                n = next;
                guarded = fguard;
                fused = ffused;
            }
            if constexpr (kFar)
#pragma unroll
                for (int k = 0; k < kTPT; ++k) op.far_finish(tx[k], ty[k], tz[k], far[k], acc[k]);
            if (G > 1) {
#pragma unroll
                for (int k = 0; k < kTPT; ++k)
                    if (act[k])
#pragma unroll
                        for (int c = 0; c < D; ++c) red[((g * gs + r) * kTPT + k) * D + c] = acc[k][c];
                __syncthreads();
                if (g == 0)
                    for (int h = 1; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < kTPT; ++k)
                            if (act[k])
#pragma unroll
                                for (int c = 0; c < D; ++c) acc[k][c] += red[((h * gs + r) * kTPT + k) * D + c];
                __syncthreads();
            }
            if (g == 0) {
                const double sc = op.scale();
                int mn = 0;
                const long long* ml = nullptr;
                if constexpr (D == 1) {
                    if (P.mcnt) {
                        const int X = P.keys[it];
                        mn = P.mcnt[X];
                        ml = P.mlist + P.moff[X];
                    }
                }
#pragma unroll
                for (int k = 0; k < kTPT; ++k)
                    if (act[k])
#pragma unroll
                        for (int c = 0; c < D; ++c) {
                            const int x = t0 + r + k * gs;
                            double v = acc[k][c] * sc;
                            for (int a = 0; a < mn; ++a) v += P.partial[ml[a] + x];  // D == 1
                            OUT[(long long)(d.x + x) * D + c] = v;
                        }
            }
        }
    }
}

// ---- symmetric PP / CC pairs (scalar kernels, targets == sources) --------------------------
// One CTA per leaf pair {A, B} listed in BOTH directions (A < B): every K(a, b) is
// evaluated ONCE and applied to both sides — row sums to A, column sums to B
// (K(b, a) = kSym K(a, b) bit-for-bit).  Same register/shared-memory structure as
// k_interact: A's targets (kTPT per thread) and their weights in registers, B (<= 256
// points) in shared memory, G thread groups splitting B in batches of 8.  Column partials
// are reduced per warp with a select-free transposed butterfly (4+2+1+1+1 shuffles per 8
// sources, each lane visiting the batch in its own XOR order), then over the group's warps
// in fixed order: deterministic, no atomics.  Both partial sums go
// to `partial`; k_interact, which runs after it, adds every block of a work item's key to
// the item's outputs in ascending block order.
struct MutualParams {
    const int4* pair;       // {A begin, |A|, B begin, |B|}, |A|, |B| <= 256; negative: proxy sets (CC)
    const long long* poff;  // partial offset of A's block (B's follows at + |A|)
    const int* anchor;      // A's begin, or -1: every rank
    int n_pairs;
    int* counter;  // work queue (persistent CTAs)
    const double *px, *py, *pz, *pw;  // particles (tree order) + weights
    const double *qx, *qy, *qz, *qw;  // proxy points + proxy weights
    double* partial;
    const double2* log_tab;
    long long own_b, own_e;
    const int* idx;    // a rank's own pairs, compacted: pair idx[0 .. *n_own)
    const int* n_own;
};

// double butterfly shuffle as two explicit 32-bit halves in one asm block (keeps the halves in place; the
// generic double overload let ptxas swap them and re-pair with moves)
__device__ __forceinline__ double shfl_xor_d(double v, int m) {
    int lo, hi;
    asm volatile("shfl.sync.bfly.b32 %0, %2, %4, 0x1f, -1;\n\tshfl.sync.bfly.b32 %1, %3, %4, 0x1f, -1;"
                 : "=r"(lo), "=r"(hi) : "r"(__double2loint(v)), "r"(__double2hiint(v)), "r"(m));
    return __hiloint2double(hi, lo);
}

#ifndef CSFS_MMINB
#define CSFS_MMINB CSFS_MINB
#endif
template <class Op>
__global__ void __launch_bounds__(kIB, CSFS_MMINB) k_mutual(MutualParams P, Op op) {
    static_assert(Op::dim == 1, "symmetric path is for scalar kernels");
    __shared__ double2 sbuf[2 * kICH];  // {x,y} then {z,w}: one base register, immediate offset
    double2* const sxy = sbuf;
    double2* const szw = sbuf + kICH;
    __shared__ double colbuf[kIB / 32][kICH];
    __shared__ double red[kIB * kMTPT];
    extern __shared__ double2 tab_sm[];  // kLogTabBytes (dynamic)
    __shared__ int pair_sh[2];
    const int tid = threadIdx.x, lane = tid & 31;
    const LogTable tab = stage_log_table(tab_sm, P.log_tab);  // synced by the loop's first barrier
    int ticket = 0, slot = 0;  // the next pair's queue ticket, fetched a pair ahead (see k_interact)
    if (tid == 0) ticket = atomicAdd(P.counter, 1);
    for (;;) {
        if (tid == 0) pair_sh[slot] = ticket;
        __syncthreads();  // also: the previous pair's shared-memory reads are done
        const int pq = pair_sh[slot];
        slot ^= 1;
        if (pq >= (P.n_own ? *P.n_own : P.n_pairs)) break;
        if (tid == 0) ticket = atomicAdd(P.counter, 1);
        const int p = P.idx ? P.idx[pq] : pq;
        if (P.anchor) {
            const long long a = P.anchor[p];
            if (a >= 0 && (a < P.own_b || a >= P.own_e)) continue;  // CTA-uniform
        }
        const int4 q = P.pair[p];
        const bool prox = q.y < 0;  // CC: both sides are proxy sets
#ifdef CSFS_FORCE_GUARD
        const bool guarded = CSFS_FORCE_GUARD;
#else
        const bool guarded = seg_guard(q.y);
#endif
        const bool fused = CSFS_FUSED_DOT && Op::kFusable && !guarded && seg_fused(q.w);
        const double* X = prox ? P.qx : P.px;
        const double* Y = prox ? P.qy : P.py;
        const double* Z = prox ? P.qz : P.pz;
        const double* Wt = prox ? P.qw : P.pw;
        const int tlen = seg_len(q.y), nb = seg_len(q.w);
        // padded to whole batches of 8 with zero-weight sources at the origin (finite K)
        for (int j = tid; j < ((nb + 7) & ~7); j += kIB) {
            const bool in = j < nb;
            sxy[j] = in ? make_double2(X[q.z + j], Y[q.z + j]) : make_double2(0.0, 0.0);
            szw[j] = in ? make_double2(Z[q.z + j], Wt[q.z + j]) : make_double2(0.0, 0.0);
        }
        const int per = (tlen + kMTPT - 1) / kMTPT;
        const int gs = min(kIB, (per + 31) & ~31);
        const int G = kIB / gs;
        const int g = tid / gs, r = tid - g * gs, wig = r >> 5;
        const bool grp = g < G;
        double tx[kMTPT], ty[kMTPT], tz[kMTPT], tw[kMTPT], acc[kMTPT];
        bool act[kMTPT];
#pragma unroll
        for (int k = 0; k < kMTPT; ++k) {
            const int t = r + k * gs;
            act[k] = grp && t < tlen;
            tx[k] = 0.0;  // padding target at the origin: 1 - x.y = 1 for every source, so its
            ty[k] = 0.0;  // (zero-weight) column terms stay finite in the unguarded path
            tz[k] = 0.0;
            tw[k] = 0.0;
            if (act[k]) {
                tx[k] = op.tgt(X[q.x + t]);
                ty[k] = op.tgt(Y[q.x + t]);
                tz[k] = op.tgt(Z[q.x + t]);
                tw[k] = Wt[q.x + t];
            }
            acc[k] = 0.0;
        }
        __syncthreads();
        if (grp) {
            // Batches of 8 consecutive sources, batch t to group t mod G.  Lane slot s holds
            // source s ^ q, q = (lane >> 2) & 7: the transposed butterfly then always keeps
            // the low half of its slots (no selects) and ends with lane holding source q's
            // column sum over the warp.  The 8 per-lane addresses of a slot are 8
            // consecutive entries: one shared-memory wavefront.
            constexpr int kB = 8;
            const int qx = (lane >> 2) & 7;
            auto sources = [&](int j, double (&c)[kB], auto kG, auto kF) {
#pragma unroll
                for (int m = 0; m < kB; ++m) {
                    c[m] = 0.0;
                    const int jm = j + (m ^ qx);
                    const double2 a = sxy[jm], b = szw[jm];
#pragma unroll
                    for (int k = 0; k < kMTPT; ++k) {
                        double K[1];
                        op.template value<decltype(kG)::value, decltype(kF)::value>(tx[k], ty[k], tz[k], a.x, a.y,
                                                                                     b.x, K, tab);
                        acc[k] = fma(b.y, K[0], acc[k]);
                        c[m] = fma(tw[k], K[0], c[m]);
                    }
                }
            };
            for (int j = g * kB; j < nb; j += kB * G) {
                double c[kB];
                if (guarded) sources(j, c, std::true_type{}, std::false_type{});
                else if (fused) sources(j, c, std::false_type{}, std::true_type{});
                else sources(j, c, std::false_type{}, std::false_type{});
                double v4[4], v2[2];
#pragma unroll
                for (int m = 0; m < 4; ++m) v4[m] = c[m] + shfl_xor_d(c[m + 4], 16);
#pragma unroll
                for (int m = 0; m < 2; ++m) v2[m] = v4[m] + shfl_xor_d(v4[m + 2], 8);
                double v = v2[0] + shfl_xor_d(v2[1], 4);
                v += shfl_xor_d(v, 2);
                v += shfl_xor_d(v, 1);
                const int jm = j + qx;
                if ((lane & 3) == 0 && jm < nb) colbuf[wig][jm] = v;
            }
        }
        // rows: combine the G groups (fixed order), then write A's block
        if (G > 1) {
#pragma unroll
            for (int k = 0; k < kMTPT; ++k)
                if (act[k]) red[(g * gs + r) * kMTPT + k] = acc[k];
        }
        __syncthreads();
        if (G > 1 && g == 0)
            for (int h = 1; h < G; ++h)
#pragma unroll
                for (int k = 0; k < kMTPT; ++k)
                    if (act[k]) acc[k] += red[(h * gs + r) * kMTPT + k];
        const long long base = P.poff[p];
        if (g == 0) {
#pragma unroll
            for (int k = 0; k < kMTPT; ++k)
                if (act[k]) P.partial[base + r + k * gs] = acc[k] * op.scale();
        }
        // columns: source j was handled by one group, whose warps wrote colbuf[0..W)[j]
        const int W = gs >> 5;
        const double f = op.scale() * Op::kSym;
        for (int j = tid; j < nb; j += kIB) {
            double v = 0.0;
            for (int w = 0; w < W; ++w) v += colbuf[w][j];
            P.partial[base + tlen + j] = v * f;
        }
    }
}

__global__ void k_aos_to_soa(const double* __restrict__ xyz, long long n, double* x, double* y, double* z) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = xyz[3 * i];
    y[i] = xyz[3 * i + 1];
    z[i] = xyz[3 * i + 2];
}

__global__ void k_direct_items(int n_items, long long nt, int4* item, int nseg) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    const long long t0 = (long long)i * kIB * kTPT;
    item[i] = make_int4(int(t0), int(min((long long)kIB * kTPT, nt - t0)), 0, nseg);
}

// Diagnostics: one functor evaluation per (x_i, y_i) pair, scale applied (= the
// reference's guarded per-pair value; guarded pairs give 0).
template <class Op>
__global__ void k_eval_pairs(Op op, const double* x, const double* y, long long n, double* out,
                             const double2* log_tab) {
    extern __shared__ double2 tab_sm[];  // kLogTabBytes (dynamic)
    const LogTable tab = stage_log_table(tab_sm, log_tab);
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc[3] = {0.0, 0.0, 0.0};
    op(op.tgt(x[3 * i]), op.tgt(x[3 * i + 1]), op.tgt(x[3 * i + 2]), y[3 * i], y[3 * i + 1], y[3 * i + 2], 1.0, acc, tab);
    for (int c = 0; c < Op::dim; ++c) out[i * Op::dim + c] = acc[c] * op.scale();
}

__global__ void k_eval_math(int fn, const double* x, long long n, double* out, const double2* log_tab) {
    extern __shared__ double2 tab_sm[];  // kLogTabBytes (dynamic)
    const LogTable tab = stage_log_table(tab_sm, log_tab);
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = x[i];
    double r = 0.0;
    switch (fn) {
        case 0: r = fast_log(v, tab); break;
        case 1: r = fast_rsqrt(v); break;
        case 2: r = fast_rcp(v); break;
        default: r = dilog_dev(v, tab); break;
    }
    out[i] = r;
}


// The evaluation kernels keep the log table in dynamic shared memory; with their static
// buffers that exceeds the 48 KB default, so opt in once per kernel.
template <class K>
void allow_table_smem(K kern) {
    CSFS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLogTabBytes)));
}

template <class Op>
int grid_for(int n_items) {
    int dev = 0, sms = 0, per = 0;
    CSFS_CK(cudaGetDevice(&dev));
    CSFS_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    allow_table_smem(k_interact<Op>);
    CSFS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_interact<Op>, kIB, kLogTabBytes));
    return std::max(1, std::min(n_items, sms * std::max(per, 1)));
}

template <class Op>
void launch(const InteractParams& p, const Op& op, cudaStream_t s) {
    if (p.n_items == 0) return;
    CSFS_CK(cudaMemsetAsync(p.counter, 0, sizeof(int), s));
    k_interact<Op><<<grid_for<Op>(p.n_items), kIB, kLogTabBytes, s>>>(p, op);
    CSFS_LAUNCH_CHECK();
}

template <class Op>
void launch_mutual(const MutualParams& m, const Op& op, cudaStream_t s) {
    if constexpr (Op::dim == 1) {
        if (m.n_pairs == 0) return;
        CSFS_CK(cudaMemsetAsync(m.counter, 0, sizeof(int), s));
        int dev = 0, sms = 0, per = 0;
        CSFS_CK(cudaGetDevice(&dev));
        CSFS_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        allow_table_smem(k_mutual<Op>);
        CSFS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mutual<Op>, kIB, kLogTabBytes));
#ifndef CSFS_MUTUAL_PERSIST
#define CSFS_MUTUAL_PERSIST 1
#endif
        const int grid = CSFS_MUTUAL_PERSIST ? std::max(1, std::min(m.n_pairs, sms * std::max(per, 1))) : m.n_pairs;
        k_mutual<Op><<<grid, kIB, kLogTabBytes, s>>>(m, op);
        CSFS_LAUNCH_CHECK();
    }
}

// Stable compaction of the work entries a rank owns (anchor < 0: every rank; else the
// anchor particle in [b, e)): idx[0 .. *count).  A partitioned call then only dequeues its
// own items instead of skipping the other ranks' ones one queue step at a time (a fixed
// ~1.4 ms per rank at C5, 14% of the evaluation at 8 ranks).
void compact_owned(const int* anchor, int n, Own own, DevBuf<int>& idx, int* count, DevBuf<int>& tiles,
                   cudaStream_t s) {
    idx.grow(std::max(n, 1));
    tiles.grow(scan_tile_ints(n, 1));
    int* out = idx.p;
    const long long b = own.b, e = own.e;
    auto f = [=] __device__(long long i, int* c) {
        const int a = anchor[i];
        c[0] = (a < 0 || (a >= b && a < e)) ? 1 : 0;
    };
    auto em = [=] __device__(long long i, const int* c, const int* pre) {
        if (c[0]) out[pre[0]] = int(i);
    };
    run_scan<1>(n, f, em, tiles.p, count, s);
}

}  // namespace

void interact(const KernelSpec& k, const DeviceTree& tgt, const DeviceTree& src, Items& items,
              double* phi_near, int* work_counter, const double2* log_tab, cudaStream_t s, Own own) {
    InteractParams p{};
    p.item = items.item;
    p.n_items = items.n_items;
    p.seg = items.seg;
    p.counter = work_counter;
    p.tpx = tgt.px;
    p.tpy = tgt.py;
    p.tpz = tgt.pz;
    p.tqx = tgt.qx;
    p.tqy = tgt.qy;
    p.tqz = tgt.qz;
    p.spx = src.px;
    p.spy = src.py;
    p.spz = src.pz;
    p.spw = src.w;
    p.sqx = src.qx;
    p.sqy = src.qy;
    p.sqz = src.qz;
    p.sqw = src.qw;
    p.out_p = phi_near;
    p.out_q = tgt.qphi;
    const bool everything = own.b <= 0 && own.e >= tgt.n;
    p.anchor = everything ? nullptr : items.anchor.p;
    p.own_b = own.b;
    p.own_e = own.e;
    p.log_tab = log_tab;
    MutualParams m{};
    if (items.mutual) {
        items.partial.grow(size_t(std::max<long long>(items.n_partial, 1)));
        m.pair = items.mpair;
        m.poff = items.mpoff;
        m.anchor = everything ? nullptr : items.manchor.p;
        m.n_pairs = items.n_mutual;
        m.counter = work_counter + 1;
        m.px = src.px;
        m.py = src.py;
        m.pz = src.pz;
        m.pw = src.w;
        m.qx = src.qx;
        m.qy = src.qy;
        m.qz = src.qz;
        m.qw = src.qw;
        m.partial = items.partial;
        m.log_tab = log_tab;
        m.own_b = own.b;
        m.own_e = own.e;
    }
    if (items.mutual) {  // k_interact adds the symmetric-pair blocks (after k_mutual, same stream)
        p.keys = items.keys;
        p.mcnt = items.mcnt;
        p.moff = items.moff;
        p.mlist = items.mlist;
        p.partial = items.partial;
    }
    if (!everything) {
        items.ocnt.grow(2);
        compact_owned(items.anchor, items.n_items, own, items.oitem, items.ocnt.p, items.otiles, s);
        p.idx = items.oitem;
        p.n_own = items.ocnt.p;
        p.anchor = nullptr;
        if (items.mutual) {
            compact_owned(items.manchor, items.n_mutual, own, items.opair, items.ocnt.p + 1, items.otiles, s);
            m.idx = items.opair;
            m.n_own = items.ocnt.p + 1;
            m.anchor = nullptr;
        }
    }
    with_op(k, [&](auto op) {
        if (items.mutual) launch_mutual(m, op, s);
        launch(p, op, s);
    });
}

void direct_allpairs(const KernelSpec& k, const double* txyz, long long nt, const double* sxyz,
                     const double* sw, long long ns, double* out, DevBuf<double>& soa,
                     DevBuf<int4>& items, DevBuf<int2>& segs, int* work_counter,
                     const double2* log_tab, cudaStream_t s) {
    if (nt == 0) return;
    soa.grow(size_t(3 * nt + 3 * ns));
    double* tx = soa.p;
    double* ty = tx + nt;
    double* tz = ty + nt;
    double* sx = tz + nt;
    double* sy = sx + ns;
    double* sz = sy + ns;
    k_aos_to_soa<<<ceil_div(nt, 256), 256, 0, s>>>(txyz, nt, tx, ty, tz);
    CSFS_LAUNCH_CHECK();
    if (ns) {
        k_aos_to_soa<<<ceil_div(ns, 256), 256, 0, s>>>(sxyz, ns, sx, sy, sz);
        CSFS_LAUNCH_CHECK();
    }
    std::vector<int2> hseg;
    const long long kSeg = 1 << 28;  // below the fused / guard flag bits
    for (long long b = 0; b < ns; b += kSeg)
        hseg.push_back(make_int2(int(b), int(std::min(kSeg, ns - b)) | kSegGuard));
    const int nseg = int(hseg.size());
    segs.grow(std::max(nseg, 1));
    if (nseg) CSFS_CK(cudaMemcpyAsync(segs.p, hseg.data(), nseg * sizeof(int2), cudaMemcpyHostToDevice, s));
    const int n_items = ceil_div(nt, kIB * kTPT);
    items.grow(n_items);
    k_direct_items<<<ceil_div(n_items, 128), 128, 0, s>>>(n_items, nt, items, nseg);
    CSFS_LAUNCH_CHECK();
    InteractParams p{};
    p.item = items;
    p.n_items = n_items;
    p.seg = segs;
    p.counter = work_counter;
    p.tpx = tx;
    p.tpy = ty;
    p.tpz = tz;
    p.spx = sx;
    p.spy = sy;
    p.spz = sz;
    p.spw = sw;
    p.out_p = out;
    p.log_tab = log_tab;
    with_op(k, [&](auto op) { launch(p, op, s); });
    CSFS_CK(cudaStreamSynchronize(s));  // hseg lifetime
}

void eval_pairs(const KernelSpec& k, const double* x, const double* y, long long n, double* out,
                const double2* log_tab, cudaStream_t s) {
    if (n == 0) return;
    with_op(k, [&](auto op) {
        allow_table_smem(k_eval_pairs<decltype(op)>);
        k_eval_pairs<<<ceil_div(n, 128), 128, kLogTabBytes, s>>>(op, x, y, n, out, log_tab);
        CSFS_LAUNCH_CHECK();
    });
}

void eval_math(int fn, const double* x, long long n, double* out, const double2* log_tab, cudaStream_t s) {
    if (n == 0) return;
    allow_table_smem(k_eval_math);
    k_eval_math<<<ceil_div(n, 128), 128, kLogTabBytes, s>>>(fn, x, n, out, log_tab);
    CSFS_LAUNCH_CHECK();
}

}  // namespace csfs_b200
