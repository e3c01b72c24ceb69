// CSTC — the cubed-sphere treecode (Barnes-Hut-style particle-cluster method): the B200
// restatement of csfs::cstc_sum (/root/reference/proj/src/summation.cpp:308-381),
// the second method behind summed_potential.
//
// One thread per target: the reference's per-target LIFO traversal of the source tree
// (roots 0..5, children pushed in quadrant order) with the point-cluster MAC
// (well_separated_pc, summation.cpp:128-130):
//   separated and big (count > n0)  -> PC: the cluster's (p+1)^2 proxy points/weights
//   not separated, internal         -> descend
//   otherwise (separated small, or non-separated leaf) -> PP: the cluster's particles
// evaluated with the same kernel functors and shared-memory log table as the FMM (staged
// per CTA).
// Targets are processed in source-tree order when targets == sources, so the 32 lanes of
// a warp (neighbours on the sphere) traverse almost identically (little divergence).
#include <cstdlib>
#include <string>

#include "engine.hpp"
#include "kernels_dev.cuh"

namespace csfs_b200 {

namespace {

#ifndef CSFS_CSTC_UNROLL
#define CSFS_CSTC_UNROLL 4
#endif
constexpr int kCstcUnroll = CSFS_CSTC_UNROLL;
constexpr int kCstcThreads = 256;  // 3 CTAs (3 x 64 KB log table) per SM
constexpr int kStack = 4 * kMaxDepth + 8;

template <class Op>
__global__ void __launch_bounds__(kCstcThreads)
    k_cstc(const double* __restrict__ txyz, long long nt, const int* __restrict__ order, TreeView S,
           const double* __restrict__ sw, const double* __restrict__ qw, double mac, int n0, Op op,
           const double2* __restrict__ log_tab, double* __restrict__ out, unsigned long long* counts) {
    constexpr int D = Op::dim;
    // the log table staged in shared memory like the FMM kernels (random 16-byte gathers
    // through L1 cost a sector per lane)
    extern __shared__ double2 tab_sm[];  // kLogTabBytes (dynamic)
    const LogTable tab = stage_log_table(tab_sm, log_tab);
    __syncthreads();
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long npp_ = 0, npc = 0;
    if (idx < nt) {
        const long long i = order ? order[idx] : idx;
        const double x = txyz[3 * i], y = txyz[3 * i + 1], z = txyz[3 * i + 2];
        const double tx = op.tgt(x), ty = op.tgt(y), tz = op.tgt(z);  // the functor's target form
        double acc[D];
#pragma unroll
        for (int d = 0; d < D; ++d) acc[d] = 0.0;
        int stack[kStack];
        int sp = 0;
        for (int r = 0; r < 6; ++r) stack[sp++] = r;
        const int npp = S.npp;
        while (sp > 0) {
            const int s = stack[--sp];
            const int b = S.begin[s], e = S.end[s];
            if (e == b) continue;
            // well_separated(target, 0, centre, radius, mac): R > 0 && 0 + r < mac R
            const double dx = __dsub_rn(x, S.cx[s]), dy = __dsub_rn(y, S.cy[s]), dz = __dsub_rn(z, S.cz[s]);
            const double R = __dsqrt_rn(dot_ref(dx, dy, dz, dx, dy, dz));
            const bool sep = R > 0.0 && __dadd_rn(0.0, S.rad[s]) < __dmul_rn(mac, R);
            if (sep) {
                if (e - b > n0) {
                    const long long q0 = (long long)s * npp;
#pragma unroll kCstcUnroll
                    for (int k = 0; k < npp; ++k) op(tx, ty, tz, S.qx[q0 + k], S.qy[q0 + k], S.qz[q0 + k], qw[q0 + k], acc, tab);
                    ++npc;
                    continue;
                }
            } else if (S.nchild[s] > 0) {
                const int4 ch = S.child[s];
                const int cs[4] = {ch.x, ch.y, ch.z, ch.w};
                for (int q = 0; q < S.nchild[s] && sp < kStack; ++q) stack[sp++] = cs[q];
                continue;
            }
#pragma unroll kCstcUnroll
            for (int j = b; j < e; ++j) op(tx, ty, tz, S.px[j], S.py[j], S.pz[j], sw[j], acc, tab);
            ++npp_;
        }
        const double sc = op.scale();
#pragma unroll
        for (int d = 0; d < D; ++d) out[i * D + d] = acc[d] * sc;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        npp_ += __shfl_xor_sync(0xffffffffu, npp_, o);
        npc += __shfl_xor_sync(0xffffffffu, npc, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&counts[0], npp_);
        atomicAdd(&counts[1], npc);
    }
}

// The same traversal, one WARP per 32 consecutive targets.  The warp walks the union of its
// lanes' traversals with a shared LIFO stack of (cluster, lane mask): a popped cluster is
// classified by every lane in its mask (the same MAC and size tests), the lanes that must
// descend push the children once with their mask, and the lanes that interact with it —
// through its proxies (PC) or its particles (PP) — evaluate it together.  Every lane still
// meets its clusters in the order of its own depth-first traversal (the union's order
// restricted to the lane's clusters), so each target's sum has the reference's order: bit
// for bit the one-thread-per-target kernel above, same pp / pc counts.  What it buys: the
// cluster's sources are loaded ONCE per warp, coalesced, staged in shared memory and read
// back as broadcasts (the next chunk's loads in flight during the current chunk's
// evaluation) instead of every lane issuing its own uniform-address loads and waiting on
// them; the stack lives in shared memory instead of 1 KB of local memory per thread.
#ifndef CSFS_CSTC_WARP_UNROLL
#define CSFS_CSTC_WARP_UNROLL 8
#endif
constexpr int kCstcWarpUnroll = CSFS_CSTC_WARP_UNROLL;
constexpr int kCstcWarpThreads = 512;  // 16 warps; 2 CTAs per SM (table 64 KB + 48 KB)
constexpr int kCstcWarps = kCstcWarpThreads / 32;
constexpr size_t kCstcWarpSmem =
    kLogTabBytes + size_t(kCstcWarps) * (64 * sizeof(double2) + kStack * sizeof(int2));

template <class Op>
__global__ void __launch_bounds__(kCstcWarpThreads, 2)
    k_cstc_warp(const double* __restrict__ txyz, long long nt, const int* __restrict__ order, TreeView S,
                const double* __restrict__ sw, const double* __restrict__ qw, double mac, int n0, Op op,
                const double2* __restrict__ log_tab, double* __restrict__ out, unsigned long long* counts) {
    constexpr int D = Op::dim;
    constexpr unsigned kFull = 0xffffffffu;
    extern __shared__ double2 dyn[];  // the log table, then per warp: 32 {x,y} + 32 {z,w}, then the stacks
    const LogTable tab = stage_log_table(dyn, log_tab);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2* const sxy = dyn + kLogTab + warp * 64;
    double2* const szw = sxy + 32;
    int2* const stack = reinterpret_cast<int2*>(dyn + kLogTab + kCstcWarps * 64) + warp * kStack;
    __syncthreads();
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = idx < nt;
    const unsigned alive = __ballot_sync(kFull, live);
    if (alive == 0) return;  // warp-uniform
    const long long i = live ? (order ? order[idx] : idx) : 0;
    const double x = live ? txyz[3 * i] : 0.0, y = live ? txyz[3 * i + 1] : 0.0, z = live ? txyz[3 * i + 2] : 1.0;
    const double tx = op.tgt(x), ty = op.tgt(y), tz = op.tgt(z);
    double acc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = 0.0;
    unsigned long long npp_ = 0, npc = 0;
    if (lane < 6) stack[lane] = make_int2(lane, int(alive));
    int sp = 6;
    __syncwarp();
    const int npp = S.npp;
    const bool unit = order != nullptr && !*S.off_sphere;  // targets are the tree's particles, all on the sphere

    // `act` lanes add the cnt sources at X/Y/Z/W[base ..) to their sums, in index order.
    // guard (warp-uniform): some active lane may hold a pair with 1 - x.y < 1e-14; without it
    // the functor's coincidence guard is compiled out — the same values (the guard only
    // drops coincident pairs), fewer integer instructions.
    auto evaluate = [&](const double* __restrict__ X, const double* __restrict__ Y, const double* __restrict__ Z,
                        const double* __restrict__ W, long long base, int cnt, bool act, bool guard) {
        double nx = 0.0, ny = 0.0, nz = 0.0, nw = 0.0;
        if (lane < cnt) {
            nx = X[base + lane];
            ny = Y[base + lane];
            nz = Z[base + lane];
            nw = W[base + lane];
        }
        for (int c0 = 0; c0 < cnt; c0 += 32) {
            __syncwarp();  // the previous chunk has been read
            sxy[lane] = make_double2(nx, ny);
            szw[lane] = make_double2(nz, nw);
            __syncwarp();
            const int j = c0 + 32 + lane;  // the next chunk's loads fly during this chunk's evaluation
            if (j < cnt) {
                nx = X[base + j];
                ny = Y[base + j];
                nz = Z[base + j];
                nw = W[base + j];
            }
            const int m = min(32, cnt - c0);
            if (act && guard) {
#pragma unroll kCstcWarpUnroll
                for (int k = 0; k < m; ++k) {
                    const double2 a = sxy[k], b = szw[k];
                    op.template eval<true, false>(tx, ty, tz, a.x, a.y, b.x, b.y, acc, tab);
                }
            } else if (act) {
#pragma unroll kCstcWarpUnroll
                for (int k = 0; k < m; ++k) {
                    const double2 a = sxy[k], b = szw[k];
                    op.template eval<false, false>(tx, ty, tz, a.x, a.y, b.x, b.y, acc, tab);
                }
            }
        }
    };

    while (sp > 0) {
        const int2 ent = stack[--sp];
        const int s = ent.x;
        const int b = S.begin[s], e = S.end[s];
        if (e == b) continue;
        const bool in = (unsigned(ent.y) >> lane) & 1u;
        // well_separated(target, 0, centre, radius, mac): R > 0 && 0 + r < mac R
        const double dx = __dsub_rn(x, S.cx[s]), dy = __dsub_rn(y, S.cy[s]), dz = __dsub_rn(z, S.cz[s]);
        const double R = __dsqrt_rn(dot_ref(dx, dy, dz, dx, dy, dz));
        const bool sep = R > 0.0 && __dadd_rn(0.0, S.rad[s]) < __dmul_rn(mac, R);
        const int nch = S.nchild[s];
        const bool pc = in && sep && (e - b > n0);
        const bool down = in && !sep && nch > 0;
        const bool pp = in && !pc && !down;
        const unsigned mdown = __ballot_sync(kFull, down);
        const unsigned mpc = __ballot_sync(kFull, pc), mpp = __ballot_sync(kFull, pp);
        // free of coincident pairs: the target is more than 1e-6 outside the sphere that holds
        // the proxies / the particles (the guard triggers below ~1.4e-7; unit vectors only —
        // known for the tree's own particles, so only when targets == sources)
        const bool gpc = !unit || !(R - S.qrad[s] > 1e-6), gpp = !unit || !(R - S.rad[s] > 1e-6);
        const bool guard_pc = __ballot_sync(kFull, pc && gpc) != 0, guard_pp = __ballot_sync(kFull, pp && gpp) != 0;
        __syncwarp();  // every lane has read this entry before its slot is overwritten
        if (mdown && sp + nch <= kStack) {  // the children in quadrant order (popped last to first)
            const int4 ch = S.child[s];
            const int cs[4] = {ch.x, ch.y, ch.z, ch.w};
            if (lane < nch) stack[sp + lane] = make_int2(cs[lane], int(mdown));
            sp += nch;
        }
        if (mpc) {
            evaluate(S.qx, S.qy, S.qz, qw, (long long)s * npp, npp, pc, guard_pc);
            npc += pc ? 1 : 0;
        }
        if (mpp) {
            evaluate(S.px, S.py, S.pz, sw, b, e - b, pp, guard_pp);
            npp_ += pp ? 1 : 0;
        }
        __syncwarp();  // the pushes are visible to the next pop
    }
    if (live) {
        const double sc = op.scale();
#pragma unroll
        for (int d = 0; d < D; ++d) out[i * D + d] = acc[d] * sc;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        npp_ += __shfl_xor_sync(kFull, npp_, o);
        npc += __shfl_xor_sync(kFull, npc, o);
    }
    if (lane == 0) {
        atomicAdd(&counts[0], npp_);
        atomicAdd(&counts[1], npc);
    }
}

}  // namespace

void cstc_eval(const KernelSpec& k, const double* txyz, long long nt, const int* order, const DeviceTree& src,
               double mac, int n0, const double2* log_tab, double* out, unsigned long long* counts,
               cudaStream_t s) {
    if (nt == 0) return;
    CSFS_CK(cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), s));
    const TreeView S = src.view();
    // CSFS_B200_CSTC=thread: the one-thread-per-target kernel (A/B and the bitwise cross-check)
    const char* mode = std::getenv("CSFS_B200_CSTC");
    const bool per_thread = mode && std::string(mode) == "thread";
    if (!per_thread) {
        with_op(k, [&](auto op) {
            auto kern = k_cstc_warp<decltype(op)>;
            CSFS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCstcWarpSmem)));
            kern<<<ceil_div(nt, kCstcWarpThreads), kCstcWarpThreads, kCstcWarpSmem, s>>>(
                txyz, nt, order, S, src.w, src.qw, mac, n0, op, log_tab, out, counts);
            CSFS_LAUNCH_CHECK();
        });
        return;
    }
    with_op(k, [&](auto op) {
        auto kern = k_cstc<decltype(op)>;
        CSFS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLogTabBytes)));
        kern<<<ceil_div(nt, kCstcThreads), kCstcThreads, kLogTabBytes, s>>>(txyz, nt, order, S, src.w, src.qw, mac, n0, op,
                                                                            log_tab, out, counts);
        CSFS_LAUNCH_CHECK();
    });
}

}  // namespace csfs_b200
