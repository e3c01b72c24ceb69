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


}  // namespace

void cstc_eval(const KernelSpec& k, const double* txyz, long long nt, const int* order, const DeviceTree& src,
               double mac, int n0, const double2* log_tab, double* out, unsigned long long* counts,
               cudaStream_t s) {
    if (nt == 0) return;
    CSFS_CK(cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), s));
    const TreeView S = src.view();
    with_op(k, [&](auto op) {
        auto kern = k_cstc<decltype(op)>;
        CSFS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLogTabBytes)));
        kern<<<ceil_div(nt, kCstcThreads), kCstcThreads, kLogTabBytes, s>>>(txyz, nt, order, S, src.w, src.qw, mac, n0, op,
                                                                            log_tab, out, counts);
        CSFS_LAUNCH_CHECK();
    });
}

}  // namespace csfs_b200
