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
//   * source points + weights stream through shared memory in SoA chunks (coalesced
//     global loads, broadcast reads in the inner loop); targets stay in registers;
//   * small target sets (49/64/81/121) are packed G groups per CTA that split the source
//     range and are combined in a fixed order at the end.
// This is FP64-pipe bound: the inner loop is the kernel functor.
#include <algorithm>

#include "engine.hpp"
#include "kernels_dev.cuh"

namespace csfs_b200 {

namespace {

constexpr int kIB = 256;   // threads per CTA
constexpr int kICH = 256;  // source points per shared-memory chunk

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
};

template <class Op>
__global__ void __launch_bounds__(kIB) k_interact(InteractParams P, Op op) {
    constexpr int D = Op::dim;
    __shared__ double sx[kICH], sy[kICH], sz[kICH], sw[kICH];
    __shared__ double red[kIB * D];
    __shared__ int item_sh;
    const int tid = threadIdx.x;
    for (;;) {
        if (tid == 0) item_sh = atomicAdd(P.counter, 1);
        __syncthreads();
        const int it = item_sh;
        __syncthreads();
        if (it >= P.n_items) break;
        if (P.anchor) {
            const int a = P.anchor[it];
            if (a >= 0 && (a < P.own_b || a >= P.own_e)) continue;  // another rank's target
        }
        const int4 d = P.item[it];
        const bool tproxy = d.y < 0;
        const int tlen = tproxy ? -d.y : d.y;
        const int gs = min(kIB, (tlen + 31) & ~31);
        const int G = kIB / gs;
        const int g = tid / gs, r = tid - g * gs;
        const double* TX = tproxy ? P.tqx : P.tpx;
        const double* TY = tproxy ? P.tqy : P.tpy;
        const double* TZ = tproxy ? P.tqz : P.tpz;
        double* OUT = tproxy ? P.out_q : P.out_p;
        for (int t0 = 0; t0 < tlen; t0 += gs) {
            const int t = t0 + r;
            const bool active = g < G && t < tlen;
            double tx = 0.0, ty = 0.0, tz = 1.0;
            if (active) {
                tx = TX[d.x + t];
                ty = TY[d.x + t];
                tz = TZ[d.x + t];
            }
            double acc[D];
#pragma unroll
            for (int k = 0; k < D; ++k) acc[k] = 0.0;
            int fill = 0;
            auto compute = [&](int n) {
                if (active) {
#pragma unroll 2
                    for (int j = g; j < n; j += G) op(tx, ty, tz, sx[j], sy[j], sz[j], sw[j], acc);
                }
            };
            for (int e = d.z; e < d.w; ++e) {
                const int2 sg = P.seg[e];
                const bool sproxy = sg.y < 0;
                const int len = sproxy ? -sg.y : sg.y;
                const double* X = sproxy ? P.sqx : P.spx;
                const double* Y = sproxy ? P.sqy : P.spy;
                const double* Z = sproxy ? P.sqz : P.spz;
                const double* W = sproxy ? P.sqw : P.spw;
                int pos = 0;
                while (pos < len) {
                    const int take = min(len - pos, kICH - fill);
                    for (int j = tid; j < take; j += kIB) {
                        const long long src = (long long)sg.x + pos + j;
                        sx[fill + j] = X[src];
                        sy[fill + j] = Y[src];
                        sz[fill + j] = Z[src];
                        sw[fill + j] = W[src];
                    }
                    fill += take;
                    pos += take;
                    if (fill == kICH) {
                        __syncthreads();
                        compute(fill);
                        __syncthreads();
                        fill = 0;
                    }
                }
            }
            if (fill) {
                __syncthreads();
                compute(fill);
                __syncthreads();
            }
            if (G > 1) {
                if (active)
#pragma unroll
                    for (int k = 0; k < D; ++k) red[(g * gs + r) * D + k] = acc[k];
                __syncthreads();
                if (g == 0 && t < tlen) {
                    for (int h = 1; h < G; ++h)
#pragma unroll
                        for (int k = 0; k < D; ++k) acc[k] += red[(h * gs + r) * D + k];
                }
                __syncthreads();
            }
            if (g == 0 && t < tlen) {
                const double sc = op.scale();
#pragma unroll
                for (int k = 0; k < D; ++k) OUT[(long long)(d.x + t) * D + k] = acc[k] * sc;
            }
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
    const long long t0 = (long long)i * kIB;
    item[i] = make_int4(int(t0), int(min((long long)kIB, nt - t0)), 0, nseg);
}

template <class F>
void with_op(const KernelSpec& k, F&& f) {
    switch (k.kind) {
        case 0: f(OpLaplace{}); break;
        case 1: f(OpBiharmonic{}); break;
        case 2: f(OpBiotSavart{}); break;
        default: {
            OpSal op;
            op.pref = 3.0 * k.rho_ratio * kInv4Pi;
            op.c1 = 1.0 - k.b0;
            op.c2 = k.a1 - k.b1;
            f(op);
        }
    }
}

template <class Op>
int grid_for(int n_items) {
    int dev = 0, sms = 0, per = 0;
    CSFS_CK(cudaGetDevice(&dev));
    CSFS_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CSFS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_interact<Op>, kIB, 0));
    return std::max(1, std::min(n_items, sms * std::max(per, 1)));
}

template <class Op>
void launch(const InteractParams& p, const Op& op, cudaStream_t s) {
    if (p.n_items == 0) return;
    CSFS_CK(cudaMemsetAsync(p.counter, 0, sizeof(int), s));
    k_interact<Op><<<grid_for<Op>(p.n_items), kIB, 0, s>>>(p, op);
    CSFS_LAUNCH_CHECK();
}

}  // namespace

void interact(const KernelSpec& k, const DeviceTree& tgt, const DeviceTree& src, const Items& items,
              double* phi_near, int* work_counter, cudaStream_t s, Own own) {
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
    with_op(k, [&](auto op) { launch(p, op, s); });
}

void direct_allpairs(const KernelSpec& k, const double* txyz, long long nt, const double* sxyz,
                     const double* sw, long long ns, double* out, DevBuf<double>& soa,
                     DevBuf<int4>& items, DevBuf<int2>& segs, int* work_counter, cudaStream_t s) {
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
    const long long kSeg = 1 << 30;
    for (long long b = 0; b < ns; b += kSeg) hseg.push_back(make_int2(int(b), int(std::min(kSeg, ns - b))));
    const int nseg = int(hseg.size());
    segs.grow(std::max(nseg, 1));
    if (nseg) CSFS_CK(cudaMemcpyAsync(segs.p, hseg.data(), nseg * sizeof(int2), cudaMemcpyHostToDevice, s));
    const int n_items = ceil_div(nt, kIB);
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
    with_op(k, [&](auto op) { launch(p, op, s); });
    CSFS_CK(cudaStreamSynchronize(s));  // hseg lifetime
}

}  // namespace csfs_b200
