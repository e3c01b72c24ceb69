// FP64 elementary functions for the evaluation kernel, sized to the FP64 pipe budget.
//
// The evaluation phases are FP64-issue bound.  libdevice's log is
// ~28 FP64 instructions, sqrt and a/b ~8 each; the kernel functors need:
//   log   -> Tang-style table method with an accurate table (Gal): x = 2^k m with
//            m in [0.7070, 1.4141) (so both sides of x = 1 have k = 0), m r_i = 1 + t,
//            |t| <= 2^-11, from a 2048-entry table of {r_i, L_i} (32 KB, dynamic shared
//            memory): r_i is chosen near 1/centre_i so that L_i = -ln r_i is within 2^-67
//            of the 2^-46 grid (tools/gen_log_table.c): one LDS.128 per lookup.  The two
//            intervals around 1 use r = 1, L = 0, so t = m - 1 is exact — branch-free.
//            k ln2 + L_i in one FMA, log1p(t) by a degree-4 polynomial: 7 FP64
//            instructions (+ one int->double conversion).  Error <= 1 ulp + |t|^5/5
//            (<= 5.6e-18 absolute, reached only in the interval just above 1, where the value
//            is ~t: up to ~100 ulp RELATIVE there); the kernels add log to O(1) terms, so
//            only the absolute error reaches them (tests/test_gpu_numerics.py).  Domain:
//            positive normals.
//   rsqrt -> MUFU.RSQ64H seed + one cubic-convergent correction (5 FP64), <= 2 ulp.
//   rcp   -> MUFU.RCP64H seed + one cubic-convergent correction (3 FP64), <= 2 ulp.
// Arguments are finite positive normals (the coincidence guard keeps 1 - x.y >= 1e-14).
#pragma once

#include "common.cuh"

namespace csfs_b200 {

// Global table (host-built by make_log_table from log_table.inc): kLogTab double2 {r_i, L_i}.
// The evaluation kernels stage it into dynamic shared memory (kLogTabBytes) per CTA.
struct LogTable {
    const double2* e;  // kLogTab
};
constexpr size_t kLogTabBytes = size_t(kLogTab) * sizeof(double2);

// Copies the global table into shared memory `sm` (kLogTab entries); the caller syncs
// before use.
__device__ __forceinline__ LogTable stage_log_table(double2* sm, const double2* g) {
    for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) sm[i] = g[i];
    return LogTable{sm};
}

constexpr int kLogOff = 0x3fe6a000;              // high word of the lowest m (~0.70703)
constexpr double kLn2 = 0x1.62e42fefa39efp-1;

__device__ __forceinline__ double fast_log(double x, const LogTable& tb) {
    const int hi = __double2hiint(x);
    const int d = hi - kLogOff;
    const int k = d >> 20;  // arithmetic shift: x = 2^k m, m in [0.7070, 1.4141)
    const int i = (d >> (20 - kLogTabBits)) & (kLogTab - 1);
    const double m = __hiloint2double(hi - (k << 20), __double2loint(x));
    const double2 e = tb.e[i];
    // |t| <= 2^-11; exact for the two intervals around m = 1 (r = 1)
    const double t = fma(m, e.x, -1.0);
    const double p = fma(fma(-1.0 / 4.0, t, 1.0 / 3.0), t, -1.0 / 2.0);
    // k ln2 + L_i in one FMA (k ln2 rounded once inside it; |k| <= 1 for most arguments)
    const double A = fma(double(k), kLn2, e.y);
    return A + fma(t * t, p, t);
}

__device__ __forceinline__ double rsqrt_seed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

__device__ __forceinline__ double rcp_seed(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

// 1/sqrt(x): y0 (~2^-23) then y = y0 (1 + e/2 + 3e^2/8), e = 1 - x y0^2  (error ~e^3)
__device__ __forceinline__ double fast_rsqrt(double x) {
    const double y = rsqrt_seed(x);
    const double h = x * y;
    const double e = fma(-h, y, 1.0);
    const double c = e * fma(e, 0.375, 0.5);
    return fma(y, c, y);
}

// 1/x: y0 then y = y0 (1 + e + e^2), e = 1 - x y0  (error ~e^3)
__device__ __forceinline__ double fast_rcp(double x) {
    const double y = rcp_seed(x);
    const double e = fma(-x, y, 1.0);
    return fma(y, fma(e, e, e), y);
}

// bary_basis_1d (interpolation.cpp:26-43) for the per-particle P2M / L2P bases: the same
// node-coincidence test and summation order, with the np + 1 IEEE divisions replaced by
// fast reciprocals (<= 2 ulp each; proxy weights/potentials move by ~1e-16 relative).
// NP > 0: compile-time node count (fully unrolled, `out` stays in registers); 0: c.np.
template <int NP = 0>
__device__ __forceinline__ void bary1d_fast(const Cheb& c, double x, double* out) {
    const int np = NP > 0 ? NP : c.np;
    bool hit = false;
#pragma unroll
    for (int k = 0; k < (NP > 0 ? NP : kMaxNp); ++k)
        if (k < np) {
            const bool h = fabs(x - c.nodes[k]) < kNodeTol;
            out[k] = h ? 1.0 : 0.0;  // indicator if some node coincides (first one wins below)
            hit = hit || h;
        }
    if (hit) {
        bool seen = false;  // the reference returns the FIRST coincident node's indicator
#pragma unroll
        for (int k = 0; k < (NP > 0 ? NP : kMaxNp); ++k)
            if (k < np) {
                if (seen) out[k] = 0.0;
                seen = seen || out[k] != 0.0;
            }
        return;
    }
    double denom = 0.0;
#pragma unroll
    for (int k = 0; k < (NP > 0 ? NP : kMaxNp); ++k)
        if (k < np) {
            const double q = c.weights[k] * fast_rcp(x - c.nodes[k]);
            out[k] = q;
            denom += q;
        }
    const double inv = fast_rcp(denom);
#pragma unroll
    for (int k = 0; k < (NP > 0 ? NP : kMaxNp); ++k)
        if (k < np) out[k] *= inv;
}

}  // namespace csfs_b200
