// FP64 elementary functions for the evaluation kernel, sized to the FP64 pipe budget.
//
// The evaluation phases are FP64-issue bound.  libdevice's log is
// ~28 FP64 instructions, sqrt and a/b ~8 each; the kernel functors need:
//   log   -> Tang-style table method: x = 2^e m, m r_i = 1 + t with |t| <= 2^-9 from a
//            512-entry shared-memory table of 16-byte entries {L_hi_i, r_i | L_lo_i}:
//            -ln r_i = L_hi + L_lo with L_hi a full double on the 2^-42 grid (so
//            e ln2_hi + L_hi is exact) while r_i and L_lo carry 21 significant bits and are
//            stored as the high words of doubles (the low words are zero): one LDS.128 per
//            lookup.  log1p(t) by a degree-6 polynomial.  The two intervals touching
//            x = 1 use r = 1 and r = 1/2 exactly, so t is exact and the result keeps full
//            relative accuracy where log(x) ~ 0 — branch-free.  12 FP64 instructions
//            (+ one int->double conversion on the XU pipe), <= 1 ulp (mpmath check in
//            tests/test_gpu_numerics.py).
//   rsqrt -> MUFU.RSQ64H seed + one cubic-convergent correction (5 FP64), <= 2 ulp.
//   rcp   -> MUFU.RCP64H seed + one cubic-convergent correction (3 FP64), <= 2 ulp.
// Arguments are finite positive normals (the coincidence guard keeps 1 - x.y >= 1e-14).
#pragma once

#include "common.cuh"

namespace csfs_b200 {

// Global table (host-built by make_log_table, kLogTab double2): .x = L_hi_i, .y = the
// 64-bit word {hi: high word of r_i, lo: high word of L_lo_i}.  Staged into shared memory
// per CTA.
struct LogTable {
    const double2* e;  // kLogTab
#if !CSFS_LOG_PACK
    const double* lo;  // kLogTab
#endif
};

struct LogTableSmem {
    double2 e[kLogTab];
#if !CSFS_LOG_PACK
    double lo[kLogTab];
#endif
};

// Copies the global table into shared memory; the caller syncs before use.
__device__ __forceinline__ LogTable stage_log_table(LogTableSmem& sm, const double2* g) {
#if CSFS_LOG_PACK
    for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) sm.e[i] = g[i];
    return LogTable{sm.e};
#else
    for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) {
        sm.e[i] = g[i];
        sm.lo[i] = g[kLogTab + i].x;
    }
    return LogTable{sm.e, sm.lo};
#endif
}

constexpr double kLn2Hi = 0x1.62e42fefa3800p-1;  // 42 significant bits: e*kLn2Hi exact
constexpr double kLn2Lo = 0x1.ef358p-45;         // ln 2 - kLn2Hi to 21 bits (|err| < 2^-66)

__device__ __forceinline__ double fast_log(double x, const LogTable& tb) {
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const int e = ((hi >> 20) & 0x7ff) - 1023;
    const int i = (hi >> (20 - kLogTabBits)) & (kLogTab - 1);
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
    const double2 ent = tb.e[i];
#if CSFS_LOG_PACK
    const double r = __hiloint2double(__double2hiint(ent.y), 0);
    const double L_lo = __hiloint2double(__double2loint(ent.y), 0);
#else
    const double r = ent.y, L_lo = tb.lo[i];
#endif
    // |t| <= 2^-9; exact for the two intervals touching x = 1 (r = 1 and r = 1/2)
    const double t = fma(m, r, -1.0);
#if CSFS_LOG_BITS >= 9
    double p = -1.0 / 6.0;
#else
    double p = 1.0 / 7.0;
    p = fma(p, t, -1.0 / 6.0);
#endif
    p = fma(p, t, 1.0 / 5.0);
    p = fma(p, t, -1.0 / 4.0);
    p = fma(p, t, 1.0 / 3.0);
    p = fma(p, t, -1.0 / 2.0);
    const double ed = double(e);
    const double small = fma(ed, kLn2Lo, L_lo);
    const double q = fma(t * t, p, small);
    const double A = fma(ed, kLn2Hi, ent.x);  // exact: both are multiples of 2^-42
    return A + (t + q);
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
