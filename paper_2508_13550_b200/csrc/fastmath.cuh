// FP64 elementary functions for the evaluation kernel, sized to the FP64 pipe budget.
//
// The evaluation phases are FP64-issue bound.  libdevice's log is
// ~28 FP64 instructions, sqrt and a/b ~8 each; the kernel functors need:
//   log   -> Tang-style table method with an accurate table (Gal): x = 2^k m with
//            m in [0.7070, 1.4141), m r_i / LAM = 1 + t, |t| <= 2^-13, from a 4096-entry
//            table of {r_i, L_i} (64 KB, dynamic shared memory; tools/gen_log_table.c):
//            r_i is stored scaled by LAM = fl(1/sqrt(3)) and chosen so that
//            L_i = -ln(r_i / LAM) is within 2^-67 of the 2^-46 grid: one LDS.128 per lookup.
//            t' = fma(m, r_i, -LAM) = LAM t (one rounding at |t'| < 2^-13), and with
//            LAM^2 = 1/3 the degree-3 log1p t + c2 t^2 + t^3/3 becomes
//            (t' + t'^2 (t' + c2/LAM)) / LAM: a DADD and two DFMA whose constants all sit in
//            uniform registers (no per-pair materialised constant), k ln2 + L_i in one FMA:
//            6 FP64 instructions (+ one int->double conversion).  c2 = -1/2 - (sqrt2-1)/2 h^2
//            (h = 2^-13) balances the truncated t^4/4 term: |error| <= 0.043 h^4 = 9.5e-18
//            ABSOLUTE + rounding (~1 ulp) — what the kernels consume: every log is added to
//            O(1) terms or multiplied by an O(10) factor (tests/test_gpu_numerics.py).  m = 1
//            sits mid-interval ([1 - 2^-14, 1 + 2^-13), r = LAM, L = 0): log(1) = 0 exactly
//            (t = m - 1 exact up to the LAM scaling).  Domain: positive normals.
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

constexpr int kLogOff = 0x3fe6a080;  // high word of the lowest m (~0.7071); m = 1 mid-interval
constexpr double kLn2 = 0x1.62e42fefa39efp-1;
constexpr double kLogLam = 0x1.279a74590331cp-1;    // fl(1/sqrt(3)): the table's r_i scale
constexpr double kLogMu = 0x1.bb67ae8584cabp+0;     // fl(1/kLogLam)
constexpr double kLogKappa = -0x1.bb67aeb36f4fbp-1; // c2 / kLogLam, c2 = -1/2 - (sqrt2-1)/2 2^-26

__device__ __forceinline__ double fast_log(double x, const LogTable& tb) {
    const int hi = __double2hiint(x);
    const int d = hi - kLogOff;
    const int k = d >> 20;  // arithmetic shift: x = 2^k m, m in [0.7070, 1.4141)
    const int i = (d >> (20 - kLogTabBits)) & (kLogTab - 1);
    // hi - k 2^20 as ONE integer multiply-add (written as k << 20 the compiler forms
    // d & 0xfff00000 and a subtraction: two instructions per log)
    int mhi;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(mhi) : "r"(k), "n"(-1048576), "r"(hi));
    const double m = __hiloint2double(mhi, __double2loint(x));
    const double2 e = tb.e[i];
    const double tp = fma(m, e.x, -kLogLam);        // LAM t, |t| <= 2^-13
    const double q = fma(tp * tp, tp + kLogKappa, tp);  // LAM log1p(t)
    // k ln2 + L_i in one FMA (k ln2 rounded once inside it; |k| <= 1 for most arguments)
    const double A = fma(double(k), kLn2, e.y);
    return fma(q, kLogMu, A);
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
