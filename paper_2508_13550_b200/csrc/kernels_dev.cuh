// Device kernel functors: the B200 form of the reference's private ops
// LaplaceOp / BiharmonicOp / BiotSavartOp / SalOp (/root/reference/proj/src/summation.cpp:32-77)
// and of dilog (kernels.cpp:13-51).
//
// Same shape as the reference op (static dim; evaluate one (x, y) pair and accumulate
// w * K(x, y)), re-derived for the FP64 pipe:
//  * `x.y` and `1 - x.y` are evaluated unfused in the reference's order (dot_ref), so the
//    near-neighbour cancellation is identical to the reference's build;
//  * the coincidence guard `1 - x.y < 1e-14` is predicated (a safe argument is evaluated
//    and the weight zeroed) instead of branched: no divergence, exact skip semantics; the
//    compare itself runs on the integer pipe (not_coincident, common.cuh);
//  * the prefactor (-1/4pi, 1/4pi, 3 rho/4pi) is applied once per target (`scale`);
//  * log / rsqrt / rcp come from fastmath.cuh (6 / 5 / 3 FP64 instructions instead of
//    libdevice's ~28 / 8+8 / 8), each within a few ulp;
//  * SAL: targets enter halved, so hom = 0.5 - t'.s = omc/2 exactly; 2/gamma = 1/s =
//    rsqrt(hom) with s = gamma/2, and log(s (1 + s)) = log(s + s^2) = log(fma(hom, 1/s,
//    hom)) since s^2 = hom — the reference's formula, without sqrt, divide, a seed rescale
//    or s itself.
#pragma once

#include "common.cuh"
#include "fastmath.cuh"

namespace csfs_b200 {

// one - x.y: F = false in the reference's unfused order (dot_ref, then one subtraction:
// 6 FP64 instructions, the reference's rounding); F = true as three fused multiply-adds
// (3 instructions).  Both forms are within a few ulp of 1 of the exact value, so they
// differ by at most ~8e-16 absolutely, i.e. 8e-16 / (1 - x.y) relatively: the fused form
// is only used on list entries whose point sets are provably more than kFuseGap apart
// (traverse.cu can_fuse: 1 - x.y >= kFuseGap^2 / 2 = 1e-5), where the per-pair difference
// in 1 - x.y is below 8e-11 relatively in the worst case.  Exact products
// commute, so the fused form keeps K(t, s) = kSym K(s, t) bit for bit (the symmetric kernel).
template <bool F>
__device__ __forceinline__ double one_minus_dot(double one, double tx, double ty, double tz, double sx, double sy,
                                                double sz) {
    if (F) return fma(-tz, sz, fma(-ty, sy, fma(-tx, sx, one)));
    return __dsub_rn(one, dot_ref(tx, ty, tz, sx, sy, sz));
}

// Each op also provides value(): the unscaled, guarded K(t, s) (0 where the guard skips),
// used by the symmetric PP/CC path, which applies one evaluation to both the target's row
// and the source's column; kSym: K(s, t) = kSym * K(t, s) (exactly: the unfused dot and
// cross products commute bit-for-bit).  eval<G> / value<G>: G = false drops the
// coincidence guard, for list entries proven free of pairs with 1 - x.y < 1e-14
// (needs_guard, traverse.cu) — the same values with 5 fewer issue slots per pair.
struct OpLaplace {
    static constexpr int kMinBlocks = 3;  // k_interact CTAs per SM (interact.cu MinBlocksOf)
    static constexpr bool kFusable = true;  // has a fused 1 - x.y form (one_minus_dot<true>)
    static constexpr int dim = 1;
    static constexpr int kUnroll = 16;  // k_interact source-loop unroll
    static constexpr double kSym = 1.0;
    __device__ __forceinline__ static double tgt(double x) { return x; }
    __device__ __forceinline__ double scale() const { return -kInv4Pi; }
    template <bool G = true, bool F = false>
    __device__ __forceinline__ void value(double tx, double ty, double tz, double sx, double sy, double sz,
                                          double* K, const LogTable& tab) const {
        const double omc = one_minus_dot<F>(1.0, tx, ty, tz, sx, sy, sz);
        const bool ok = !G || not_coincident(omc);
        const double v = fast_log(G ? safe_omc(ok, omc) : omc, tab);
        K[0] = ok ? v : 0.0;
    }
    template <bool G = true, bool F = false>
    __device__ __forceinline__ void eval(double tx, double ty, double tz, double sx, double sy, double sz, double sw,
                                         double* acc, const LogTable& tab) const {
        const double omc = one_minus_dot<F>(1.0, tx, ty, tz, sx, sy, sz);
        const bool ok = !G || not_coincident(omc);
        const double v = fast_log(G ? safe_omc(ok, omc) : omc, tab);
        acc[0] = fma(ok ? sw : 0.0, v, acc[0]);
    }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc,
                                               const LogTable& tab) const {
        eval<true>(tx, ty, tz, sx, sy, sz, sw, acc, tab);
    }
};

// Li2 on the kernel's domain u in [0, 1] (u = min(1, (1 + x.y)/2) >= -1e-16).
// Reference (kernels.cpp:13-51): reflection Li2(u) = pi^2/6 - ln(u) ln(1-u) - Li2(1-u) for
// u > 1/2, then the power series of Li2 on [0, 1/2] (up to 80 terms, each a division).
// Here the base region uses the Bernoulli series Li2(y) = sum_n B_n z^(n+1)/(n+1)! with
// z = -ln(1-y) in [0, ln 2]: the terms through B14 z^15/15!, a degree-6 Horner polynomial in
// z^2 (no divisions); the first dropped term, B16 z^17/17!, is <= 3.9e-17 (6.7e-17
// relative, 0.6 ulp) at z = ln 2 and falls off as z^17.  For u > 1/2, z = -ln(u) is the
// log already needed by the reflection term, so that branch costs two logs, the other one.
__device__ __forceinline__ double li2_bernoulli(double z) {
    const double w = z * z;
    double p = 0x1.f63f1e311ac24p-41;  // B14/15!
    p = fma(p, w, -0x1.658a4b8f16a75p-35);
    p = fma(p, w, 0x1.04d7f65caf373p-29);
    p = fma(p, w, -0x1.8a86a49f629d1p-24);
    p = fma(p, w, 0x1.3d079fb6ef3e3p-18);
    p = fma(p, w, -0x1.23456789abcdfp-12);
    p = fma(p, w, 0x1.c71c71c71c71cp-6);  // B2/3! = 1/36
    // z - z^2/4 + z^3 p(z^2) = z + z^2 (z p - 1/4): two FMAs after the Horner chain; the
    // rounding of (z p - 1/4) moves the result by <= z^2/4 2^-53 <= 1.3e-17 absolutely
    return fma(w, fma(z, p, -0.25), z);
}

// C = false: z = -log(t) without the compensation term, which only corrects t's own
// rounding (<= 2^-53 absolutely) — 4 FP64 instructions and a MUFU fewer (kept for A/B; the
// kernels use C = true here and dilog_far on the provably far entries).
// Branch-free: both regions run the same instructions on selected operands — the log of
// a = (u > 1/2 ? u : 1 - u) gives z, the second log is ln(1 - u) for the reflection term
// (of 1.0 below 1/2: exactly 0, unused) — because a data-dependent branch around every
// evaluation (BSSY / BRA / BSYNC) keeps the compiler from interleaving the independent
// evaluations of a source batch: the biharmonic loops then ran one dependent FP64 chain at
// a time per warp (41% FP64 pipe, "wait" the top stall, ncu round 2).  Nearly every
// evaluation has u > 1/2 (x.y > 0: all PP / CP and the deep CC entries), which needed both
// logs before too; the few below 1/2 now pay a second log.
template <bool C = true>
__device__ __forceinline__ double dilog_dev(double u, const LogTable& tab) {
    constexpr double kPi2Over6 = kPi * kPi / 6.0;
    const bool hi = u > 0.5;
    const double t = 1.0 - u;  // exact for u > 1/2 (Sterbenz); 0 only when u == 1 (selected away)
    const double la = fast_log(hi ? u : t, tab);
    const double lb = fast_log(hi ? t : 1.0, tab);
    double z = -la;
    if (C) {
        // u <= 1/2: z = -log1p(-u) via the compensated form log(t) - ((t - 1) + u)/t: the
        // correction (t - 1) + u is t's rounding error (|.| <= 2^-53), so the bare MUFU
        // reciprocal (2^-20) is enough — it moves z by < 2^-72
        const double zc = -(la - ((t - 1.0) + u) * rcp_seed(t));
        z = hi ? z : zc;
    }
    const double li = li2_bernoulli(z);
    const double r = kPi2Over6 - la * lb - li;  // the reflection Li2(u) = pi^2/6 - ln u ln(1-u) - Li2(1-u)
    return hi ? ((u == 1.0) ? kPi2Over6 : r) : li;
}

// The provably far entries (kSegFused: every pair within one hemisphere and > kFuseGap apart,
// so 1/2 + 2.9e-3 <= u <= 1 - 5e-6): always the reflection region, no select, no clamp, no
// u == 1 case — bit for bit what dilog_dev<false> returns there.
__device__ __forceinline__ double dilog_far(double u, const LogTable& tab) {
    constexpr double kPi2Over6 = kPi * kPi / 6.0;
    const double la = fast_log(u, tab);
    const double lb = fast_log(1.0 - u, tab);  // 1 - u exact (Sterbenz)
    return kPi2Over6 - la * lb - li2_bernoulli(-la);
}

// BiharmonicOp: dilog(u) / 4pi, u = min(1, (1 + x.y)/2).  Targets enter halved (exact), so
// the reference's 0.5 (1 + x.y) is 0.5 + t'.s bit for bit (scaling by 2 commutes with the
// roundings): unfused in the reference's order, one DMUL fewer.  On the provably far entries
// (F) u is three FMAs; it then differs from the reference's rounding by a few ulp of 1,
// which moves the kernel by <= |dilog'(u)| 4e-16 = |ln(1 - u)/u| 4e-16 <= 5e-15 absolutely
// (1 - u >= 5e-6 there) — u = (1 + x.y)/2 has no near-coincidence cancellation to
// preserve.  The symmetric kernel keeps K(t, s) = K(s, t) bit for bit (exact products commute).
#ifndef CSFS_BIH_MINB
#define CSFS_BIH_MINB 3
#endif
#ifndef CSFS_BIH_UNROLL
#define CSFS_BIH_UNROLL 8
#endif
struct OpBiharmonic {
    static constexpr int kMinBlocks = CSFS_BIH_MINB;
    static constexpr bool kFusable = true;  // has a fused form (u from three FMAs)
    static constexpr int dim = 1;
    static constexpr int kUnroll = CSFS_BIH_UNROLL;
    static constexpr double kSym = 1.0;
    __device__ __forceinline__ static double tgt(double x) { return 0.5 * x; }
    __device__ __forceinline__ double scale() const { return kInv4Pi; }
    // the reference's u = min(1, 0.5 (1 + x.y)), unfused, in its order
    __device__ __forceinline__ static double u_ref(double tx, double ty, double tz, double sx, double sy, double sz) {
        const double u0 = __dadd_rn(0.5, dot_ref(tx, ty, tz, sx, sy, sz));
        return (u0 < 1.0) ? u0 : 1.0;  // std::min(1.0, u0)
    }
    template <bool G = true, bool F = false>  // regular at coincidence: no guard either way
    __device__ __forceinline__ void value(double tx, double ty, double tz, double sx, double sy, double sz,
                                          double* K, const LogTable& tab) const {
        K[0] = F ? dilog_far(fma(tz, sz, fma(ty, sy, fma(tx, sx, 0.5))), tab)
                 : dilog_dev<true>(u_ref(tx, ty, tz, sx, sy, sz), tab);
    }
    template <bool G = true, bool F = false>
    __device__ __forceinline__ void eval(double tx, double ty, double tz, double sx, double sy, double sz, double sw,
                                         double* acc, const LogTable& tab) const {
        double K[1];
        value<G, F>(tx, ty, tz, sx, sy, sz, K, tab);
        acc[0] = fma(sw, K[0], acc[0]);
    }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc,
                                               const LogTable& tab) const {
        eval<true>(tx, ty, tz, sx, sy, sz, sw, acc, tab);
    }
};

struct OpBiotSavart {
    static constexpr bool kFusable = true;  // has a fused 1 - x.y form (one_minus_dot<true>)
    // far entries (the fused ones): sum_s a_s (t x s) = t x (sum_s a_s s), a_s = w_s/(1 - t.s):
    // eval_far accumulates the moment sum_s a_s s (3 FMAs per pair instead of a cross product
    // and 3 FMAs) and far_finish adds t x moment once per target.  Far pairs are > kFuseGap
    // apart, so the moment has no near-coincidence cancellation to preserve.
#ifndef CSFS_BS_FAR_MOMENT
#define CSFS_BS_FAR_MOMENT 1
#endif
    static constexpr bool kFarFactored = CSFS_BS_FAR_MOMENT;
    static constexpr int dim = 3;
    __device__ __forceinline__ void eval_far(double tx, double ty, double tz, double sx, double sy, double sz,
                                             double sw, double* m, const LogTable&) const {
        const double omc = one_minus_dot<true>(1.0, tx, ty, tz, sx, sy, sz);
        const double a = sw * fast_rcp(omc);
        m[0] = fma(a, sx, m[0]);
        m[1] = fma(a, sy, m[1]);
        m[2] = fma(a, sz, m[2]);
    }
    __device__ __forceinline__ static void far_finish(double tx, double ty, double tz, const double* m, double* acc) {
        acc[0] += fma(ty, m[2], -(tz * m[1]));
        acc[1] += fma(tz, m[0], -(tx * m[2]));
        acc[2] += fma(tx, m[1], -(ty * m[0]));
    }
    static constexpr double kSym = -1.0;  // cross(s, t) = -cross(t, s), 1 - s.t = 1 - t.s
    __device__ __forceinline__ static double tgt(double x) { return x; }
    __device__ __forceinline__ double scale() const { return -kInv4Pi; }
    template <bool G = true, bool F = false>
    __device__ __forceinline__ void value(double tx, double ty, double tz, double sx, double sy, double sz,
                                          double* K, const LogTable&) const {
        const double omc = one_minus_dot<F>(1.0, tx, ty, tz, sx, sy, sz);
        const bool ok = !G || not_coincident(omc);
        const double a = ok ? fast_rcp(G ? safe_omc(ok, omc) : omc) : 0.0;
        K[0] = a * __dsub_rn(__dmul_rn(ty, sz), __dmul_rn(tz, sy));
        K[1] = a * __dsub_rn(__dmul_rn(tz, sx), __dmul_rn(tx, sz));
        K[2] = a * __dsub_rn(__dmul_rn(tx, sy), __dmul_rn(ty, sx));
    }
    template <bool G = true, bool F = false>
    __device__ __forceinline__ void eval(double tx, double ty, double tz, double sx, double sy, double sz, double sw,
                                         double* acc, const LogTable&) const {
        const double omc = one_minus_dot<F>(1.0, tx, ty, tz, sx, sy, sz);
        const bool ok = !G || not_coincident(omc);
        const double a = (ok ? sw : 0.0) * fast_rcp(G ? safe_omc(ok, omc) : omc);
        // cross(x, y) unfused, in the reference's order (geometry.hpp:20-22): for close
        // pairs the components cancel, and a contracted form would differ from it.  On the
        // provably far entries that take the fused 1 - x.y (F) the contracted form is used
        // too: it differs by < 1 ulp of the products, an absolute ~1e-16 on O(1) terms.
        double cx, cy, cz;
#ifndef CSFS_BS_FUSED_CROSS
#define CSFS_BS_FUSED_CROSS 1
#endif
        if (F && CSFS_BS_FUSED_CROSS) {
            cx = fma(ty, sz, -(tz * sy));
            cy = fma(tz, sx, -(tx * sz));
            cz = fma(tx, sy, -(ty * sx));
        } else {
            cx = __dsub_rn(__dmul_rn(ty, sz), __dmul_rn(tz, sy));
            cy = __dsub_rn(__dmul_rn(tz, sx), __dmul_rn(tx, sz));
            cz = __dsub_rn(__dmul_rn(tx, sy), __dmul_rn(ty, sx));
        }
        acc[0] = fma(a, cx, acc[0]);
        acc[1] = fma(a, cy, acc[1]);
        acc[2] = fma(a, cz, acc[2]);
    }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc, const LogTable& tab) const {
        eval<true>(tx, ty, tz, sx, sy, sz, sw, acc, tab);
    }
};

// SalOp (summation.cpp:63-76): pref (c1/gamma - c2 log(s (1 + s))), gamma = sqrt(2 omc),
// s = gamma/2.  The constant c1 is folded into scale() (one FMA per pair instead of a
// multiply and an FMA): K' = 2/gamma + k log(s (1 + s)), k = -2 c2/c1, scale = pref c1 / 2
// (the factor 2 comes from the halved targets, below).  The c1 == 0 case (pure log
// kernel) is the kLogOnly instantiation: K' = log(...), scale = -pref c2.
template <bool kLogOnly>
#ifndef CSFS_SAL_UNROLL
#define CSFS_SAL_UNROLL 16
#endif
#ifndef CSFS_SAL_MINB
#define CSFS_SAL_MINB 2
#endif
struct OpSalT {
    static constexpr bool kFusable = true;
    static constexpr int dim = 1;
    static constexpr int kUnroll = CSFS_SAL_UNROLL;
    static constexpr int kMinBlocks = CSFS_SAL_MINB;
    static constexpr double kSym = 1.0;
    double scale_, k;
    __host__ static OpSalT make(double pref, double c1, double c2) {
        OpSalT op;
        op.scale_ = kLogOnly ? -pref * c2 : 0.5 * (pref * c1);
        op.k = kLogOnly ? 0.0 : -2.0 * (c2 / c1);
        return op;
    }
    __device__ __forceinline__ double scale() const { return scale_; }
    // Targets enter halved (exact): every product of the dot, the dot itself and
    // hom = 0.5 - t'.s are then exactly half of the reference's, so hom = omc/2 bit for bit
    // and the guard compares it with 1e-14/2.  The MUFU seed is taken on hom directly:
    // y ~ 1/sqrt(hom) = 2/gamma.
    __device__ __forceinline__ static double tgt(double x) { return 0.5 * x; }
    // 2/gamma and log(s (1 + s)), s = gamma/2 = sqrt(hom): cubic correction of the seed,
    // e = 1 - hom y^2, c = e/2 + 3e^2/8, 2/gamma = 1/s = y (1 + c); then s (1 + s) = s + s^2
    // = hom (1/s) + hom in ONE fma (s^2 = hom: no separate s), within ~3 ulp like the
    // s-then-fma(s, s, s) form it replaces.  Returns 2/gamma + 2k log(...) (scale() carries
    // the 1/2), or the log alone.
    __device__ __forceinline__ double kernel(double hom, const LogTable& tab) const {
        const double y = rsqrt_seed(hom);
        const double h = hom * y;
        const double e = fma(-h, y, 1.0);
        const double c = e * fma(e, 0.375, 0.5);
        const double r2 = fma(y, c, y);  // 2/gamma = 1/s
        const double L = fast_log(fma(hom, r2, hom), tab);
        return kLogOnly ? L : fma(k, L, r2);
    }
    template <bool G = true, bool F = false>
    __device__ __forceinline__ void value(double tx, double ty, double tz, double sx, double sy, double sz,
                                          double* K, const LogTable& tab) const {
        const double hom = one_minus_dot<F>(0.5, tx, ty, tz, sx, sy, sz);
        const bool ok = !G || not_coincident_half(hom);
        const double v = kernel(G ? safe_omc(ok, hom) : hom, tab);
        K[0] = ok ? v : 0.0;
    }
    template <bool G = true, bool F = false>
    __device__ __forceinline__ void eval(double tx, double ty, double tz, double sx, double sy, double sz, double sw,
                                         double* acc, const LogTable& tab) const {
        const double hom = one_minus_dot<F>(0.5, tx, ty, tz, sx, sy, sz);
        const bool ok = !G || not_coincident_half(hom);
        const double v = kernel(G ? safe_omc(ok, hom) : hom, tab);
        acc[0] = fma(ok ? sw : 0.0, v, acc[0]);
    }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc,
                                               const LogTable& tab) const {
        eval<true>(tx, ty, tz, sx, sy, sz, sw, acc, tab);
    }
};
using OpSal = OpSalT<false>;
using OpSalLog = OpSalT<true>;

// Calls f(op) with the device functor of a KernelSpec (kernel kind + SAL parameters).
template <class KS, class F>
void with_op(const KS& k, F&& f) {
    switch (k.kind) {
        case 0: f(OpLaplace{}); break;
        case 1: f(OpBiharmonic{}); break;
        case 2: f(OpBiotSavart{}); break;
        default: {
            const double pref = 3.0 * k.rho_ratio * kInv4Pi, c1 = 1.0 - k.b0, c2 = k.a1 - k.b1;
            if (c1 != 0.0) f(OpSal::make(pref, c1, c2));
            else f(OpSalLog::make(pref, c1, c2));
        }
    }
}

}  // namespace csfs_b200
