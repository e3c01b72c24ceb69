// Device kernel functors: the B200 form of the reference's private ops
// LaplaceOp / BiharmonicOp / BiotSavartOp / SalOp (/root/reference/proj/src/summation.cpp:32-77)
// and of dilog (kernels.cpp:13-51).
//
// Same shape as the reference op (static dim; evaluate one (x, y) pair and accumulate
// w * K(x, y)), with two B200-specific changes that do not alter the value beyond
// roundoff:
//  * the coincidence guard `1 - x.y < 1e-14` is predicated (a safe argument is
//    evaluated and the weight is zeroed) instead of branched, so a warp never diverges;
//  * the constant prefactor (-1/4pi, 1/4pi, 3 rho/4pi) is applied once per target by
//    the caller (`scale`) instead of once per pair.
// `x.y` and `1 - x.y` are evaluated unfused in the reference's order (dot_ref), which
// keeps the near-neighbour cancellation identical to the reference's build
// (contraction alone moves results by up to 1.1e-11).
#pragma once

#include "common.cuh"

namespace csfs_b200 {

struct OpLaplace {
    static constexpr int dim = 1;
    __device__ __forceinline__ double scale() const { return -kInv4Pi; }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc) const {
        const double omc = __dsub_rn(1.0, dot_ref(tx, ty, tz, sx, sy, sz));
        const bool ok = !(omc < kCoincidenceTol);
        const double v = log(ok ? omc : 1.0);
        acc[0] = fma(ok ? sw : 0.0, v, acc[0]);
    }
};

// Li2 on the kernel's domain u in [0, 1] (u = min(1, (1 + x.y)/2) >= -1e-16).
// Reference (kernels.cpp:13-51): reflection Li2(u) = pi^2/6 - ln(u) ln(1-u) - Li2(1-u) for
// u > 1/2, then the power series of Li2 on [0, 1/2] (up to 80 terms, each a division).
// Here the base region uses the Bernoulli series Li2(y) = sum_n B_n z^(n+1)/(n+1)! with
// z = -ln(1-y) in [0, ln 2]: 10 terms reach < 2e-17 relative, as a degree-9 Horner
// polynomial in z^2 (no divisions).  For u > 1/2, z = -ln(u) is the log already needed
// by the reflection term, so that branch costs two logs, the other one.
__device__ __forceinline__ double li2_bernoulli(double z) {
    const double w = z * z;
    double p = -0x1.7e168b15d7793p-57;  // B20/21!
    p = fma(p, w, 0x1.04805fdce7819p-51);
    p = fma(p, w, -0x1.6731c59dbd7dep-46);
    p = fma(p, w, 0x1.f63f1e311ac24p-41);
    p = fma(p, w, -0x1.658a4b8f16a75p-35);
    p = fma(p, w, 0x1.04d7f65caf373p-29);
    p = fma(p, w, -0x1.8a86a49f629d1p-24);
    p = fma(p, w, 0x1.3d079fb6ef3e3p-18);
    p = fma(p, w, -0x1.23456789abcdfp-12);
    p = fma(p, w, 0x1.c71c71c71c71cp-6);  // B2/3! = 1/36
    // z - z^2/4 + z^3 p(z^2)
    return fma(z * w, p, fma(-0.25 * z, z, z));
}

__device__ __forceinline__ double dilog_dev(double u) {
    constexpr double kPi2Over6 = kPi * kPi / 6.0;
    if (u > 0.5) {
        const double y = 1.0 - u;  // exact (Sterbenz)
        const double lu = log(u);
        const double ly = log(y);
        const double r = kPi2Over6 - lu * ly - li2_bernoulli(-lu);
        return (u == 1.0) ? kPi2Over6 : r;
    }
    // z = -log1p(-u) via the compensated form log(t) - ((t - 1) + u)/t, t = 1 - u
    const double t = 1.0 - u;
    const double z = -(log(t) - ((t - 1.0) + u) / t);
    return li2_bernoulli(z);
}

struct OpBiharmonic {
    static constexpr int dim = 1;
    __device__ __forceinline__ double scale() const { return kInv4Pi; }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc) const {
        const double d = dot_ref(tx, ty, tz, sx, sy, sz);
        const double u0 = __dmul_rn(0.5, __dadd_rn(1.0, d));
        const double u = (u0 < 1.0) ? u0 : 1.0;  // std::min(1.0, u0)
        acc[0] = fma(sw, dilog_dev(u), acc[0]);
    }
};

struct OpBiotSavart {
    static constexpr int dim = 3;
    __device__ __forceinline__ double scale() const { return -kInv4Pi; }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc) const {
        const double omc = __dsub_rn(1.0, dot_ref(tx, ty, tz, sx, sy, sz));
        const bool ok = !(omc < kCoincidenceTol);
        const double a = (ok ? sw : 0.0) / (ok ? omc : 1.0);
        const double cx = ty * sz - tz * sy;
        const double cy = tz * sx - tx * sz;
        const double cz = tx * sy - ty * sx;
        acc[0] = fma(a, cx, acc[0]);
        acc[1] = fma(a, cy, acc[1]);
        acc[2] = fma(a, cz, acc[2]);
    }
};

struct OpSal {
    static constexpr int dim = 1;
    double pref, c1, c2;  // SalOp (summation.cpp:64-68)
    __device__ __forceinline__ double scale() const { return pref; }
    __device__ __forceinline__ void operator()(double tx, double ty, double tz, double sx, double sy,
                                               double sz, double sw, double* acc) const {
        const double omc = __dsub_rn(1.0, dot_ref(tx, ty, tz, sx, sy, sz));
        const bool ok = !(omc < kCoincidenceTol);
        const double g2 = 2.0 * (ok ? omc : 1.0);
        const double gamma = sqrt(g2);
        const double s = 0.5 * gamma;
        const double v = c1 / gamma - c2 * log(s * (1.0 + s));
        acc[0] = fma(ok ? sw : 0.0, v, acc[0]);
    }
};

}  // namespace csfs_b200
