// Shared device helpers for the B200 CSFMM engine (sm_100a only).
//
// The numerics here restate the reference's L0 layer
// (/root/reference/proj/src/geometry.cpp:19-52, interpolation.cpp:14-68) in the
// operation order the reference's (non-FMA) build executes, so that tree
// topology, interaction lists and proxy bases agree with the reference's own
// csfmm_sum.  Only libm differences (glibc vs libdevice atan/tan/log, <=2 ulp)
// remain; SURVEY.md §0.7 shows the decision margins are >= 1e-7 relative.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace csfs_b200 {

constexpr int kMaxNp = 32;  // degree <= 31
constexpr double kPi = 3.14159265358979323846;
constexpr double kInv4Pi = 1.0 / (4.0 * kPi);
constexpr double kCoincidenceTol = 1e-14;  // kernels.hpp:28
constexpr double kNodeTol = 1e-14;         // interpolation.cpp:8
constexpr int kMaxDepth = 60;              // cluster_tree.cpp:11
constexpr double kMinExtent = 1e-13;       // cluster_tree.cpp:12
constexpr int kLogTabBits = 12;            // fastmath.cuh log table: 4096 mantissa intervals
constexpr int kLogTab = 1 << kLogTabBits;
constexpr int kLogTabWords = kLogTab;      // double2 words of the global table

// Error classes that map onto the C-ABI return codes (include/csfs_b200.h).
struct InvalidArgument : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    std::string msg = std::string(what) + " failed at " + file + ":" + std::to_string(line) +
                      ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) throw OutOfMemory(msg);
    throw CudaFailure(msg);
}
#define CSFS_CK(x) ::csfs_b200::cuda_check((x), #x, __FILE__, __LINE__)
// Every kernel launch of the engine goes through this check; it also counts launches so
// bench.py can report how many of OUR kernels ran in its timed region.
unsigned long long& launch_counter();
#define CSFS_LAUNCH_CHECK()                                                                  \
    do {                                                                                     \
        ++::csfs_b200::launch_counter();                                                     \
        ::csfs_b200::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);   \
    } while (0)

// Second-kind Chebyshev grid (interpolation.cpp:14-24), passed by value into kernels.
// Nodes/weights are computed on the host with the same libm call the reference makes
// (std::cos), so they are bit-identical to the reference's ChebyshevGrid1D.
struct Cheb {
    int np;
    double nodes[kMaxNp];
    double weights[kMaxNp];
};

// x.y exactly as the reference's non-contracted dot (geometry.hpp:19):
// ((ax*bx + ay*by) + az*bz), every product and sum rounded separately.
__device__ __forceinline__ double dot_ref(double ax, double ay, double az, double bx, double by,
                                          double bz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(ay, by)), __dmul_rn(az, bz));
}

// !(omc < kCoincidenceTol) (kernels.hpp:28) on the integer pipe: for IEEE doubles the
// signed 64-bit order of the bit patterns equals the numeric order on non-negative values,
// and every negative value (sign bit set, incl. -0.0) compares below the positive
// threshold, as it does numerically.  Saves a DSETP per pair on the FP64 pipe.
__device__ __forceinline__ bool not_coincident(double omc) {
    return __double_as_longlong(omc) >= __double_as_longlong(kCoincidenceTol);
}

// The same test on hom = omc / 2 (exact: functors that take halved targets, OpSalT).
__device__ __forceinline__ bool not_coincident_half(double hom) {
    return __double_as_longlong(hom) >= __double_as_longlong(0.5 * kCoincidenceTol);
}

// `ok ? omc : (a value in [1, 1 + 2^-20))` with a single 32-bit select: the skipped pair
// only needs a safe finite argument for the log / rsqrt / rcp that follow.
__device__ __forceinline__ double safe_omc(bool ok, double omc) {
    return __hiloint2double(ok ? __double2hiint(omc) : 0x3ff00000, __double2loint(omc));
}

// bary_basis_1d (interpolation.cpp:26-43), same node test, same summation order.
__device__ __forceinline__ void bary1d(const Cheb& c, double x, double* out) {
    const int np = c.np;
    int hit = -1;
    for (int k = 0; k < np; ++k)
        if (fabs(__dsub_rn(x, c.nodes[k])) < kNodeTol) {
            hit = k;
            break;
        }
    if (hit >= 0) {
        for (int j = 0; j < np; ++j) out[j] = (j == hit) ? 1.0 : 0.0;
        return;
    }
    double denom = 0.0;
    for (int k = 0; k < np; ++k) {
        const double q = __ddiv_rn(c.weights[k], __dsub_rn(x, c.nodes[k]));
        out[k] = q;
        denom = __dadd_rn(denom, q);
    }
    const double inv = __ddiv_rn(1.0, denom);
    for (int k = 0; k < np; ++k) out[k] = __dmul_rn(out[k], inv);
}

// CellInterpolant::ref_xi (interpolation.hpp:44-45)
__device__ __forceinline__ double ref_coord(double v, double mid, double half) {
    return half > 0.0 ? __ddiv_rn(__dsub_rn(v, mid), half) : 0.0;
}

// face_point_from_plane + face_unproject (geometry.cpp:37-52)
__device__ __forceinline__ void face_unproject(int face, double xi, double eta, double& x,
                                               double& y, double& z) {
    const double X = tan(xi), Y = tan(eta);
    const double s =
        __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(X, X)), __dmul_rn(Y, Y))));
    const double sX = __dmul_rn(s, X), sY = __dmul_rn(s, Y);
    switch (face) {
        case 0: x = s; y = sX; z = sY; break;
        case 1: x = -sX; y = s; z = sY; break;
        case 2: x = -s; y = -sX; z = sY; break;
        case 3: x = sX; y = -s; z = sY; break;
        case 4: x = -sY; y = sX; z = s; break;
        default: x = sY; y = sX; z = -s; break;
    }
}

// face_project (geometry.cpp:19-35): argmax over (x, y, -x, -y, z, -z) with strict '>'
// so ties go to the lowest face id; X/Y ratios then atan.
__device__ __forceinline__ void face_project(double px, double py, double pz, int& face,
                                             double& xi, double& eta) {
    // the running maximum in a register (an indexed v[6] lives in local memory: 37% of
    // k_face_label's stall samples, ncu round 2); the same comparisons in the same order
    int f = 0;
    double m = px;
    if (py > m) { f = 1; m = py; }
    if (-px > m) { f = 2; m = -px; }
    if (-py > m) { f = 3; m = -py; }
    if (pz > m) { f = 4; m = pz; }
    if (-pz > m) { f = 5; m = -pz; }
    // X = nx / den, Y = ny / den with the reference's operands per face (:26-33)
    double nx, ny, den;
    switch (f) {
        case 0: nx = py; ny = pz; den = px; break;
        case 1: nx = -px; ny = pz; den = py; break;
        case 2: nx = py; ny = -pz; den = px; break;
        case 3: nx = -px; ny = -pz; den = py; break;
        case 4: nx = py; ny = -px; den = pz; break;
        default: nx = -py; ny = -px; den = pz; break;
    }
    const double X = __ddiv_rn(nx, den), Y = __ddiv_rn(ny, den);
    face = f;
    xi = atan(X);
    eta = atan(Y);
}

// Order-preserving map of doubles onto uint64 so min/max reductions can use integer
// atomics (exact, order independent, hence deterministic).
__device__ __forceinline__ unsigned long long ord_enc(double v) {
    unsigned long long u = __double_as_longlong(v);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double ord_dec(unsigned long long u) {
    u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
    double d;
    memcpy(&d, &u, sizeof d);
    return d;
}

inline int ceil_div(long long a, long long b) { return int((a + b - 1) / b); }

}  // namespace csfs_b200
