// Device-resident RK4 stage arithmetic of the barotropic vorticity driver
// bve_step (/root/reference/proj/src/applications.cpp:378-412, remesh off): the four
// Biot-Savart CSFMM evaluations run on the device (csfs_b200_bve_step, capi.cu) and the
// stage updates below keep positions/vorticity in HBM between them, in the reference's
// operation order (Vec3 ops geometry.hpp:16-23, normalized = a / sqrt(dot(a, a))).
#include "engine.hpp"

namespace csfs_b200 {

namespace {

__device__ __forceinline__ void normalize_ref(double& x, double& y, double& z) {
    const double n = __dsqrt_rn(dot_ref(x, y, z, x, y, z));
    x = __ddiv_rn(x, n);
    y = __ddiv_rn(y, n);
    z = __ddiv_rn(z, n);
}

// w = zeta * area (biot_savart_velocity, applications.cpp:188)
__global__ void k_weights(long long n, const double* __restrict__ zeta, const double* __restrict__ area,
                          double* __restrict__ w) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) w[i] = __dmul_rn(zeta[i], area[i]);
}

// advance (applications.cpp:388-393): pos = normalized(x0 + h k), zeta = zeta0 - 2 Omega h k.z,
// fused with the next stage's weights w = zeta * area.
__global__ void k_advance(long long n, const double* __restrict__ x0, const double* __restrict__ z0,
                          const double* __restrict__ k, double h, double omega, const double* __restrict__ area,
                          double* __restrict__ pos, double* __restrict__ zeta, double* __restrict__ w) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double kx = k[3 * i], ky = k[3 * i + 1], kz = k[3 * i + 2];
    double x = __dadd_rn(x0[3 * i], __dmul_rn(h, kx));
    double y = __dadd_rn(x0[3 * i + 1], __dmul_rn(h, ky));
    double z = __dadd_rn(x0[3 * i + 2], __dmul_rn(h, kz));
    normalize_ref(x, y, z);
    pos[3 * i] = x;
    pos[3 * i + 1] = y;
    pos[3 * i + 2] = z;
    const double zt = __dsub_rn(z0[i], __dmul_rn(__dmul_rn(__dmul_rn(2.0, omega), h), kz));
    zeta[i] = zt;
    w[i] = __dmul_rn(zt, area[i]);
}

// final update (applications.cpp:404-408):
// du = (dt/6) * (k1 + 2 k2 + 2 k3 + k4); x = normalized(x + du); zeta -= 2 Omega du.z
__global__ void k_rk4_final(long long n, double* __restrict__ x, double* __restrict__ zeta,
                            const double* __restrict__ k1, const double* __restrict__ k2,
                            const double* __restrict__ k3, const double* __restrict__ k4, double dt,
                            double omega) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c = dt / 6.0;
    double du[3];
    for (int d = 0; d < 3; ++d) {
        const long long j = 3 * i + d;
        const double s = __dadd_rn(__dadd_rn(__dadd_rn(k1[j], __dmul_rn(2.0, k2[j])), __dmul_rn(2.0, k3[j])), k4[j]);
        du[d] = __dmul_rn(c, s);
    }
    double px = __dadd_rn(x[3 * i], du[0]);
    double py = __dadd_rn(x[3 * i + 1], du[1]);
    double pz = __dadd_rn(x[3 * i + 2], du[2]);
    normalize_ref(px, py, pz);
    x[3 * i] = px;
    x[3 * i + 1] = py;
    x[3 * i + 2] = pz;
    zeta[i] = __dsub_rn(zeta[i], __dmul_rn(__dmul_rn(2.0, omega), du[2]));
}

}  // namespace

void bve_weights(long long n, const double* zeta, const double* area, double* w, cudaStream_t s) {
    k_weights<<<ceil_div(n, 256), 256, 0, s>>>(n, zeta, area, w);
    CSFS_LAUNCH_CHECK();
}

void bve_advance(long long n, const double* x0, const double* z0, const double* k, double h, double omega,
                 const double* area, double* pos, double* zeta, double* w, cudaStream_t s) {
    k_advance<<<ceil_div(n, 256), 256, 0, s>>>(n, x0, z0, k, h, omega, area, pos, zeta, w);
    CSFS_LAUNCH_CHECK();
}

void bve_final(long long n, double* x, double* zeta, const double* k1, const double* k2, const double* k3,
               const double* k4, double dt, double omega, cudaStream_t s) {
    k_rk4_final<<<ceil_div(n, 256), 256, 0, s>>>(n, x, zeta, k1, k2, k3, k4, dt, omega);
    CSFS_LAUNCH_CHECK();
}

}  // namespace csfs_b200
