// Scattered-data remesh of the barotropic vorticity driver: bve_remesh
// (/root/reference/proj/src/applications.cpp:329-371, with SphereBuckets :198-263 and
// quadratic_fit_at_center :267-325).  For every grid centre: its k nearest deformed
// particles (k = min(max(neighbors, 6), n)) found through lat-lon buckets, a Gaussian-
// weighted 6-term quadratic least-squares fit in the centre's face-local (xi, eta), and
// the fit evaluated at the centre.
//
// B200 layout: the particles are bucketed once per call (one counting pass + a scan + an
// atomic fill, then each bucket's indices sorted ascending so every later step is
// deterministic), and one thread per grid centre runs the ring search, a register-resident
// top-k (key (d^2, index), the order std::partial_sort on pairs gives), and the 6x6 solve.
// This file is compiled with -fmad=false: the reference build does not contract, and the
// ring cut-offs, pivots and the singular-stencil fallback compare rounded values.
#include <algorithm>
#include <cmath>

#include "engine.hpp"
#include "scan.cuh"

namespace csfs_b200 {

namespace {

constexpr double kTwoPi = 2.0 * kPi;

struct Buckets {
    int rows, cols;
    const int* start;  // rows*cols + 1 offsets into idx
    const int* idx;    // particle indices, ascending within a bucket
};

// SphereBuckets::row_of / col_of (applications.cpp:234-242)
__device__ __forceinline__ int row_of(double z, int rows) {
    const double th = acos(fmin(fmax(z, -1.0), 1.0));
    return min(rows - 1, int(th / kPi * rows));
}
__device__ __forceinline__ int col_of(double x, double y, int cols) {
    double lon = atan2(y, x);
    if (lon < 0) lon += kTwoPi;
    return min(cols - 1, int(lon / kTwoPi * cols));
}

__global__ void k_bucket_count(long long n, const double* __restrict__ xyz, int rows, int cols,
                               int* __restrict__ bucket, int* __restrict__ count) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    const int b = row_of(z, rows) * cols + col_of(x, y, cols);
    bucket[i] = b;
    atomicAdd(&count[b], 1);
}

__global__ void k_bucket_fill(long long n, const int* __restrict__ bucket, const int* __restrict__ start,
                              int* __restrict__ cursor, int* __restrict__ idx) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = bucket[i];
    idx[start[b] + atomicAdd(&cursor[b], 1)] = int(i);
}

// each bucket ascending (the reference fills its buckets in index order)
__global__ void k_bucket_sort(int nb, const int* __restrict__ start, int* __restrict__ idx) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int s = start[b], e = start[b + 1];
    for (int a = s + 1; a < e; ++a) {
        const int v = idx[a];
        int c = a - 1;
        while (c >= s && idx[c] > v) {
            idx[c + 1] = idx[c];
            --c;
        }
        idx[c + 1] = v;
    }
}

// Visits the cells of ring `ring` around (bi, bj) in the reference's order
// (gather_ring, applications.cpp:246-258); f(bucket) per cell, columns wrap.
template <class F>
__device__ __forceinline__ void for_ring(const Buckets& B, int bi, int bj, int ring, F&& f) {
    for (int di = -ring; di <= ring; ++di) {
        const int i = bi + di;
        if (i < 0 || i >= B.rows) continue;
        const bool edge_row = (di == -ring || di == ring);
        for (int dj = -ring; dj <= ring; dj += (edge_row || dj == ring) ? 1 : 2 * ring) {
            const int j = ((bj + dj) % B.cols + B.cols) % B.cols;
            f(i * B.cols + j);
        }
    }
}

// face_plane_coords (geometry.cpp:54-66)
__device__ __forceinline__ bool face_plane(int face, double px, double py, double pz, double& X, double& Y) {
    double axis;
    switch (face) {
        case 0: axis = px; X = py / px; Y = pz / px; break;
        case 1: axis = py; X = -px / py; Y = pz / py; break;
        case 2: axis = -px; X = py / px; Y = -pz / px; break;
        case 3: axis = -py; X = -px / py; Y = -pz / py; break;
        case 4: axis = pz; X = py / pz; Y = -px / pz; break;
        default: axis = -pz; X = -py / pz; Y = -px / pz; break;
    }
    return axis > 1e-12;
}

// One usable neighbour's stencil entry: (du, dv) in the centre's face-local angles.
struct Stencil {
    int face;
    double xi, eta;
    const double* pos;
    __device__ __forceinline__ void at(int j, double& du, double& dv) const {
        double X, Y;
        face_plane(face, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], X, Y);
        du = atan(X) - xi;
        dv = atan(Y) - eta;
    }
};

// quadratic_fit_at_center (applications.cpp:267-325) with the Gaussian weights of
// bve_remesh (:357-362): w_s = exp(-4 r_s^2 / d0), d0 = max(max_s r_s^2, 1e-30); normal
// equations of {1, x, y, x^2, xy, y^2} (x = du/h, y = dv/h, h = sqrt(max r^2)), Gaussian
// elimination with partial pivoting; a pivot below 1e-10 * A00 falls back to the weighted
// mean.  The stencil (usable neighbour ids uj[0..m)) is re-derived per pass instead of
// being kept in per-thread arrays: same values, a fraction of the local-memory traffic.
// f(j): the field at particle j.  Returns the fit at the centre.
template <class F>
__device__ double quadratic_fit(const Stencil& st, int m, const int* uj, F&& f) {
    constexpr int M = 6;
    double scale = 0.0;
    for (int s = 0; s < m; ++s) {
        double du, dv;
        st.at(uj[s], du, dv);
        scale = fmax(scale, du * du + dv * dv);
    }
    const double d0 = fmax(scale, 1e-30);
    const double h = sqrt(fmax(scale, 1e-30));
    double A[M][M], b[M];
    for (int i = 0; i < M; ++i) {
        b[i] = 0.0;
        for (int j = 0; j < M; ++j) A[i][j] = 0.0;
    }
    for (int s = 0; s < m; ++s) {
        double du, dv;
        st.at(uj[s], du, dv);
        const double wgt = exp(-4.0 * (du * du + dv * dv) / d0);
        const double fs = f(uj[s]);
        const double x = du / h, y = dv / h;
        const double row[M] = {1.0, x, y, x * x, x * y, y * y};
#pragma unroll
        for (int i = 0; i < M; ++i) {
            b[i] += wgt * row[i] * fs;
#pragma unroll
            for (int j = i; j < M; ++j) A[i][j] += wgt * row[i] * row[j];
        }
    }
#pragma unroll
    for (int i = 1; i < M; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) A[i][j] = A[j][i];
    const double diag_scale = A[0][0];
#pragma unroll
    for (int col = 0; col < M; ++col) {
        int best = col;
#pragma unroll
        for (int r = col + 1; r < M; ++r)
            if (fabs(A[r][col]) > fabs(A[best][col])) best = r;
        if (best != col) {
#pragma unroll
            for (int r = col + 1; r < M; ++r)
                if (r == best) {
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        const double t = A[col][j];
                        A[col][j] = A[r][j];
                        A[r][j] = t;
                    }
                    const double t = b[col];
                    b[col] = b[r];
                    b[r] = t;
                }
        }
        const double d = A[col][col];
        if (fabs(d) < 1e-10 * diag_scale) {  // weight-starved or collinear stencil: weighted mean
            double num = 0.0, den = 0.0;
            for (int s = 0; s < m; ++s) {
                double du, dv;
                st.at(uj[s], du, dv);
                const double wgt = exp(-4.0 * (du * du + dv * dv) / d0);
                num += wgt * f(uj[s]);
                den += wgt;
            }
            return den > 0.0 ? num / den : (m == 0 ? 0.0 : f(uj[0]));
        }
#pragma unroll
        for (int r = col + 1; r < M; ++r) {
            const double fac = A[r][col] / d;
#pragma unroll
            for (int j = col; j < M; ++j) A[r][j] -= fac * A[col][j];
            b[r] -= fac * b[col];
        }
    }
    double x[M];
#pragma unroll
    for (int i = M - 1; i >= 0; --i) {
        double s = b[i];
#pragma unroll
        for (int j = i + 1; j < M; ++j) s -= A[i][j] * x[j];
        x[i] = s / A[i][i];
    }
    return x[0];
}

__global__ void __launch_bounds__(128) k_remesh(long long n, int k, Buckets B, const double* __restrict__ pos,
                                                const double* __restrict__ zeta, const double* __restrict__ tracer,
                                                const double* __restrict__ grid, double* __restrict__ new_zeta,
                                                double* __restrict__ new_tracer) {
    const long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= n) return;
    const double qx = grid[3 * gi], qy = grid[3 * gi + 1], qz = grid[3 * gi + 2];
    int face;
    double xi, eta;
    face_project(qx, qy, qz, face, xi, eta);
    const int bi = row_of(qz, B.rows), bj = col_of(qx, qy, B.cols);

    // knn (applications.cpp:208-231): rings until >= k candidates (counted with repeats,
    // ring >= 1), then one more ring; the k smallest (d^2, index) among the candidates
    int ring = 0;
    long long cand = 0;
    const int max_ring = max(B.rows, B.cols / 2);
    while (ring <= max_ring) {
        for_ring(B, bi, bj, ring, [&](int c) { cand += B.start[c + 1] - B.start[c]; });
        if (cand >= k && ring >= 1) break;
        ++ring;
    }
    double kd[kRemeshMaxK];
    int ki[kRemeshMaxK];
    int cnt = 0;
    // rings 0..ring already counted (0..max_ring when the loop ran out), plus ring + 1
    const int last_counted = ring <= max_ring ? ring : max_ring;
    for (int rr = 0; rr <= last_counted + 1; ++rr) {
        const int rg = rr <= last_counted ? rr : ring + 1;
        for_ring(B, bi, bj, rg, [&](int c) {
            for (int a = B.start[c]; a < B.start[c + 1]; ++a) {
                const int id = B.idx[a];
                const double dx = pos[3 * id] - qx, dy = pos[3 * id + 1] - qy, dz = pos[3 * id + 2] - qz;
                const double d = dx * dx + dy * dy + dz * dz;
                if (cnt == k && (d > kd[k - 1] || (d == kd[k - 1] && id >= ki[k - 1]))) continue;
                int p = cnt;
                while (p > 0 && (kd[p - 1] > d || (kd[p - 1] == d && ki[p - 1] > id))) --p;
                if (p > 0 && kd[p - 1] == d && ki[p - 1] == id) continue;  // repeated cell (column wrap)
                for (int q = (cnt < k ? cnt : k - 1); q > p; --q) {
                    kd[q] = kd[q - 1];
                    ki[q] = ki[q - 1];
                }
                kd[p] = d;
                ki[p] = id;
                if (cnt < k) ++cnt;
            }
        });
    }

    // stencil in the centre's face plane (applications.cpp:341-350): the usable neighbours
    int uj[kRemeshMaxK];
    int m = 0;
    for (int s = 0; s < cnt; ++s) {
        const int j = ki[s];
        double X, Y;
        if (face_plane(face, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], X, Y)) uj[m++] = j;
    }
    if (m < 6) {  // not enough usable neighbours: nearest value
        new_zeta[gi] = cnt == 0 ? zeta[gi] : zeta[ki[0]];
        if (tracer) new_tracer[gi] = cnt == 0 ? tracer[gi] : tracer[ki[0]];
        return;
    }
    const Stencil st{face, xi, eta, pos};
    new_zeta[gi] = quadratic_fit(st, m, uj, [&](int j) { return zeta[j]; });
    if (tracer) new_tracer[gi] = quadratic_fit(st, m, uj, [&](int j) { return tracer[j]; });
}

}  // namespace

void bve_remesh(double* xyz, double* zeta, double* tracer, const double* grid, long long n, int neighbors,
                DevBuf<int>& ibuf, DevBuf<double>& dbuf, cudaStream_t s) {
    if (n <= 0) return;
    const int k = int(std::min<long long>(std::max(neighbors, 6), n));
    const int rows = std::max(4, int(std::sqrt(double(n) / 8.0)));  // SphereBuckets ctor (:201-202)
    const int cols = 2 * rows;
    const int nb = rows * cols;
    ibuf.grow(size_t(2 * n + 2 * (nb + 1)) + size_t(scan_tile_ints(nb, 1)) + 1);
    int* bucket = ibuf.p;
    int* idx = bucket + n;
    int* count = idx + n;   // nb + 1 (then reused as the fill cursor)
    int* start = count + nb + 1;
    int* tiles = start + nb + 1;
    int* grand = tiles + scan_tile_ints(nb, 1);
    dbuf.grow(size_t(2 * n));
    double* nz = dbuf.p;
    double* nt = dbuf.p + n;
    CSFS_CK(cudaMemsetAsync(count, 0, (nb + 1) * sizeof(int), s));
    k_bucket_count<<<ceil_div(n, 256), 256, 0, s>>>(n, xyz, rows, cols, bucket, count);
    CSFS_LAUNCH_CHECK();
    run_scan<1>(
        nb + 1, [count] __device__(long long i, int* c) { c[0] = count[i]; },
        [start] __device__(long long i, const int*, const int* pre) { start[i] = pre[0]; }, tiles, grand, s);
    CSFS_CK(cudaMemsetAsync(count, 0, (nb + 1) * sizeof(int), s));
    k_bucket_fill<<<ceil_div(n, 256), 256, 0, s>>>(n, bucket, start, count, idx);
    CSFS_LAUNCH_CHECK();
    k_bucket_sort<<<ceil_div(nb, 256), 256, 0, s>>>(nb, start, idx);
    CSFS_LAUNCH_CHECK();
    const Buckets B{rows, cols, start, idx};
    k_remesh<<<ceil_div(n, 128), 128, 0, s>>>(n, k, B, xyz, zeta, tracer, grid, nz, nt);
    CSFS_LAUNCH_CHECK();
    // state.positions = grid_centers; zeta (and tracer) <- the fitted values (:368-370)
    CSFS_CK(cudaMemcpyAsync(xyz, grid, size_t(3 * n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CSFS_CK(cudaMemcpyAsync(zeta, nz, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (tracer) CSFS_CK(cudaMemcpyAsync(tracer, nt, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

}  // namespace csfs_b200
