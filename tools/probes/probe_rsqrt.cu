// Developer probe: accuracy of the MUFU.RSQ64H seed (rsqrt.approx.ftz.f64) and of one
// quadratic / cubic Newton step from it, over x in [1e-6, 4) (the SAL kernel's 2(1 - x.y)
// range on far entries down to the guard), measured against 1/sqrt in long double on the
// host.  The question behind the SAL functor's rsqrt step (kernels_dev.cuh).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/probe_rsqrt.cu -o tools/probes/probe_rsqrt
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void k_rsqrt(const double* x, double* seed, double* quad, double* cubic, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = x[i];
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
    seed[i] = y;
    const double h = v * y;
    quad[i] = y * fma(-0.5 * h, y, 1.5);
    const double e = fma(-h, y, 1.0);
    cubic[i] = fma(y, e * fma(e, 0.375, 0.5), y);
}

int main() {
    const int n = 1 << 22;
    std::vector<double> x(n);
    srand(7);
    for (int i = 0; i < n; ++i) {  // log-uniform over [1e-6, 4)
        const double u = (rand() + 0.5) / (RAND_MAX + 1.0);
        x[i] = 1e-6 * std::pow(4e6, u);
    }
    double *dx, *ds, *dq, *dc;
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&ds, n * 8);
    cudaMalloc(&dq, n * 8);
    cudaMalloc(&dc, n * 8);
    cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
    k_rsqrt<<<(n + 255) / 256, 256>>>(dx, ds, dq, dc, n);
    std::vector<double> s(n), q(n), c(n);
    cudaMemcpy(s.data(), ds, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(q.data(), dq, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(c.data(), dc, n * 8, cudaMemcpyDeviceToHost);
    double ms = 0, mq = 0, mc = 0, bq = 0;
    for (int i = 0; i < n; ++i) {
        const long double r = 1.0L / sqrtl((long double)x[i]);
        const double es = (double)fabsl((s[i] - r) / r), eq = (double)((q[i] - r) / r),
                     ec = (double)fabsl((c[i] - r) / r);
        ms = es > ms ? es : ms;
        mq = fabs(eq) > mq ? fabs(eq) : mq;
        bq += eq;
        mc = ec > mc ? ec : mc;
    }
    printf("seed max rel %.3e (2^%.2f)\nquadratic max rel %.3e, mean signed %.3e\ncubic max rel %.3e\n", ms,
           std::log2(ms), mq, bq / n, mc);
    return 0;
}
